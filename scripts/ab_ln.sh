#!/bin/bash
# A/B of the fused GEMM + LayerNorm variants (CORA_LN_FULLROW = 0 / 1 / 2) on the layer step: GPU parity of the
# fused-LN tests for each, then the layer time (scripts/time_layer.py) alternating
for v in 3; do
  CORA_LN_FULLROW=$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "layernorm_fused or large_mean or layer_c3 or full_batch or aligned" --timeout 120 -p no:cacheprovider 2>&1 | tail -1 | sed "s/^/fullrow=$v tests: /"
done
for rep in 1 2; do
  for v in 0 3; do
    CORA_LN_FULLROW=$v timeout 120 python scripts/time_layer.py C4-wiki512 2>&1 | tail -3 | sed "s/^/fullrow=$v /"
  done
done
