#!/bin/bash
# A/B: the fused LN GEMMs with the rows of their last partial wave on the spare SMs (default) vs without
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "layer or forward or stack" --timeout 300 -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2; do
  timeout 120 python scripts/time_layer.py C4-wiki512 2>&1 | tail -2 | sed "s/^/spare   /"
  CORA_NO_SPARE_SMS=1 timeout 120 python scripts/time_layer.py C4-wiki512 2>&1 | tail -2 | sed "s/^/nospare /"
done
