#!/bin/bash
# Attention development loop on one GPU call: attention parity tests, then the probe (bidirectional and causal).
mkdir -p gpurun_out/dev
OUT=gpurun_out/dev
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "attention or layer_c3 or full_batch" --timeout 120 -p no:cacheprovider > $OUT/tests.log 2>&1
echo "tests exit $?"; tail -3 $OUT/tests.log
CFGS=${CFGS:-L512x256,L4096x32,C4-wiki512,C3,ds:race:128,ds:mnli:128,ds:cola:512}
timeout 300 python scripts/attn_probe.py $CFGS 20 2>&1
