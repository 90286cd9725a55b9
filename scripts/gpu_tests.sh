#!/bin/bash
# run GPU test groups separately so a hang in one group does not hide the others
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
for k in layout layernorm softmax linear attention layer; do
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "$k" --timeout 180 -p no:cacheprovider > gpurun_out/t_$k.log 2>&1
  echo "$k exit $?" >> gpurun_out/summary.txt
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
