mkdir -p gpurun_out/s2c
timeout 600 python -m pytest tests/ -q -m gpu -x --timeout 180 -p no:cacheprovider > gpurun_out/s2c/tests.log 2>&1; echo "tests $?" >> gpurun_out/s2c/summary.txt
for v in main poly0 poly2 poly3; do
  if [ $v = main ]; then lib=""; else lib=paper_2110_10221_b200/variants/lib$v.so; fi
  CORA_LIB_PATH=$lib timeout 300 python scripts/time_attention.py C4-wiki512,C3,C2-mnli 50 > gpurun_out/s2c/attn_$v.txt 2>&1
done
CORA_DEBUG=1 timeout 300 python scripts/time_layer.py C4-wiki512 200 > gpurun_out/s2c/layer.txt 2>&1
cat gpurun_out/s2c/summary.txt gpurun_out/s2c/attn_*.txt gpurun_out/s2c/layer.txt
