mkdir -p gpurun_out
for i in 1 2; do
for v in base ffma2; do
  echo "== $v" >> gpurun_out/attn_ab.txt
  CORA_LIB_PATH=variants/$v.so timeout 300 python scripts/time_attention.py C4-wiki512,C3,ds:cola:512 50 >> gpurun_out/attn_ab.txt 2>&1
done
done
cat gpurun_out/attn_ab.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "attention" -p no:cacheprovider 2>&1 | tail -2 >> gpurun_out/attn_ab.txt
