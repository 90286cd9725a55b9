mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "attention" --timeout 300 -p no:cacheprovider > gpurun_out/t_attn.log 2>&1
echo "attn tests exit $?" > gpurun_out/attn_ab.txt
tail -3 gpurun_out/t_attn.log >> gpurun_out/attn_ab.txt
for i in 1 2; do for v in prev cur; do echo "== $v" >> gpurun_out/attn_ab.txt; CORA_LIB_PATH=variants/$v.so timeout 120 python scripts/time_attention.py C4-wiki512,C3,C2-mnli 50 >> gpurun_out/attn_ab.txt 2>&1; done; done
for i in 1 2; do for v in prev cur; do echo "== $v" >> gpurun_out/attn_ab.txt; CORA_LIB_PATH=variants/$v.so timeout 300 python scripts/time_layer.py C4-wiki512 200 >> gpurun_out/attn_ab.txt 2>&1; done; done
