CFGS=C2-mnli,ds:mnli:128,ds:cola:128,ds:cola:512,ds:mrpc:128,C3
for v in pack nopack; do
  if [ $v = pack ]; then lib=""; else lib=paper_2110_10221_b200/variants/libnopack.so; fi
  echo "== $v"
  CORA_LIB_PATH=$lib python scripts/time_attention.py $CFGS 30 2>&1 | grep attention
  CORA_LIB_PATH=$lib python scripts/time_prelude.py $CFGS 2>&1 | grep prelude
  for c in ds:mnli:128 ds:cola:512; do CORA_LIB_PATH=$lib python scripts/time_layer.py $c 50 2>&1 | grep no-events; done
done
