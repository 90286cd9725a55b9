#!/bin/bash
# A/B of library variants (variants/<name>.so) on the attention kernel alone, twice, alternating
mkdir -p gpurun_out
out=gpurun_out/attn_ab.txt
rm -f $out
for i in 1 2; do
  for v in "$@"; do
    echo "== $v" >> $out
    CORA_LIB_PATH=variants/$v.so timeout 300 python scripts/time_attention.py C4-wiki512,C3,ds:cola:512 50 >> $out 2>&1
  done
done
cat $out
