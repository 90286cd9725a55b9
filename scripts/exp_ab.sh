#!/bin/bash
# A/B of library variants in variants/*.so: shard makespans (time_shards) twice, alternating
mkdir -p gpurun_out
out=gpurun_out/ab.txt
rm -f $out
for i in 1 2; do
  for v in "$@"; do
    echo "== $v" >> $out
    CORA_LIB_PATH=variants/$v.so timeout 300 python scripts/time_shards.py C4-wiki512 30 >> $out 2>&1
  done
done
cat $out
