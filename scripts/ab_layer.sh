#!/bin/bash
# A/B of library variants (variants/<name>.so) on the graph-captured C4 step, alternating, 3 rounds.
#   bash scripts/ab_layer.sh cur prev [config]
mkdir -p gpurun_out
out=gpurun_out/ab_layer.txt
rm -f $out
cfg=${CFG:-C4-wiki512}
for i in 1 2 3; do
  for v in "$@"; do
    echo "== $v" >> $out
    CORA_LIB_PATH=variants/$v.so timeout 300 python scripts/time_layer.py $cfg 200 >> $out 2>&1
  done
done
cat $out
