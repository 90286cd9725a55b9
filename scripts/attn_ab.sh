#!/bin/bash
# A/B of attention library variants in one GPU call, alternating, twice: "cur" = the in-tree library,
# other names = variants/<name>.so (built with paper_2110_10221_b200/build.py -D... --out=variants/<name>.so)
CFGS=${CFGS:-L4096x32,C4-wiki512}
for rep in 1 2; do
  for v in "$@"; do
    case $v in
      cur) CAUSAL=0 timeout 100 python scripts/attn_probe.py $CFGS 20 | sed "s/^/$v  /" ;;
      *) CORA_LIB_PATH=variants/$v.so CAUSAL=0 timeout 100 python scripts/attn_probe.py $CFGS 20 | sed "s/^/$v  /" ;;
    esac
  done
done
