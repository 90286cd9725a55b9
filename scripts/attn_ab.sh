#!/bin/bash
# A/B of attention variants in one GPU call, alternating, twice: "old" = the two-CTA kernel of the
# in-tree library (CORA_ATTN_PP=0), "cur" = the in-tree library, other names = variants/<name>.so
CFGS=${CFGS:-L4096x32,C4-wiki512}
for rep in 1 2; do
  for v in "$@"; do
    case $v in
      old) CORA_ATTN_PP=0 CAUSAL=0 timeout 100 python scripts/attn_probe.py $CFGS 20 | sed "s/^/$v  /" ;;
      cur) CAUSAL=0 timeout 100 python scripts/attn_probe.py $CFGS 20 | sed "s/^/$v  /" ;;
      *) CORA_LIB_PATH=variants/$v.so CAUSAL=0 timeout 100 python scripts/attn_probe.py $CFGS 20 | sed "s/^/$v  /" ;;
    esac
  done
done
