#!/bin/bash
# attention A/B over library variants (variants/<name>.so), alternating, 2 rounds: time_attention.py
out=gpurun_out/attn_var_ab.txt
: > $out
for i in 1 2; do for v in "$@"; do echo "== $v" >> $out; CORA_LIB_PATH=variants/$v.so timeout 120 python scripts/time_attention.py ${CFGS:-C4-wiki512,C3,C2-mnli} 50 >> $out 2>&1; done; done
cat $out
