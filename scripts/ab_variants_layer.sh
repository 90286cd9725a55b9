#!/bin/bash
# A/B of library variants (variants/<name>.so) on the layer step (scripts/time_layer.py), alternating, twice
for rep in 1 2; do
  for v in "$@"; do
    CORA_LIB_PATH=variants/$v.so timeout 120 python scripts/time_layer.py ${CFG:-C4-wiki512} 2>&1 | tail -2 | sed "s/^/$v  /"
  done
done
