#!/bin/bash
# e2e (host buffers) with and without the cached graph, and the chunk count sweep
for k in 8 16; do
  echo "chunks $k graph"; CORA_HOST_CHUNKS=$k timeout 120 python scripts/time_e2e.py 2>&1 | tail -2
  echo "chunks $k nograph"; CORA_HOST_NO_GRAPH=1 CORA_HOST_CHUNKS=$k timeout 120 python scripts/time_e2e.py 2>&1 | tail -2
done
