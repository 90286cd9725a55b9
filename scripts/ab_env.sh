#!/bin/bash
# A/B of an environment switch on the driver-style bench (20 steps, 5 warm-up), alternating, 3 rounds:
#   VAR=CORA_GEMM_DYN VALUES="1 0" bash scripts/ab_env.sh
out=gpurun_out/ab_env.txt
: > $out
for i in 1 2 3; do
  for v in ${VALUES:-1 0}; do
    r=$(env $VAR=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-stack --no-ex2 2>/dev/null \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), {k: round(x*1e3,1) for k, x in d['ms_percentiles'].items()})")
    echo "$VAR=$v $r" >> $out
    sleep 5
  done
done
cat $out
