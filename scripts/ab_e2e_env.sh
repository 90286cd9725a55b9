#!/bin/bash
# e2e A/B of an environment switch (bench.py's e2e leg, 20 steps): VAR=... VALUES="..." bash scripts/ab_e2e_env.sh
out=gpurun_out/ab_e2e.txt; : > $out
for i in 1 2 3; do for v in ${VALUES:-1 0}; do
r=$(env $VAR=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-stack --no-ex2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), round(d['e2e']['ms_per_step']*1e3,1), round(d['e2e']['value'],1))")
echo "$VAR=$v step/e2e $r" >> $out; done; done
cat $out
