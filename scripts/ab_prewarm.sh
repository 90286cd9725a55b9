out=gpurun_out/prewarm.txt; : > $out
for i in 1 2 3; do for pw in 0 3; do
r=$(timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-stack --no-ex2 --prewarm $pw 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), {k: round(x*1e3,1) for k, x in d['ms_percentiles'].items()})")
echo "prewarm=$pw $r" >> $out; sleep 5; done; done
