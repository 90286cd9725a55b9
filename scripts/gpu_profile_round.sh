#!/bin/bash
# One GPU call for the round's evidence: GPU tests, bench line, ncu launch list, ncu full capture of the
# attention kernel and of the FF2 + LN2 kernel, config sweep, shard makespans.  Output: gpurun_out/$1/
TAG=${1:-round}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
: > "$OUT/summary.txt"
timeout 600 python -m pytest tests/ -q -m gpu -x --timeout 180 -p no:cacheprovider > "$OUT/tests.log" 2>&1
echo "tests exit $?" >> "$OUT/summary.txt"
# the driver's command (20 timed steps after 5 warm-up) is the headline; 200 steps show the power-capped state
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > "$OUT/bench.json" 2> "$OUT/bench.err"
echo "bench exit $?" >> "$OUT/summary.txt"
sleep 10
timeout 900 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu --no-stack > "$OUT/bench200.json" 2> "$OUT/bench200.err"
echo "bench200 exit $?" >> "$OUT/summary.txt"
timeout 600 python scripts/step_modes.py C4-wiki512 300 > "$OUT/step_modes.txt" 2>&1
echo "step_modes exit $?" >> "$OUT/summary.txt"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-clocks --no-stack --no-ex2 > "$OUT/ncu_bench.log" 2>&1
echo "ncu launches exit $?" >> "$OUT/summary.txt"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attention_fwd|gemm_bf16_tn_kernel<256, (6, 1, 4|3, 1, 2)" -s 6 -c 3 \
  -o "$OUT/prof" python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-clocks --no-stack --no-ex2 > "$OUT/ncu_full.log" 2>&1
echo "ncu full exit $?" >> "$OUT/summary.txt"
timeout 600 python scripts/sweep.py --steps 30 > "$OUT/sweep.jsonl" 2> "$OUT/sweep.err"
echo "sweep exit $?" >> "$OUT/summary.txt"
timeout 300 python scripts/time_shards.py C4-wiki512 30 > "$OUT/shards.txt" 2>&1
echo "shards exit $?" >> "$OUT/summary.txt"
if [ -f variants/kspan.so ]; then
  CORA_LIB_PATH=variants/kspan.so timeout 300 python scripts/kspan.py C4-wiki512,C4-race,shard8,C2-mnli 9 > "$OUT/kspan.txt" 2>&1
  echo "kspan exit $?" >> "$OUT/summary.txt"
fi
cat "$OUT/summary.txt"
