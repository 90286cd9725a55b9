#!/bin/bash
# One GPU call: GPU tests, the bench line, the ncu launch list, and (FULL=<kernel regex>) one
# `ncu --set full` capture.  Everything lands in gpurun_out/$TAG/.
TAG=${1:-${TAG:-run}}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
: > "$OUT/summary.txt"
if [ -z "$SKIP_TESTS" ]; then
  timeout 600 python -m pytest tests/ -q -m gpu -x --timeout 180 -p no:cacheprovider > "$OUT/tests.log" 2>&1
  echo "tests exit $?" >> "$OUT/summary.txt"
fi
timeout 900 python bench.py ${BENCH_ARGS} > "$OUT/bench.json" 2> "$OUT/bench.err"
echo "bench exit $?" >> "$OUT/summary.txt"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-clocks --no-stack --no-ex2 > "$OUT/ncu_bench.log" 2>&1
echo "ncu launches exit $?" >> "$OUT/summary.txt"
if [ -n "$FULL" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$FULL" -s "${FULL_SKIP:-20}" \
    -c "${FULL_COUNT:-5}" -o "$OUT/prof" python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-clocks --no-stack --no-ex2 \
    > "$OUT/ncu_full.log" 2>&1
  echo "ncu full exit $?" >> "$OUT/summary.txt"
fi
cat "$OUT/summary.txt"
