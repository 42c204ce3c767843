#!/usr/bin/env bash
# Round-2 comparison of Q-band implementations 0 (warp per rating) and 4
# (chained item runs) over the BASELINE configs on one B200.
# Usage (under gpurun, from the repo root): scripts/r02_sweep.sh OUTDIR
set -u
OUT=${1:-gpurun_out/r02}; mkdir -p "$OUT"
: > "$OUT/ksweep.jsonl"
for k in 32 64 128 256; do
  for p in f32 f16; do
    for impl in 0 4; do
      timeout 200 python bench.py --steps 8 --warmup 3 --k $k --precision $p --no-e2e --no-cpu \
        --qband-impl $impl > /tmp/r02.log 2>&1
      tail -1 /tmp/r02.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'k': $k, 'precision': '$p', 'impl': $impl, 'value': d['value'], 'rmse': d['rmse'], 'frac': d['roofline']['frac'], 'row_tiles': d['config']['row_tiles']}))" >> "$OUT/ksweep.jsonl" 2>&1 || tail -2 /tmp/r02.log >> "$OUT/ksweep.jsonl"
    done
  done
done
for w in ml1m yahoo; do
  for impl in 0 4; do
    timeout 400 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu \
      --qband-impl $impl > "$OUT/bench_${w}_impl$impl.log" 2>&1
  done
done
