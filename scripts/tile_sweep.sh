#!/usr/bin/env bash
# Row-tile sweep of the Q-band kernel (NF k=128 by default) on one B200.
# Usage (under gpurun, from the repo root): scripts/tile_sweep.sh OUT.jsonl [extra bench args]
set -u
OUT=${1:-gpurun_out/tile_sweep.jsonl}; shift || true
: > "$OUT"
for impl in 0 2; do
  for mb in 0 16 24 32 48 64 96; do
    timeout 200 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu --qband-impl $impl \
      --tile-mb $mb "$@" > /tmp/ts.log 2>&1
    tail -1 /tmp/ts.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'impl': $impl, 'tile_mb': $mb, 'value': d['value'], 'ms_per_step': d['ms_per_step'], 'rmse': d['rmse'], 'row_tiles': d['config']['row_tiles'], 'clocks': d['clocks']}))" >> "$OUT" 2>&1 || tail -3 /tmp/ts.log >> "$OUT"
  done
done
