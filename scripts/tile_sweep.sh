#!/usr/bin/env bash
# Row-tile sweep of the default Q-band kernel (NF k=128 by default) on one B200.
# Usage (under gpurun, from the repo root): scripts/tile_sweep.sh OUT.jsonl "MB MB ..." [extra bench args]
set -u
OUT=${1:-gpurun_out/tile_sweep.jsonl}; LIST=${2:-"0 16 24 32 48 64"}; shift 2 || true
: > "$OUT"
for mb in $LIST; do
  timeout 200 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu --tile-mb $mb "$@" > /tmp/ts.log 2>&1
  tail -1 /tmp/ts.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'tile_mb': $mb, 'args': '$*', 'impl': d['config']['qband_impl'], 'value': d['value'], 'ms_per_step': d['ms_per_step'], 'rmse': d['rmse'], 'row_tiles': d['config']['row_tiles'][:2], 'clocks': d['clocks']}))" >> "$OUT" 2>&1 || tail -3 /tmp/ts.log >> "$OUT"
done
