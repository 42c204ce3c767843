#!/usr/bin/env bash
# Q-band implementation / chain-configuration sweep on one B200 (NF k=128 by
# default).  Usage (under gpurun, from the repo root):
#   scripts/impl_sweep.sh OUT.jsonl "impl:cfg impl:cfg ..." [extra bench args]
set -u
OUT=${1:-gpurun_out/impl_sweep.jsonl}; LIST=${2:-"0:1 3:1 4:0 4:1 4:2 4:3"}; shift 2 || true
: > "$OUT"
for ic in $LIST; do
  impl=${ic%%:*}; cfg=${ic##*:}
  timeout 200 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu --qband-impl $impl \
    --chain-cfg $cfg "$@" > /tmp/is.log 2>&1
  tail -1 /tmp/is.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'impl': $impl, 'cfg': $cfg, 'args': '$*', 'value': d['value'], 'ms_per_step': d['ms_per_step'], 'rmse': d['rmse'], 'row_tiles': d['config']['row_tiles'], 'clocks': d['clocks']}))" >> "$OUT" 2>&1 || tail -3 /tmp/is.log >> "$OUT"
done
