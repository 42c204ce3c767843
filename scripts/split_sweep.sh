#!/usr/bin/env bash
# Item-run split sweep (implementation 5) over workloads; one JSON line per run.
# Usage (under gpurun): scripts/split_sweep.sh OUT.jsonl
set -u
OUT=${1:-gpurun_out/split_sweep.jsonl}; : > "$OUT"
run() {  # label, then bench args
  local label=$1; shift
  timeout 900 python bench.py --no-e2e --no-cpu "$@" > /tmp/sp.log 2>&1
  tail -1 /tmp/sp.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print(json.dumps({'label': '$label', 'args': '$*', 'value': d['value'], 'impl': c.get('qband_impl'), 'split': c.get('item_run_split'), 'rmse': d['rmse'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> "$OUT" 2>&1 || tail -2 /tmp/sp.log >> "$OUT"
}
for sp in 4 5 6 8; do run nf --steps 8 --warmup 3 --split $sp; done
for sp in 2 4 5; do run nf_k256 --steps 8 --warmup 3 --k 256 --split $sp; done
for sp in 4 5 8; do run nf_f16 --steps 8 --warmup 3 --precision f16 --split $sp; done
for sp in 2 4 8 16; do run ml1m --workload ml1m --steps 20 --warmup 3 --split $sp; done
for sp in 2 3; do run hugewiki --workload hugewiki --steps 3 --warmup 3 --split $sp; done
for sp in 2; do run yahoo --workload yahoo --steps 5 --warmup 3 --split $sp; done
