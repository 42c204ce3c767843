#!/usr/bin/env bash
# Default-policy check over the BASELINE configs and the multi-GPU projections.
set -u
OUT=${1:-gpurun_out/policy.jsonl}; : > "$OUT"
run() {
  local label=$1; shift
  timeout 900 python bench.py --no-e2e --no-cpu "$@" > /tmp/pc.log 2>&1
  tail -1 /tmp/pc.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print(json.dumps({'label': '$label', 'args': '$*', 'value': d['value'], 'impl': c.get('qband_impl'), 'split': c.get('item_run_split'), 'rmse': d['rmse'], 'sm_mhz': (d.get('clocks') or {}).get('sm_mhz')}))" >> "$OUT" 2>&1 || tail -2 /tmp/pc.log >> "$OUT"
}
run nf --steps 8 --warmup 3
run nf_f16 --steps 8 --warmup 3 --precision f16
for k in 32 64 256; do run nf_k$k --steps 8 --warmup 3 --k $k; run nf_k${k}_f16 --steps 8 --warmup 3 --k $k --precision f16; done
run ml1m --workload ml1m --steps 20 --warmup 3
run yahoo --workload yahoo --steps 5 --warmup 3
run hugewiki --workload hugewiki --steps 3 --warmup 3
for w in 2 4 8; do run sim_nf_weak_$w --sim-world $w --steps 3 --warmup 3; done
for w in 2 4 8; do run sim_hw_strong_$w --workload hugewiki --scaling strong --sim-world $w --steps 3 --warmup 3; done
