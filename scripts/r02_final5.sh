#!/usr/bin/env bash
# Closing batch with P by stores: GPU tests, smoke, default-policy check over
# the BASELINE configs and the multi-GPU projections (Netflix weak, Hugewiki
# and Yahoo strong); run under gpurun from the repo root.
set -u
OUT=${1:-gpurun_out/r02f5}; mkdir -p "$OUT"
timeout 1200 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "rc=$?" >> "$OUT/smoke.log"
scripts/policy_check.sh "$OUT/policy_check.jsonl"
for w in 2 4 8; do
  timeout 900 python bench.py --no-e2e --no-cpu --workload yahoo --scaling strong --sim-world $w \
    --steps 3 --warmup 3 2>>"$OUT/err.log" | tail -1 >> "$OUT/sim_yahoo_strong.jsonl"
done
echo done
