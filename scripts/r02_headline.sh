#!/usr/bin/env bash
# Headline lines with the final profiles (traffic, L2 ceiling): default bench
# x2, reference arm, ML-1M; run under gpurun from the repo root.
set -u
OUT=${1:-gpurun_out/r02h}; mkdir -p "$OUT"
for i in 1 2; do timeout 400 python bench.py > "$OUT/bench_headline_$i.log" 2>&1; done
timeout 400 python bench.py --impl reference > "$OUT/bench_reference.log" 2>&1
timeout 400 python bench.py --workload ml1m --steps 20 > "$OUT/bench_ml1m.log" 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "rc=$?" >> "$OUT/smoke.log"
echo done
