#!/usr/bin/env bash
# Round-2 measurement batch on one B200 (run under gpurun from the repo root).
set -u
OUT=${1:-gpurun_out/r02m}; mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > "$OUT/gpu.csv" 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 400 python bench.py --steps 10 --warmup 3 > "$OUT/bench_headline.log" 2>&1
timeout 200 python bench.py --workload ml1m --steps 20 --warmup 3 --no-e2e > "$OUT/bench_ml1m.log" 2>&1
timeout 400 python bench.py --workload yahoo --steps 5 --warmup 3 --no-e2e --no-cpu > "$OUT/bench_yahoo.log" 2>&1
timeout 900 python bench.py --workload hugewiki --steps 3 --warmup 3 --no-e2e --no-cpu > "$OUT/bench_hugewiki.log" 2>&1
echo done
