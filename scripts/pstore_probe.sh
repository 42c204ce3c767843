#!/usr/bin/env bash
# P write-back of the chained kernel, plain stores (--pstore 1) vs vector
# reductions (--pstore 0): throughput per k x precision, and NF k=128 test
# RMSE over 10 epochs with each; run under gpurun from the repo root.
set -u
OUT=${1:-gpurun_out/pstore2}; mkdir -p "$OUT"
for ps in 0 1; do
  for kp in "128 f32" "256 f32" "64 f32" "128 f16"; do
    set -- $kp
    timeout 200 python bench.py --steps 8 --warmup 3 --k $1 --precision $2 --no-cpu --no-e2e \
      --pstore $ps 2>>"$OUT/err.log" | tail -1 >> "$OUT/bench.jsonl"
  done
done
for ps in 1 0; do
  timeout 600 python scripts/quality.py netflix --modes qband --epochs 10 --pstore $ps \
    > "$OUT/quality_pstore$ps.json" 2>>"$OUT/err.log"
done
echo done
