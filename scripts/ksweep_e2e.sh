#!/usr/bin/env bash
# GPU tests, then the k x precision sweep with e2e (default layout and
# kernel); run under gpurun from the repo root.
set -u
OUT=${1:-gpurun_out/ksweep_e2e}; mkdir -p "$OUT"
timeout 1200 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
: > "$OUT/ksweep.jsonl"
for k in 32 64 128 256; do
  for p in f32 f16; do
    timeout 200 python bench.py --steps 8 --warmup 3 --k $k --precision $p --no-cpu 2>>"$OUT/err.log" \
      | tail -1 >> "$OUT/ksweep.jsonl"
  done
done
echo done
