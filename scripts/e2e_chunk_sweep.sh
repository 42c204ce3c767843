#!/usr/bin/env bash
# e2e chunking sweep on one B200 (run under gpurun from the repo root):
# row tiles per streamed chunk x staging buffers, every chunk uploaded every
# epoch (no reuse), plus the reuse variant for comparison.
set -u
OUT=${1:-gpurun_out/e2e_chunks}; mkdir -p "$OUT"
timeout 600 python -m pytest tests/test_gpu_engine.py -q -k streaming > "$OUT/pytest_streaming.log" 2>&1
echo "rc=$?" >> "$OUT/pytest_streaming.log"
for t in 1 2 4 8; do
  for b in 2 3; do
    timeout 300 python bench.py --steps 10 --warmup 3 --stream-tiles $t --stream-buffers $b \
      2>>"$OUT/err.log" | tail -1 >> "$OUT/sweep.jsonl"
  done
done
timeout 300 python bench.py --steps 10 --warmup 3 --stream-tiles 1 --stream-reuse \
  2>>"$OUT/err.log" | tail -1 >> "$OUT/sweep.jsonl"
echo done
