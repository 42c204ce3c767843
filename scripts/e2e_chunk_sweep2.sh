#!/usr/bin/env bash
# e2e chunk plan sweep (tiles per chunk, last chunk, staging buffers), every
# chunk uploaded every epoch; run under gpurun from the repo root.
set -u
OUT=${1:-gpurun_out/e2e_chunks3}; mkdir -p "$OUT"
timeout 600 python -m pytest tests/test_gpu_engine.py -q -k streaming > "$OUT/pytest_streaming.log" 2>&1
echo "rc=$?" >> "$OUT/pytest_streaming.log"
for cfg in "7 1 3" "7 1 2" "4 1 3" "3 1 3" "8 0 2"; do
  set -- $cfg
  timeout 300 python bench.py --steps 10 --warmup 3 --stream-tiles $1 --stream-last $2 \
    --stream-buffers $3 2>>"$OUT/err.log" | tail -1 >> "$OUT/sweep.jsonl"
done
echo done
