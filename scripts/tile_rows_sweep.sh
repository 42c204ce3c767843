#!/usr/bin/env bash
# Row-tile cap of 65536 users (16-bit tile-relative ids on the host stream)
# against byte-sized tiles only, for the k x precision points it changes; run
# under gpurun from the repo root.
set -u
OUT=${1:-gpurun_out/tile_rows}; mkdir -p "$OUT"
for kp in "32 f32" "32 f16" "64 f32" "64 f16" "128 f16"; do
  set -- $kp
  for cap in 0 65536; do
    timeout 200 python bench.py --steps 8 --warmup 3 --k $1 --precision $2 --no-cpu \
      --tile-rows $cap 2>>"$OUT/err.log" | tail -1 >> "$OUT/sweep.jsonl"
  done
done
echo done
