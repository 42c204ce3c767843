#!/usr/bin/env bash
# 24-warp chain configurations (2, 3) against the automatic one at k >= 128,
# fp16 (and fp32 k=256); run under gpurun from the repo root.
set -u
OUT=${1:-gpurun_out/largek}; mkdir -p "$OUT"
for kp in "128 f16" "256 f16" "256 f32"; do
  set -- $kp
  for c in -1 2 3; do
    timeout 200 python bench.py --steps 8 --warmup 3 --k $1 --precision $2 --no-cpu --no-e2e \
      --chain-cfg $c 2>>"$OUT/err.log" | tail -1 | sed "s/^/{\"cfg\": $c, \"line\": /; s/\$/}/" >> "$OUT/sweep.jsonl"
  done
done
