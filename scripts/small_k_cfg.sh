#!/usr/bin/env bash
# 24-warp chain configurations (2, 3) against the automatic one at small k;
# run under gpurun from the repo root.
set -u
OUT=${1:-gpurun_out/smallk}; mkdir -p "$OUT"
for kp in "32 f32" "32 f16" "64 f16" "64 f32"; do
  set -- $kp
  for c in -1 2 3; do
    timeout 200 python bench.py --steps 8 --warmup 3 --k $1 --precision $2 --no-cpu --no-e2e \
      --chain-cfg $c 2>>"$OUT/err.log" | tail -1 | sed "s/^/{\"cfg\": $c, \"line\": /; s/\$/}/" >> "$OUT/sweep.jsonl"
  done
done
