#!/usr/bin/env bash
# Stores vs reductions for the P write-back at every k x precision, and NF
# test RMSE over 10 epochs with each where stores are candidates; run under
# gpurun from the repo root.
set -u
OUT=${1:-gpurun_out/pstore3}; mkdir -p "$OUT"
for k in 32 64 128 256; do
  for p in f32 f16; do
    for ps in 0 1; do
      timeout 200 python bench.py --steps 8 --warmup 3 --k $k --precision $p --no-cpu --no-e2e \
        --pstore $ps 2>>"$OUT/err.log" | tail -1 >> "$OUT/bench.jsonl"
    done
  done
done
for ps in 1 0; do
  timeout 600 python scripts/quality.py netflix --modes qband_f16 --epochs 10 --pstore $ps \
    > "$OUT/quality_k128_f16_pstore$ps.json" 2>>"$OUT/err.log"
  for k in 64 32; do
    timeout 600 python scripts/quality.py netflix --k $k --modes qband --epochs 10 --pstore $ps \
      > "$OUT/quality_k${k}_f32_pstore$ps.json" 2>>"$OUT/err.log"
  done
done
echo done
