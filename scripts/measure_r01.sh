#!/usr/bin/env bash
# Round-1 measurement batch on one B200 (run under gpurun from the repo root).
# Every bench line lands in gpurun_out/; each run is bounded by `timeout`.
set -u
OUT=gpurun_out
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > "$OUT/gpu.csv" 2>&1
lscpu > "$OUT/lscpu.txt" 2>&1

# 1) headline: Netflix-shaped k=128 fp32, full line (e2e + CPU baseline)
timeout 400 python bench.py --steps 10 --warmup 3 > "$OUT/bench_headline.log" 2>&1

# 2) k sweep x storage precision (BASELINE configs[4])
: > "$OUT/ksweep.jsonl"
for k in 32 64 128 256; do
  for p in f32 f16; do
    timeout 200 python bench.py --steps 8 --warmup 3 --k $k --precision $p --no-e2e --no-cpu \
      > "$OUT/ks_${k}_${p}.log" 2>&1
    tail -1 "$OUT/ks_${k}_${p}.log" >> "$OUT/ksweep.jsonl"
  done
done

# 3) ML-1M-shaped (configs[0]) and Yahoo-R1-shaped (configs[2]) on one GPU
timeout 200 python bench.py --workload ml1m --steps 20 --warmup 3 --no-e2e > "$OUT/bench_ml1m.log" 2>&1
timeout 400 python bench.py --workload yahoo --steps 5 --warmup 3 --no-e2e --no-cpu > "$OUT/bench_yahoo.log" 2>&1

# 4) the reference arm (CPU port of the reference's stream-only path, all host threads)
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > "$OUT/bench_reference.log" 2>&1
echo done
