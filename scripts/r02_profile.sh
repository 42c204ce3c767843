#!/usr/bin/env bash
# Round-2 evidence batch on one B200 (run under gpurun from the repo root):
# L2 microbenchmark, ncu of the default kernel, launch list, GPU tests,
# headline bench and the k x precision sweep with the default implementation.
set -u
OUT=${1:-gpurun_out/r02p}; mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > "$OUT/gpu.csv" 2>&1
./scripts/l2_rowbench 32 > "$OUT/l2_rowbench.jsonl" 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:qchain_kernel -s 4 -c 1 \
  -o "$OUT/qchain_nf_k128_f32" python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > "$OUT/ncu_full.log" 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:qchain_kernel -s 4 -c 1 \
  -o "$OUT/qchain_nf_k128_f16" python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --precision f16 > "$OUT/ncu_full16.log" 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$OUT/launches_nf_k128_f32.csv" python bench.py --steps 2 --warmup 1 > "$OUT/ncu_launches.log" 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 400 python bench.py --steps 10 --warmup 3 > "$OUT/bench_headline.log" 2>&1
: > "$OUT/ksweep.jsonl"
for k in 32 64 128 256; do
  for p in f32 f16; do
    timeout 200 python bench.py --steps 8 --warmup 3 --k $k --precision $p --no-e2e --no-cpu > /tmp/ks.log 2>&1
    tail -1 /tmp/ks.log >> "$OUT/ksweep.jsonl"
  done
done
echo done
