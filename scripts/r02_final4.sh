#!/usr/bin/env bash
# Evidence after the P write-back by stores (one B200, under gpurun from the
# repo root): L2 microbenchmark with store modes, headline bench x2,
# reference arm, ncu of the default kernel, launch list, k x precision sweep.
set -u
OUT=${1:-gpurun_out/r02f4}; mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > "$OUT/gpu.csv" 2>&1
./scripts/l2_rowbench 32 > "$OUT/l2_rowbench.jsonl" 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "rc=$?" >> "$OUT/smoke.log"
for i in 1 2; do timeout 400 python bench.py > "$OUT/bench_headline_$i.log" 2>&1; done
timeout 400 python bench.py --impl reference > "$OUT/bench_reference.log" 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:qchain_kernel -s 4 -c 1 \
  -o "$OUT/qchain_nf_k128_f32_default" python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > "$OUT/ncu_full.log" 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$OUT/launches_nf_k128_f32.csv" python bench.py --steps 2 --warmup 3 > "$OUT/ncu_launches.log" 2>&1
: > "$OUT/ksweep.jsonl"
for k in 32 64 128 256; do
  for p in f32 f16; do
    timeout 200 python bench.py --steps 8 --warmup 3 --k $k --precision $p --no-cpu 2>>"$OUT/err.log" \
      | tail -1 >> "$OUT/ksweep.jsonl"
  done
done
for cfg in "yahoo" "hugewiki"; do
  timeout 600 python bench.py --workload $cfg --steps 5 --warmup 3 --no-cpu --no-e2e 2>>"$OUT/err.log" \
    | tail -1 >> "$OUT/configs.jsonl"
done
echo done
