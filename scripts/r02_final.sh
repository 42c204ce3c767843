#!/usr/bin/env bash
# Round-2 final evidence batch on one B200 (run under gpurun from the repo root).
set -u
OUT=${1:-gpurun_out/r02f}; mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > "$OUT/gpu.csv" 2>&1
lscpu > "$OUT/lscpu.txt" 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python __graft_entry__.py --smoke > "$OUT/smoke.log" 2>&1; echo "rc=$?" >> "$OUT/smoke.log"
for i in 1 2; do timeout 400 python bench.py --steps 10 --warmup 3 > "$OUT/bench_headline_$i.log" 2>&1; done
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > "$OUT/bench_reference.log" 2>&1
: > "$OUT/ksweep.jsonl"
for k in 32 64 128 256; do
  for p in f32 f16; do
    timeout 200 python bench.py --steps 8 --warmup 3 --k $k --precision $p --no-e2e --no-cpu > /tmp/ks.log 2>&1
    tail -1 /tmp/ks.log >> "$OUT/ksweep.jsonl"
  done
done
timeout 200 python bench.py --workload ml1m --steps 20 --warmup 3 --no-e2e > "$OUT/bench_ml1m.log" 2>&1
timeout 400 python bench.py --workload yahoo --steps 5 --warmup 3 --no-e2e --no-cpu > "$OUT/bench_yahoo.log" 2>&1
timeout 900 python bench.py --workload hugewiki --steps 3 --warmup 3 --no-e2e --no-cpu > "$OUT/bench_hugewiki.log" 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:qchain_kernel -s 4 -c 1 \
  -o "$OUT/qchain_nf_k128_f32" python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > "$OUT/ncu_full.log" 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$OUT/launches_nf_k128_f32.csv" python bench.py --steps 2 --warmup 1 > "$OUT/ncu_launches.log" 2>&1
echo done
for w in 2 4 8; do timeout 600 python bench.py --sim-world $w --steps 3 --warmup 3 > "$OUT/sim_world$w.log" 2>&1; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29537 bench.py --gpus 2 --steps 3 --warmup 3 > "$OUT/bench_n2_shared_gpu.log" 2>&1
echo done2
