#!/usr/bin/env bash
# Round-2 closing evidence batch on one B200 (run under gpurun from the repo root).
set -u
OUT=${1:-gpurun_out/r02z}; mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > "$OUT/gpu.csv" 2>&1
timeout 1200 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python __graft_entry__.py --smoke > "$OUT/smoke.log" 2>&1; echo "rc=$?" >> "$OUT/smoke.log"
for i in 1 2; do timeout 400 python bench.py --steps 10 --warmup 3 > "$OUT/bench_headline_$i.log" 2>&1; done
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > "$OUT/bench_reference.log" 2>&1
scripts/policy_check.sh "$OUT/policy_check.jsonl"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29541 bench.py --gpus 2 --steps 3 --warmup 3 > "$OUT/bench_n2_shared_gpu.log" 2>&1
echo done
