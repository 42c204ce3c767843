#!/bin/bash
# ncu --set full of the run-group kernel at fp32 k=32 and fp16 k=128.
O=gpurun_out/${1:-s3o}; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:runs_kernel -s 6 -c 1 \
  -o $O/runs_k32_f32 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --k 32 > $O/ncu_k32.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:runs_kernel -s 6 -c 1 \
  -o $O/runs_k128_f16 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --precision f16 > $O/ncu_f16.log 2>&1
ls $O
