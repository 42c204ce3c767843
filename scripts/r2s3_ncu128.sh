#!/bin/bash
# one ncu --set full capture of the run-group kernel at NF k=128 fp32
O=gpurun_out/${1:-s3s}; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:runs_kernel -s 6 -c 1 \
  -o $O/runs_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_full.log 2>&1
ls $O
