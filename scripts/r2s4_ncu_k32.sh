#!/bin/bash
# one ncu --set full capture of the run-group kernel at NF k=32 fp32 (wide configuration)
O=gpurun_out/${1:-s4ncu32}; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:runs_kernel -s 6 -c 1 \
  -o $O/runs_k32 python bench.py --k 32 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu.log 2>&1
ls $O
