#!/bin/bash
# one ncu --set full capture of the run-group kernel at the 8-GPU geometry (rank 0's band, 17 column bands)
O=gpurun_out/${1:-s4ncu8}; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:runs_kernel -s 20 -c 1 \
  -o $O/runs_sim8 python bench.py --sim-world 8 --steps 1 --warmup 2 --no-e2e --no-cpu > $O/ncu.log 2>&1
ls $O
