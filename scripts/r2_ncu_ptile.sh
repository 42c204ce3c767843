#!/bin/bash
mkdir -p gpurun_out/r2n
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ptile -s 6 -c 1 \
  -o gpurun_out/r2n/ptile_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --qband-impl 7 \
  > gpurun_out/r2n/ncu.log 2>&1
tail -3 gpurun_out/r2n/ncu.log
