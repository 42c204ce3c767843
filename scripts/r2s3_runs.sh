#!/bin/bash
# Implementation 8 (run groups over a tile-resident P): parity, throughput at
# every k x precision and on the other workloads, quality gate, one ncu capture.
O=gpurun_out/${1:-s3d}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -k "runs or ptile" -q -x > $O/pytest_runs.log 2>&1; tail -n 3 $O/pytest_runs.log
for p in f32 f16; do for k in 32 64 128 256; do
  timeout 300 python bench.py --steps 10 --warmup 3 --qband-impl 8 --no-e2e --no-cpu --k $k --precision $p \
    > $O/impl8_${p}_k$k.json 2> $O/impl8_${p}_k$k.err
done; done
for w in ml1m yahoo hugewiki; do
  timeout 900 python bench.py --steps 5 --warmup 3 --workload $w --qband-impl 8 --no-e2e --no-cpu \
    > $O/${w}_impl8.json 2> $O/${w}_impl8.err
done
timeout 900 python -m pytest tests/test_gpu_quality_gate.py -k "tile_resident" -q -x -s > $O/pytest_quality.log 2>&1; tail -n 2 $O/pytest_quality.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:runs_kernel -s 6 -c 1 \
  -o $O/runs_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --qband-impl 8 \
  > $O/ncu_full.log 2>&1
ls $O | wc -l
