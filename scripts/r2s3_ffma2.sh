#!/bin/bash
# Implementation 7 with packed fp32 pairs (FFMA2/FMUL2, in-place update):
# parity tests, throughput at every k x precision, one ncu capture.
O=gpurun_out/s3c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -k "ptile" -q -x > $O/pytest_ptile.log 2>&1; tail -n 2 $O/pytest_ptile.log
for p in f32 f16; do for k in 32 64 128 256; do
  timeout 300 python bench.py --steps 10 --warmup 3 --qband-impl 7 --no-e2e --no-cpu --k $k --precision $p \
    > $O/impl7_${p}_k$k.json 2> $O/impl7_${p}_k$k.err
done; done
for w in yahoo hugewiki; do
  timeout 900 python bench.py --steps 5 --warmup 3 --workload $w --qband-impl 7 --no-e2e --no-cpu \
    > $O/${w}_impl7.json 2> $O/${w}_impl7.err
done
timeout 900 python -m pytest tests/test_gpu_quality_gate.py -k "tile_resident" -q -x -s > $O/pytest_quality.log 2>&1; tail -n 2 $O/pytest_quality.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ptile -s 6 -c 1 \
  -o $O/ptile_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --qband-impl 7 \
  > $O/ncu_full.log 2>&1
ls $O | wc -l
