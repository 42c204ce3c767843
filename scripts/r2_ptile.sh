#!/bin/bash
mkdir -p gpurun_out/r2p
timeout 900 python -m pytest tests/test_gpu_kernels.py -k "ptile" -x -q > gpurun_out/r2p/pytest_ptile.log 2>&1
tail -3 gpurun_out/r2p/pytest_ptile.log
for k in 128; do
timeout 600 python bench.py --steps 10 --warmup 3 --qband-impl 7 --no-e2e --no-cpu > gpurun_out/r2p/bench_impl7_k$k.json 2> gpurun_out/r2p/bench_impl7_k$k.err
done
timeout 900 python -m pytest tests/test_gpu_quality_gate.py -k "tile_resident" -x -q -s > gpurun_out/r2p/pytest_quality.log 2>&1
tail -3 gpurun_out/r2p/pytest_quality.log
