#!/bin/bash
mkdir -p gpurun_out/r2q
timeout 1500 python -m pytest tests/test_gpu_quality_gate.py tests/test_gpu_multi_bench.py -x -q -s > gpurun_out/r2q/pytest.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2q/bench.json 2> gpurun_out/r2q/bench.err
tail -3 gpurun_out/r2q/pytest.log
