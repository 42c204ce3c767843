#!/bin/bash
# GPU suite + smoke + short bench (round 2 iteration check)
mkdir -p gpurun_out/r2c
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/r2c/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2c/bench.json 2> gpurun_out/r2c/bench.err
tail -3 gpurun_out/r2c/pytest_gpu.log
