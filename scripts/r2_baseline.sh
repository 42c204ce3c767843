#!/bin/bash
# Round-2 baseline on one B200: GPU suite, headline bench, launch list that
# includes the training launches, one full ncu capture of the hot kernel.
set -x
mkdir -p gpurun_out/r2b
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2b/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2b/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b/bench.json 2> gpurun_out/r2b/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2b/launches_all.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu \
  > gpurun_out/r2b/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qchain -s 6 -c 1 \
  -o gpurun_out/r2b/qchain_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu \
  > gpurun_out/r2b/ncu_full.log 2>&1
ls -la gpurun_out/r2b
