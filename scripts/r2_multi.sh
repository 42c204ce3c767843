#!/bin/bash
# N>1 on one matrix: band coherence, the 2-rank yahoo strong gate, distributed tests,
# then the two bench lines for the record.
mkdir -p gpurun_out/r2m
timeout 1500 python -m pytest tests/test_gpu_multi_bench.py tests/test_gpu_distributed.py -x -q > gpurun_out/r2m/pytest.log 2>&1
timeout 900 python bench.py --gpus 2 --workload yahoo --scaling strong --steps 10 --warmup 3 --no-cpu > gpurun_out/r2m/yahoo_n2_strong.json 2> gpurun_out/r2m/yahoo_n2_strong.err
timeout 900 python bench.py --gpus 1 --workload yahoo --steps 10 --warmup 3 --no-cpu > gpurun_out/r2m/yahoo_n1.json 2> gpurun_out/r2m/yahoo_n1.err
tail -3 gpurun_out/r2m/pytest.log
