#!/bin/bash
mkdir -p gpurun_out/r2d
ls oracle/_ref > gpurun_out/r2d/ref_ls.txt
timeout 1200 python -m pytest tests/test_gpu_reference_dropin.py -x -q -s > gpurun_out/r2d/pytest.log 2>&1
tail -3 gpurun_out/r2d/pytest.log
