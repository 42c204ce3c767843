#!/bin/bash
O=gpurun_out/${1:-s3x}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_distributed.py -q -x > $O/pytest.log 2>&1; tail -n 2 $O/pytest.log
