#!/bin/bash
O=gpurun_out/${1:-s4stale}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -k "default_layout or tile_resident_policy" -q -s > $O/pytest.log 2>&1; tail -n 1 $O/pytest.log
timeout 900 python scripts/stale_margin.py 32,64,128 > $O/margin.jsonl 2> $O/margin.err; cat $O/margin.jsonl
