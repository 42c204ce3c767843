#!/bin/bash
# Implementation 7 vs the default layout on the other BASELINE workloads, and
# the multi-rank GPU tests with the shared-memory lease table.
O=gpurun_out/s3b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi_bench.py tests/test_gpu_distributed.py -q -x > $O/pytest_multi.log 2>&1; tail -n 2 $O/pytest_multi.log
for w in ml1m yahoo hugewiki; do
  for i in -1 7; do
    timeout 900 python bench.py --steps 5 --warmup 3 --workload $w --qband-impl $i --no-e2e --no-cpu \
      > $O/${w}_impl$i.json 2> $O/${w}_impl$i.err
  done
done
timeout 600 python bench.py --gpus 2 --workload yahoo --scaling strong --steps 4 --warmup 3 --no-cpu \
  > $O/yahoo_n2_shm.json 2> $O/yahoo_n2_shm.err
timeout 600 python bench.py --gpus 2 --workload yahoo --scaling strong --steps 4 --warmup 3 --no-cpu --lease store \
  > $O/yahoo_n2_store.json 2> $O/yahoo_n2_store.err
ls -la $O
