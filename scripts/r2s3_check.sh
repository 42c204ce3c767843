#!/bin/bash
# Re-run what changed: the descriptor-load fix in runs.cuh, the updated
# layout tests, the multi-rank run-group path, k sweep, the headline bench,
# and ncu of the run-group kernel.
O=gpurun_out/${1:-s3g}; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_gpu_distributed.py tests/test_gpu_quality_gate.py -q > $O/pytest.log 2>&1; tail -n 3 $O/pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_default.json 2> $O/bench_default.err
for p in f32 f16; do for k in 32 64 128 256; do
  timeout 300 python bench.py --steps 10 --warmup 3 --k $k --precision $p --no-cpu --no-e2e \
    > $O/default_${p}_k$k.json 2> $O/default_${p}_k$k.err
done; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:runs_kernel -s 6 -c 1 \
  -o $O/runs_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_full.log 2>&1
ls $O | wc -l
