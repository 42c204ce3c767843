#!/bin/bash
# compute-sanitizer over the run-group kernel's parity tests and the streamed
# epoch: memcheck (out-of-bounds / misaligned, incl. the TMA tile copies) and
# synccheck (barrier / mbarrier misuse).
O=gpurun_out/${1:-s3l}; mkdir -p $O
timeout 1200 compute-sanitizer --tool memcheck --target-processes all --print-limit 20 \
  python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -k "runs" -q -x > $O/memcheck_runs.log 2>&1
tail -n 4 $O/memcheck_runs.log
timeout 1200 compute-sanitizer --tool synccheck --target-processes all --print-limit 20 \
  python -m pytest tests/test_gpu_kernels.py -k "runs_equal" -q -x > $O/synccheck_runs.log 2>&1
tail -n 4 $O/synccheck_runs.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 \
  python -c "import __graft_entry__ as g; g.smoke()" > $O/memcheck_smoke.log 2>&1
tail -n 3 $O/memcheck_smoke.log
