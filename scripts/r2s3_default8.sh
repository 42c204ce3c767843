#!/bin/bash
# The tile-resident default (implementation 8 / 7 by data.tile_resident_impl):
# smoke, the GPU suite, the default bench (with e2e through StreamingEpoch),
# the k x precision sweep and the other workloads on the automatic layout,
# the launch list of the bench and one full ncu capture of the hot kernel.
O=gpurun_out/${1:-s3f}; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -n 3 $O/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_default.json 2> $O/bench_default.err
for p in f32 f16; do for k in 32 64 128 256; do
  timeout 300 python bench.py --steps 10 --warmup 3 --k $k --precision $p --no-cpu \
    > $O/default_${p}_k$k.json 2> $O/default_${p}_k$k.err
done; done
for w in ml1m yahoo hugewiki; do
  timeout 900 python bench.py --steps 5 --warmup 3 --workload $w --no-e2e --no-cpu \
    > $O/${w}_default.json 2> $O/${w}_default.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:runs_kernel -s 6 -c 1 \
  -o $O/runs_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_full.log 2>&1
ls $O | wc -l
