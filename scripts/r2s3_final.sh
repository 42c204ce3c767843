#!/bin/bash
# Round-2 evidence on the run-group default: smoke, GPU suite, the default
# bench line, the reference arm, N=2 (two ranks on the box's GPU), the
# per-GPU rate of the 2/4/8-GPU geometries (--sim-world), the launch list.
O=gpurun_out/${1:-s3k}; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -n 2 $O/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu > $O/bench_n2_weak.json 2> $O/bench_n2_weak.err
timeout 900 python bench.py --gpus 2 --workload yahoo --scaling strong --steps 5 --warmup 3 --no-cpu > $O/bench_n2_yahoo_strong.json 2> $O/bench_n2_yahoo_strong.err
for n in 2 4 8; do
  timeout 900 python bench.py --sim-world $n --steps 5 --warmup 3 --no-cpu --no-e2e > $O/sim${n}_netflix_weak.json 2> $O/sim${n}_netflix_weak.err
  timeout 900 python bench.py --sim-world $n --workload hugewiki --scaling strong --steps 3 --warmup 3 --no-cpu --no-e2e > $O/sim${n}_hugewiki_strong.json 2> $O/sim${n}_hugewiki_strong.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/launches.log 2>&1
ls $O | wc -l
