#!/bin/bash
# Round 2, session 3: re-establish the GPU state after a container reset.
# Smoke, the GPU suite, the default bench, implementation 7 (tile-resident P)
# at every k x precision, and one full ncu capture of the ptile kernel.
O=gpurun_out/s3a; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -n 2 $O/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_default.json 2> $O/bench_default.err
for p in f32 f16; do for k in 32 64 128 256; do
  timeout 300 python bench.py --steps 10 --warmup 3 --qband-impl 7 --no-e2e --no-cpu --k $k --precision $p \
    > $O/impl7_${p}_k$k.json 2> $O/impl7_${p}_k$k.err
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --k $k --precision $p \
    > $O/default_${p}_k$k.json 2> $O/default_${p}_k$k.err
done; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ptile -s 6 -c 1 \
  -o $O/ptile_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --qband-impl 7 \
  > $O/ncu_full.log 2>&1
ls -la $O
