#!/bin/bash
# Quick loop: run-group parity tests, the k x precision sweep, one ncu capture.
O=gpurun_out/${1:-s3h}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -k "runs" -q -x > $O/pytest.log 2>&1; tail -n 2 $O/pytest.log
for p in f32 f16; do for k in 32 64 128 256; do
  timeout 300 python bench.py --steps 10 --warmup 3 --k $k --precision $p --no-cpu --no-e2e \
    > $O/default_${p}_k$k.json 2> $O/default_${p}_k$k.err
  python -c "import json;d=json.load(open('$O/default_${p}_k$k.json'));print('$p $k',d['layout']['qband_impl'],round(d['value']/1e9,2))"
done; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:runs_kernel -s 6 -c 1 \
  -o $O/runs_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_full.log 2>&1
ls $O | wc -l
