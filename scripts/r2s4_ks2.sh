#!/bin/bash
# after the chain-configuration change: run-group parity + quality tests, k x precision sweep
O=gpurun_out/${1:-s4ks2}; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_gpu_quality_gate.py -k "runs or streaming or default_layout or quality" -q > $O/pytest_runs.log 2>&1; tail -n 1 $O/pytest_runs.log
for p in f32 f16; do for k in 32 64 128 256; do
  timeout 300 python bench.py --steps 6 --warmup 3 --k $k --precision $p --no-cpu --no-e2e > $O/default_k${k}_$p.json 2> $O/default_k${k}_$p.err
  python -c "import json;d=json.load(open('$O/default_k${k}_$p.json'));print('default k$k $p',round(d['value']/1e9,3),round(d['roofline']['mean_launch_ms'],3),d['rmse']['test'])"
done; done
