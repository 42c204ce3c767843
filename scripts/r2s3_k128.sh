#!/bin/bash
# k=128 A/B: throughput (fp32, fp16), parity tests of the run-group kernel.
O=gpurun_out/${1:-s3n}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -k "runs" -q -x > $O/pytest.log 2>&1; tail -n 1 $O/pytest.log
for p in f32 f16; do for r in 1 2; do
  timeout 300 python bench.py --steps 10 --warmup 3 --k 128 --precision $p --no-cpu --no-e2e > $O/k128_${p}_$r.json 2> $O/k128_${p}_$r.err
  python -c "import json;d=json.load(open('$O/k128_${p}_$r.json'));print('$p run $r',round(d['value']/1e9,2),round(d['roofline']['mean_launch_ms'],3))"
done; done
