#!/bin/bash
# The next P tile prefetched into L2: N=1 sweep, the 8-GPU geometry's per-GPU rate.
O=gpurun_out/${1:-s3u}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -k "runs" -q -x > $O/pytest.log 2>&1; tail -n 1 $O/pytest.log
for p in f32; do for k in 32 128 256; do
  timeout 300 python bench.py --steps 10 --warmup 3 --k $k --precision $p --no-cpu --no-e2e > $O/default_${p}_k$k.json 2> $O/default_${p}_k$k.err
  python -c "import json;d=json.load(open('$O/default_${p}_k$k.json'));print('$p $k',round(d['value']/1e9,2))"
done; done
for n in 4 8; do
  timeout 900 python bench.py --sim-world $n --steps 5 --warmup 3 --no-cpu --no-e2e > $O/sim${n}.json 2> $O/sim${n}.err
  python -c "import json;d=json.load(open('$O/sim${n}.json'));print('sim $n',round(d['value']/1e9,2))"
done
