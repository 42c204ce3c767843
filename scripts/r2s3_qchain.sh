#!/bin/bash
# The chained kernel (implementations 4-6) with the rating folded into the
# reduction: its parity tests and the workloads that use it.
O=gpurun_out/${1:-s3z}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_kernels.py -k "qband or qchain or chain or split or default_layout or pstore" -q -x > $O/pytest.log 2>&1; tail -n 1 $O/pytest.log
for w in yahoo hugewiki ml1m; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-e2e > $O/$w.json 2> $O/$w.err
  python -c "import json;d=json.load(open('$O/$w.json'));print('$w',d['layout']['qband_impl'],round(d['value']/1e9,2))"
done
timeout 300 python bench.py --qband-impl 5 --steps 10 --warmup 3 --no-cpu --no-e2e > $O/nf_impl5.json 2> $O/nf_impl5.err
python -c "import json;d=json.load(open('$O/nf_impl5.json'));print('nf impl5',round(d['value']/1e9,2))"
