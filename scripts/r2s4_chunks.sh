#!/bin/bash
# chunked P-tile write-back / load overlap A/B at N=1 and at the 8-GPU geometry
O=gpurun_out/${1:-s4chunks}; mkdir -p $O
cp paper_2006_15980_b200/lib/libhmf.so /tmp/libhmf_default.so
mkdir -p /tmp/var_default; cp /tmp/libhmf_default.so /tmp/var_default/libhmf.so
for v in /tmp/var_default build/var/*; do
  n=$(basename $v); cp $v/libhmf.so paper_2006_15980_b200/lib/libhmf.so
  timeout 600 python -m pytest tests/test_gpu_kernels.py -k "runs" -q > $O/pytest_$n.log 2>&1; echo "$n $(tail -n 1 $O/pytest_$n.log)"
  for r in 1 2; do
    timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e > $O/${n}_n1_$r.json 2> $O/${n}_n1_$r.err
    python -c "import json;d=json.load(open('$O/${n}_n1_$r.json'));print('$n n1',round(d['value']/1e9,3),d['rmse']['test'])"
    timeout 600 python bench.py --sim-world 8 --steps 5 --warmup 3 --no-cpu --no-e2e > $O/${n}_sim8_$r.json 2> $O/${n}_sim8_$r.err
    python -c "import json;d=json.load(open('$O/${n}_sim8_$r.json'));print('$n sim8',round(d['value']/1e9,3),d['rmse']['test'])"
  done
done
cp /tmp/libhmf_default.so paper_2006_15980_b200/lib/libhmf.so
