#!/bin/bash
# A/B of build/var/* variants against the default build on the given k/precision pairs
O=gpurun_out/${1:-s4ab}; shift; mkdir -p $O
PAIRS=${PAIRS:-"128 f32"}
cp paper_2006_15980_b200/lib/libhmf.so /tmp/libhmf_default.so
mkdir -p /tmp/var_default; cp /tmp/libhmf_default.so /tmp/var_default/libhmf.so
for v in /tmp/var_default build/var/*; do
  n=$(basename $v); cp $v/libhmf.so paper_2006_15980_b200/lib/libhmf.so
  [ $n != var_default ] && { timeout 600 python -m pytest tests/test_gpu_kernels.py -k "runs_equal" -q > $O/pytest_$n.log 2>&1; echo "$n $(tail -n 1 $O/pytest_$n.log)"; }
  echo "$PAIRS" | tr ',' '\n' | while read k p; do for r in 1 2; do
    timeout 300 python bench.py --steps 6 --warmup 3 --k $k --precision $p --no-cpu --no-e2e > $O/${n}_k${k}_${p}_$r.json 2> $O/${n}_k${k}_${p}_$r.err
    python -c "import json;d=json.load(open('$O/${n}_k${k}_${p}_$r.json'));print('$n k$k $p',round(d['value']/1e9,3),round(d['roofline']['mean_launch_ms'],3),d['rmse']['test'])"
  done; done
done
cp /tmp/libhmf_default.so paper_2006_15980_b200/lib/libhmf.so
