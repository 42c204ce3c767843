#!/bin/bash
# k x precision sweep of the default build (run-group kernel) + parity tests
# of every run-group configuration; optional variants in build/var.
O=gpurun_out/${1:-s4ks}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -k "runs or streaming or default_layout" -q > $O/pytest_runs.log 2>&1; tail -n 1 $O/pytest_runs.log
for p in f32 f16; do for k in 32 64 128 256; do
  timeout 300 python bench.py --steps 6 --warmup 3 --k $k --precision $p --no-cpu --no-e2e > $O/default_k${k}_$p.json 2> $O/default_k${k}_$p.err
  python -c "import json;d=json.load(open('$O/default_k${k}_$p.json'));print('default k$k $p',round(d['value']/1e9,3),round(d['roofline']['mean_launch_ms'],3),d['rmse']['test'])"
done; done
cp paper_2006_15980_b200/lib/libhmf.so /tmp/libhmf_default.so
for v in build/var/*; do
  n=$(basename $v); k=$(echo $n | sed 's/k\([0-9]*\)f.*/\1/'); p=f$(echo $n | sed 's/k[0-9]*f\([0-9]*\)_.*/\1/')
  cp $v/libhmf.so paper_2006_15980_b200/lib/libhmf.so
  for r in 1 2; do
    timeout 300 python bench.py --steps 6 --warmup 3 --k $k --precision $p --no-cpu --no-e2e > $O/${n}_$r.json 2> $O/${n}_$r.err
    python -c "import json;d=json.load(open('$O/${n}_$r.json'));print('$n',round(d['value']/1e9,3),round(d['roofline']['mean_launch_ms'],3),d['rmse']['test'])"
  done
done
cp /tmp/libhmf_default.so paper_2006_15980_b200/lib/libhmf.so
