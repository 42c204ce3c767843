#!/bin/bash
# k=256 run-group configuration A/B: LPC x warps per CTA (build/var/*).
O=gpurun_out/${1:-s4k256}; mkdir -p $O
cp paper_2006_15980_b200/lib/libhmf.so /tmp/libhmf_default.so
for v in k256_16_16 k256_8_8 k256_8_10; do
  cp build/var/$v/libhmf.so paper_2006_15980_b200/lib/libhmf.so
  timeout 600 python -m pytest tests/test_gpu_kernels.py -k "runs and 256" -q -x > $O/pytest_$v.log 2>&1; echo "$v $(tail -n 1 $O/pytest_$v.log)"
  for p in f32 f16; do for r in 1 2; do
    timeout 300 python bench.py --steps 6 --warmup 3 --k 256 --precision $p --no-cpu --no-e2e > $O/${v}_${p}_$r.json 2> $O/${v}_${p}_$r.err
    python -c "import json;d=json.load(open('$O/${v}_${p}_$r.json'));print('$v $p run $r',round(d['value']/1e9,3),round(d['roofline']['mean_launch_ms'],3),d['rmse'] if 'rmse' in d else '')"
  done; done
done
cp /tmp/libhmf_default.so paper_2006_15980_b200/lib/libhmf.so
