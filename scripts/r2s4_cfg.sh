#!/bin/bash
# Run-group chain configuration A/B per (k, precision): the default build vs
# build/var/<k><prec>_<lpc>_<wpb> variants (scripts/build_variant.sh).
O=gpurun_out/${1:-s4cfg}; mkdir -p $O
cp paper_2006_15980_b200/lib/libhmf.so /tmp/libhmf_default.so
run() {  # name k prec
  for r in 1 2; do
    timeout 300 python bench.py --steps 6 --warmup 3 --k $2 --precision $3 --no-cpu --no-e2e > $O/$1_k$2_$3_$r.json 2> $O/$1_k$2_$3_$r.err
    python -c "import json;d=json.load(open('$O/$1_k$2_$3_$r.json'));print('$1 k$2 $3 run $r',round(d['value']/1e9,3),round(d['roofline']['mean_launch_ms'],3),d['rmse']['test'])"
  done
}
for kp in "128 f32" "64 f32" "32 f32" "128 f16" "64 f16" "32 f16"; do
  set -- $kp
  cp /tmp/libhmf_default.so paper_2006_15980_b200/lib/libhmf.so
  run default $1 $2
  for v in build/var/k$1$2_*; do
    n=$(basename $v)
    cp $v/libhmf.so paper_2006_15980_b200/lib/libhmf.so
    dt=float32; [ $2 = f16 ] && dt=float16
    timeout 600 python -m pytest tests/test_gpu_kernels.py -k "runs_equal" -q > $O/pytest_$n.log 2>&1; echo "$n $(tail -n 1 $O/pytest_$n.log)"
    run $n $1 $2
  done
done
cp /tmp/libhmf_default.so paper_2006_15980_b200/lib/libhmf.so
