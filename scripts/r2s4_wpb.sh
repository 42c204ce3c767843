#!/bin/bash
# k=32 fp32 run groups: quality on narrow 2 %-density blocks vs warps per CTA
O=gpurun_out/${1:-s4wpb}; mkdir -p $O
cp paper_2006_15980_b200/lib/libhmf.so /tmp/libhmf_default.so
for v in build/var/*; do
  n=$(basename $v); cp $v/libhmf.so paper_2006_15980_b200/lib/libhmf.so
  timeout 600 python -m pytest tests/test_gpu_kernels.py -k "default_layout_quality_matches_whole_runs and 32-float32" -q -s > $O/$n.log 2>&1
  echo "$n $(grep -o "'default': ([^)]*)" $O/$n.log) $(tail -n 1 $O/$n.log)"
done
cp /tmp/libhmf_default.so paper_2006_15980_b200/lib/libhmf.so
