#!/bin/bash
# two CTAs per SM on half-size P tiles (8 warps each) vs one CTA of 16 warps
O=gpurun_out/${1:-s4half}; mkdir -p $O
cp paper_2006_15980_b200/lib/libhmf.so /tmp/libhmf_default.so
for cfg in "default:" "default:--tile-rows 208" "k128f32_8_8:--tile-rows 208" "k128f32_8_8:"; do
  v=${cfg%%:*}; a=${cfg#*:}
  if [ $v = default ]; then cp /tmp/libhmf_default.so paper_2006_15980_b200/lib/libhmf.so; else cp build/var/$v/libhmf.so paper_2006_15980_b200/lib/libhmf.so; fi
  n=${v}_$(echo $a | tr -d ' -'); 
  timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e $a > $O/$n.json 2> $O/$n.err
  python -c "import json;d=json.load(open('$O/$n.json'));print('$n',round(d['value']/1e9,3),d['rmse']['test'])"
done
cp /tmp/libhmf_default.so paper_2006_15980_b200/lib/libhmf.so
