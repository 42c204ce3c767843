#!/bin/bash
# ML-1M (BASELINE configs[0]) throughput: the automatic layout and variants,
# 20 timed epochs as in round 2's earlier measurement.
O=gpurun_out/${1:-s3m}; mkdir -p $O
for i in -1 4 6 0; do
  timeout 300 python bench.py --workload ml1m --steps 20 --warmup 3 --no-e2e --no-cpu --qband-impl $i > $O/ml1m_impl$i.json 2> $O/ml1m_impl$i.err
  python -c "import json;d=json.load(open('$O/ml1m_impl$i.json'));print('impl $i',d['layout']['qband_impl'],d['layout']['item_run_split'],round(d['value']/1e9,2),round(d['roofline']['mean_launch_ms']*1e3,1),'us/launch',round(d['ms_per_step']*1e3,1),'us/step')"
done
for s in 1 2 4 8 16; do
  timeout 300 python bench.py --workload ml1m --steps 20 --warmup 3 --no-e2e --no-cpu --split $s > $O/ml1m_split$s.json 2> $O/ml1m_split$s.err
  python -c "import json;d=json.load(open('$O/ml1m_split$s.json'));print('split $s',d['layout']['qband_impl'],d['layout']['item_run_split'],round(d['value']/1e9,2),round(d['roofline']['mean_launch_ms']*1e3,1),'us/launch',round(d['ms_per_step']*1e3,1),'us/step')"
done
timeout 600 nsys --version > /dev/null 2>&1 || true
