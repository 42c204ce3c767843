#!/bin/bash
# Round-2 closing evidence: smoke, the default bench line, the reference arm,
# N=2 on the box's GPU under both lease policies, the launch list.
O=gpurun_out/${1:-s4final}; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_default.json 2> $O/bench_default.err
python -c "import json;d=json.load(open('$O/bench_default.json'));print('default',round(d['value']/1e9,3),'e2e',round(d['e2e']['value']/1e9,3),d['clocks'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
python -c "import json;d=json.load(open('$O/bench_reference.json'));print('reference',d['value'],d.get('unit'))"
for pol in free quota; do
  timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu --policy $pol > $O/bench_n2_weak_$pol.json 2> $O/bench_n2_weak_$pol.err
  python -c "import json;d=json.load(open('$O/bench_n2_weak_$pol.json'));print('n2 $pol',round(d['value']/1e9,3),d['rmse'],d['leases'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/launches.log 2>&1
ls $O | wc -l
