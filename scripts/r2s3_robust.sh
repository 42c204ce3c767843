#!/bin/bash
# Robustness sweep of bench.py's flags (each must print one JSON line, rc 0).
O=gpurun_out/${1:-s3y}; mkdir -p $O
run() {
  name=$1; shift
  timeout 900 python bench.py "$@" > $O/$name.json 2> $O/$name.err
  rc=$?
  python -c "
import json,sys
try:
    d=json.loads(open('$O/$name.json').read().strip().splitlines()[-1])
    e=d.get('e2e') or {}
    print('$name rc=$rc', d.get('layout',{}).get('qband_impl'), round(d['value']/1e9,3), 'e2e', e.get('value') and round(e['value']/1e9,2))
except Exception as ex:
    print('$name rc=$rc FAILED', ex)
"
}
run ml1m --workload ml1m --steps 5 --warmup 3 --no-cpu
run yahoo --workload yahoo --steps 3 --warmup 3 --no-cpu
run f16 --precision f16 --steps 5 --warmup 3 --no-cpu
run impl7 --qband-impl 7 --steps 3 --warmup 3 --no-cpu --no-e2e
run impl5 --qband-impl 5 --steps 3 --warmup 3 --no-cpu
run impl0 --qband-impl 0 --steps 3 --warmup 3 --no-cpu --no-e2e
run hogwild --kernel hogwild --steps 3 --warmup 3 --no-cpu
run n2 --gpus 2 --steps 3 --warmup 3 --no-cpu
run skew --item-skew 0.8 --steps 3 --warmup 3 --no-cpu --no-e2e
run ref_ml1m --impl reference --workload ml1m --steps 3 --warmup 3
