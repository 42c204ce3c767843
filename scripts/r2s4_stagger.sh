#!/bin/bash
# staggered P-tile switches (bench --tile-stagger) at N=1 and the 8-GPU geometry
O=gpurun_out/${1:-s4stag}; mkdir -p $O
for a in "" "--tile-stagger"; do n=x$(echo $a | tr -d ' -'); for r in 1 2; do
  timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e $a > $O/${n}_n1_$r.json 2> $O/${n}_n1_$r.err
  python -c "import json;d=json.load(open('$O/${n}_n1_$r.json'));print('$n n1',round(d['value']/1e9,3),d['rmse']['test'])"
  timeout 600 python bench.py --sim-world 8 --steps 5 --warmup 3 --no-cpu --no-e2e $a > $O/${n}_sim8_$r.json 2> $O/${n}_sim8_$r.err
  python -c "import json;d=json.load(open('$O/${n}_sim8_$r.json'));print('$n sim8',round(d['value']/1e9,3),d['rmse']['test'])"
done; done
