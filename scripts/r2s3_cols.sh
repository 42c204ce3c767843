#!/bin/bash
# Per-GPU rate of rank 0's share of an 8-GPU job against the column-band count
# (2N+1 vs 3N+1), NF weak and Hugewiki strong; pairs with scripts/lease_sim.py.
O=gpurun_out/${1:-s3v}; mkdir -p $O
for c in 2 3; do
  timeout 900 python bench.py --sim-world 8 --cols-per-gpu $c --steps 5 --warmup 3 --no-cpu --no-e2e > $O/sim8_nf_c$c.json 2> $O/sim8_nf_c$c.err
  python -c "import json;d=json.load(open('$O/sim8_nf_c$c.json'));print('nf cols/gpu $c',d['layout']['grid'],round(d['value']/1e9,2))"
  timeout 900 python bench.py --sim-world 8 --cols-per-gpu $c --workload hugewiki --scaling strong --steps 3 --warmup 3 --no-cpu --no-e2e > $O/sim8_hw_c$c.json 2> $O/sim8_hw_c$c.err
  python -c "import json;d=json.load(open('$O/sim8_hw_c$c.json'));print('hw cols/gpu $c',d['layout']['grid'],round(d['value']/1e9,2))"
done
