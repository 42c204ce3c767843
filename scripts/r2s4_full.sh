#!/bin/bash
O=gpurun_out/${1:-s4full}; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -n 2 $O/pytest_gpu.log
for r in 1 2; do timeout 300 python bench.py --steps 6 --warmup 3 --k 32 --precision f32 --no-cpu --no-e2e > $O/k32_f32_$r.json 2> $O/k32_f32_$r.err
python -c "import json;d=json.load(open('$O/k32_f32_$r.json'));print('k32 f32',round(d['value']/1e9,3),d['roofline']['kernel'],d['rmse']['test'])"; done
timeout 1200 python scripts/stale_margin.py 64,128 --shape 120000,17700,25000000 --lrs 0.005,0.01 --dtypes float32 --epochs 5 > $O/margin_nf.jsonl 2> $O/margin_nf.err; cat $O/margin_nf.jsonl
