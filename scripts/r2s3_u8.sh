#!/bin/bash
# e2e with 1-byte user ids (run groups over <= 256-row tiles, 5 B/rating):
# resident throughput at 256-row tiles, the default bench line, streaming tests.
O=gpurun_out/${1:-s3w}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_engine.py -k "streaming" -q -x > $O/pytest.log 2>&1; tail -n 1 $O/pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --tile-rows 256 > $O/resident_256.json 2> $O/resident_256.err
python -c "import json;d=json.load(open('$O/resident_256.json'));print('resident 256-row tiles',round(d['value']/1e9,2))"
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_default.json 2> $O/bench_default.err
python -c "import json;d=json.load(open('$O/bench_default.json'));e=d['e2e'];print('default',round(d['value']/1e9,2),'e2e',round(e['value']/1e9,2),e['h2d_bytes_per_step'],e['ms_per_step'],e['test_rmse_after'])"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --stream-tile-rows 0 > $O/bench_u16.json 2> $O/bench_u16.err
python -c "import json;d=json.load(open('$O/bench_u16.json'));e=d['e2e'];print('u16 stream',round(e['value']/1e9,2),e['h2d_bytes_per_step'])"
for k in 32 64 256; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --k $k > $O/bench_k$k.json 2> $O/bench_k$k.err
python -c "import json;d=json.load(open('$O/bench_k$k.json'));e=d['e2e'];print('k $k',round(d['value']/1e9,2),'e2e',round(e['value']/1e9,2),e['h2d_bytes_per_step'])"
done
