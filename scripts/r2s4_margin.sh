#!/bin/bash
O=gpurun_out/${1:-s4margin}; mkdir -p $O
timeout 900 python scripts/stale_margin.py 32,64,128 > $O/default.jsonl 2> $O/default.err; cat $O/default.jsonl
cp paper_2006_15980_b200/lib/libhmf.so /tmp/libhmf_default.so
for v in build/var/*; do n=$(basename $v); cp $v/libhmf.so paper_2006_15980_b200/lib/libhmf.so
  timeout 600 python scripts/stale_margin.py 64 > $O/$n.jsonl 2> $O/$n.err; echo "== $n"; cat $O/$n.jsonl; done
cp /tmp/libhmf_default.so paper_2006_15980_b200/lib/libhmf.so
