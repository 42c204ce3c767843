mkdir -p gpurun_out/probe
for a in "64 f32 65536" "64 f32" "128 f32" "32 f32 65536" "128 f16 65536"; do
  timeout 200 python scripts/stream_chunk_probe.py $a >> gpurun_out/probe/chunks.jsonl 2>>gpurun_out/probe/err.log
done
