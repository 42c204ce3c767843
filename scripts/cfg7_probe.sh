mkdir -p gpurun_out/cfg7
for kp in "32 f32" "32 f16" "64 f32" "64 f16"; do
  set -- $kp
  for c in -1 7; do
    timeout 200 python bench.py --steps 8 --warmup 3 --k $1 --precision $2 --no-cpu --no-e2e \
      --chain-cfg $c 2>>gpurun_out/cfg7/err.log | tail -1 | sed "s/^/{\"cfg\": $c, \"line\": /; s/\$/}/" >> gpurun_out/cfg7/sweep.jsonl
  done
done
