set -x
SEL='kv_stable or (grouped and (32-8 or 28-4)) or graph or append_plain'
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_gpu_attn.py -q -x -k "$SEL" > gpurun_out/r02j_san_attn_$tool.log 2>&1; echo "attn $tool rc=$?"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_gpu_swap.py -q -x > gpurun_out/r02j_san_swap_$tool.log 2>&1; echo "swap $tool rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 40 -c 1 -o gpurun_out/r02j_ncu_c3 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-prefill --no-swap > gpurun_out/r02j_ncu_c3.log 2>&1; echo ncu_c3=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 30 -c 1 -o gpurun_out/r02j_ncu_c4n8 python tools/shard_time.py c4 --n 8 --reps 1 > gpurun_out/r02j_ncu_c4n8.log 2>&1; echo ncu_c4n8=$?
