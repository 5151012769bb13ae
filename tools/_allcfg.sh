for c in c1 c2 c2s c4 c5; do timeout 600 python bench.py --config $c --no-prefill > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?" >> gpurun_out/allcfg.log; done
