timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo "bench exit $?"
tail -1 gpurun_out/bench_c3.log
