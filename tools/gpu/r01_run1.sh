set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo "bench exit $?"
timeout 600 python bench.py --steps 3 --warmup 3 --config C5 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo "bench c5 exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fine -c 1 -o gpurun_out/fine_c3 python tools/run_kernel.py --config C3 --what fine --reps 1 > gpurun_out/ncu_fine_c3.log 2>&1; echo "ncu fine c3 $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fine -c 1 -o gpurun_out/fine_c5 python tools/run_kernel.py --config C5 --what fine --reps 1 --slices 1184 > gpurun_out/ncu_fine_c5.log 2>&1; echo "ncu fine c5 $?"
