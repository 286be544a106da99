# session 3 re-entry: parity, bench (C3, with cpu baseline), launch list, ncu full of fine C5 + pipe C3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_c3.log
timeout 300 python tools/run_kernel.py --config C5 --what fine --reps 3 --slices 1184 2>&1 | tail -1
timeout 300 python tools/run_kernel.py --config C3 --what fine --reps 3 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine -c 1 -o gpurun_out/fine_c5 python tools/run_kernel.py --config C5 --what fine --reps 1 --slices 296 > gpurun_out/ncu2.log 2>&1; echo "ncu c5 $?"
