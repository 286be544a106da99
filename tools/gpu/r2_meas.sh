# round-2 measurement set: parity, bench (C3 + cpu baseline), launch list of the bench, ncu of the
# headline kernel (k_parareal_pipe, C3, 5 iterations) with its DP flop count, variant timings
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; echo "bench exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c5-iteration > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches $?"
python tools/launch_summary.py gpurun_out/launches_r2.csv "C3 bench" > gpurun_out/launches_r2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_parareal_pipe -c 1 -o gpurun_out/r2_pipe_c3 python tools/run_kernel.py --config C3 --what parareal --reps 1 --iters 5 > gpurun_out/ncu_pipe.log 2>&1; echo "ncu pipe $?"
python tools/ncu_summary.py gpurun_out/r2_pipe_c3.ncu-rep > gpurun_out/r2_pipe_c3.txt 2>&1
python tools/ncu_dpflops.py gpurun_out/r2_pipe_c3.ncu-rep > gpurun_out/r2_pipe_c3_dp.json 2>&1
python tools/ncu_lines.py gpurun_out/r2_pipe_c3.ncu-rep 40 > gpurun_out/r2_pipe_c3_lines.txt 2>&1
rm -f gpurun_out/r2_pipe_c3.ncu-rep
timeout 300 python tools/run_kernel.py --what avg --reps 3 2>&1 | tail -1
