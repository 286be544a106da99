# round-2 measurement set after the triad coarse sweeps and the batched triad N-bar (same commands as r2_final.sh)
# bench, ncu --set full of every hot kernel (C5 fine, C3 fine, C4 N-bar, the C3 pipelined solve), DP flops
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_u.json 2> gpurun_out/bench_u.err; echo "bench exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_u.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c5-iteration > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches $?"
python tools/launch_summary.py gpurun_out/launches_u.csv "C3 bench" > gpurun_out/launches_u.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine -c 1 -o gpurun_out/u_fine_c5 python tools/run_kernel.py --config C5 --what fine --reps 1 --slices 592 > gpurun_out/ncu_t1.log 2>&1; echo "ncu c5 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine -c 1 -o gpurun_out/u_fine_c3 python tools/run_kernel.py --config C3 --what fine --reps 1 > gpurun_out/ncu_t2.log 2>&1; echo "ncu c3 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_avg -c 1 -o gpurun_out/u_avg_c4 python tools/run_kernel.py --what avg --reps 1 --slices 1184 > gpurun_out/ncu_t3.log 2>&1; echo "ncu c4 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_parareal_pipe -c 1 -o gpurun_out/u_pipe_c3 python tools/run_kernel.py --config C3 --what parareal --reps 1 --iters 5 > gpurun_out/ncu_t4.log 2>&1; echo "ncu pipe $?"
for r in u_fine_c5 u_fine_c3 u_avg_c4 u_pipe_c3; do
  python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.txt 2>&1
  python tools/ncu_dpflops.py gpurun_out/$r.ncu-rep > gpurun_out/${r}_dp.json 2>&1
  python tools/ncu_lines.py gpurun_out/$r.ncu-rep 40 > gpurun_out/${r}_lines.txt 2>&1
done
rm -f gpurun_out/u_pipe_c3.ncu-rep
du -sh gpurun_out/* | sort -h | tail -5
