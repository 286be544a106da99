# round measurement set: bench (C3, with cpu baseline), launch list, ncu --set full of the bench's
# standalone fine kernel (C3), the C5 fine kernel (592 slices = 2 waves of 148 two-pair CTAs) and C4 N-bar
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
[ -z "$NOBENCH" ] && { timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_c3.log; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine -c 1 -o gpurun_out/m_fine_c5 python tools/run_kernel.py --config C5 --what fine --reps 1 --slices 592 > gpurun_out/ncu_m1.log 2>&1; echo "ncu c5 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine -c 1 -o gpurun_out/m_fine_c3 python tools/run_kernel.py --config C3 --what fine --reps 1 > gpurun_out/ncu_m2.log 2>&1; echo "ncu c3 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_avg -c 1 -o gpurun_out/m_avg_c4 python tools/run_kernel.py --what avg --reps 1 --slices 1184 > gpurun_out/ncu_m3.log 2>&1; echo "ncu c4 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_parareal_pipe -c 1 -o gpurun_out/m_pipe_c3 python tools/run_kernel.py --config C3 --what parareal --reps 1 > gpurun_out/ncu_m4.log 2>&1; echo "ncu pipe $?"
for r in m_fine_c5 m_fine_c3 m_avg_c4 m_pipe_c3; do python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.txt 2>&1; done
python tools/launch_summary.py gpurun_out/launches_c3.csv "C3 bench" > gpurun_out/launches_c3.txt 2>&1
rm -f gpurun_out/m_pipe_c3.ncu-rep
du -sh gpurun_out/*
