# round-2 measurement refresh after the die-homing work: parity, smoke, bench, launch list, ncu of the
# pipelined solve (the fine / N-bar kernels are unchanged since r2_final.sh)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke $?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err; echo "bench exit $?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref2.json 2> gpurun_out/bench_ref2.err; echo "ref exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c5-iteration > gpurun_out/ncu_launch2.log 2>&1; echo "ncu launches $?"
python tools/launch_summary.py gpurun_out/launches_final2.csv "C3 bench" > gpurun_out/launches_final2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_parareal_pipe -c 1 -o gpurun_out/g_pipe_c3 python tools/run_kernel.py --config C3 --what parareal --reps 1 --iters 5 > gpurun_out/ncu_g4.log 2>&1; echo "ncu pipe $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_coarse_sweep -c 1 -o gpurun_out/g_coarse_c3 python tools/c3_bulk_prof.py > gpurun_out/ncu_g5.log 2>&1; echo "ncu coarse $?"
for r in g_pipe_c3 g_coarse_c3; do
  python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.txt 2>&1
  python tools/ncu_dpflops.py gpurun_out/$r.ncu-rep > gpurun_out/${r}_dp.json 2>&1
  python tools/ncu_lines.py gpurun_out/$r.ncu-rep 40 > gpurun_out/${r}_lines.txt 2>&1
done
rm -f gpurun_out/g_pipe_c3.ncu-rep gpurun_out/g_coarse_c3.ncu-rep
