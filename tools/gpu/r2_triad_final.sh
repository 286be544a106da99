# round-2 numbers after the triad work: bench, C1/C2/C3 solves in both N-bar forms, C5 sweep, ncu of the C5 triad sweep
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_t2.json 2> gpurun_out/bench_t2.err; echo "bench exit $?"
for c in C1 C2 C3; do timeout 300 python tools/c3_ab.py $c 5 2>&1 | sed "s/^/$c triad /" | tail -1; RSW_COARSE_TRIAD=0 timeout 300 python tools/c3_ab.py $c 5 2>&1 | sed "s/^/$c quadrature /" | tail -1; done
timeout 300 python tools/c5_sweep.py 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_coarse_sweep -c 1 -o gpurun_out/t_sweep_c5 python tools/c5_sweep.py > gpurun_out/ncu_t5.log 2>&1; echo "ncu c5 sweep $?"
python tools/ncu_summary.py gpurun_out/t_sweep_c5.ncu-rep > gpurun_out/t_sweep_c5.txt 2>&1
python tools/ncu_dpflops.py gpurun_out/t_sweep_c5.ncu-rep > gpurun_out/t_sweep_c5_dp.json 2>&1
rm -f gpurun_out/t_sweep_c5.ncu-rep
