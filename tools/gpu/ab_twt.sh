# A/B of the twiddle policies (fft_tw_src) of the n >= 512 kernels: parity with the default build, then
# C5 fine (4096 slices) and C4 N-bar timings for TWT = 0 (register powers), 1 (smem table), 2 (TMEM)
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
for v in variants/librsw_twt0.so variants/librsw_twt1.so paper_1303_6615_b200/librsw.so; do
  echo "== $v"
  RSW_LIB=$v timeout 300 python tools/run_kernel.py --config C5 --what fine --reps 3 2>&1 | tail -1
  RSW_LIB=$v timeout 300 python tools/run_kernel.py --what avg --reps 3 2>&1 | tail -1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine -c 1 -o gpurun_out/ab_fine_c5 python tools/run_kernel.py --config C5 --what fine --reps 1 --slices 592 > gpurun_out/ncu_ab1.log 2>&1; echo "ncu c5 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_avg -c 1 -o gpurun_out/ab_avg_c4 python tools/run_kernel.py --what avg --reps 1 --slices 1184 > gpurun_out/ncu_ab2.log 2>&1; echo "ncu c4 $?"
for r in ab_fine_c5 ab_avg_c4; do python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.txt 2>&1; cat gpurun_out/$r.txt; done
