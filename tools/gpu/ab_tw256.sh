# A/B: n = 256 fine kernels (k_fine, pipelined fine workers) reading full twiddle tables from TMEM
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
RSW_LIB=variants/librsw_tw256.so timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "pipelined or c3 or fine_sizes or virtual" > gpurun_out/pytest_v.log 2>&1; echo "pytest variant exit $?"; tail -2 gpurun_out/pytest_v.log
for v in paper_1303_6615_b200/librsw.so variants/librsw_tw256.so; do
  echo "== $v"
  RSW_LIB=$v timeout 300 python tools/run_kernel.py --config C3 --what fine --reps 3 2>&1 | tail -1
  RSW_LIB=$v RSW_PIPE_TRACE=1 timeout 120 python tools/pipe_check.py C3 2>&1 | grep -E "sweep 0 stage|fine k=4|schedule=2|bitwise" | tail -4
  RSW_LIB=$v RSW_PROFILE_COARSE=1 timeout 300 python tools/coarse_timing.py C3 2>&1 | tail -1
done
