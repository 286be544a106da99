timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/run_kernel.py --what avg --reps 5 2>&1 | tail -1
RSW_COARSE_TRIAD=0 timeout 300 python tools/run_kernel.py --what avg --reps 5 2>&1 | tail -1
for v in avgb4 avgb16; do RSW_LIB=variants/$v.so timeout 300 python tools/run_kernel.py --what avg --reps 5 2>&1 | sed "s/^/$v /" | tail -1; done
