timeout 300 python tools/c5_sweep.py 2>&1 | tail -2
RSW_COARSE_TRIAD=0 timeout 300 python tools/c5_sweep.py 2>&1 | tail -2
timeout 300 python tools/run_kernel.py --what avg --reps 5 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
