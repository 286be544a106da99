timeout 300 python tools/c5_sweep.py 2>&1 | tail -2
RSW_TRIAD_WIDE_OFF=1 timeout 300 python tools/c5_sweep.py 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
