RSW_PIPE_TRACE=1 timeout 120 python tools/pipe_check.py C3 2>&1 | grep -E "sweep [05]:|C3" | tail -4
timeout 300 python tools/c3_ab.py C3 7 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
