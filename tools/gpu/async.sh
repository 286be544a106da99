timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "averaged or small_M or triad" > gpurun_out/pytest_avg.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_avg.log
timeout 120 python tools/c4_time.py 2>&1 | tail -1
RSW_LIB=variants/async0.so timeout 120 python tools/c4_time.py 2>&1 | tail -1
timeout 120 python tools/c4_time.py 2>&1 | tail -1
