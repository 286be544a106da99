RSW_PIPE_TRACE=1 timeout 120 python tools/pipe_check.py C3 2>&1 | grep -E "stage|sweep [0-9]|triad|C3" | tail -16
timeout 300 python tools/c3_ab.py C3 7 2>&1 | tail -1
RSW_LIB=variants/nb8.so timeout 300 python tools/c3_ab.py C3 7 2>&1 | tail -1
for o in 3 5; do RSW_PIPE_TRIAD_NOWN=$o timeout 300 python tools/c3_ab.py C3 5 2>&1 | sed "s/^/NOWN=$o /" | tail -1; done
RSW_PIPE_NG=4 timeout 300 python tools/c3_ab.py C3 5 2>&1 | sed "s/^/NG=4 /" | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -4 gpurun_out/pytest_gpu.log
