for c in C1 C2 C3; do timeout 300 python tools/c3_ab.py $c 5 2>&1 | sed "s/^/$c /" | tail -1; done
RSW_PIPE_EXTRA_FINE=1 timeout 300 python tools/c3_ab.py C2 5 2>&1 | sed "s/^/C2 extra /" | tail -1
RSW_PIPE_NG=6 timeout 300 python tools/c3_ab.py C2 5 2>&1 | sed "s/^/C2 NG6 /" | tail -1
RSW_PIPE_NG=12 timeout 300 python tools/c3_ab.py C2 5 2>&1 | sed "s/^/C2 NG12 /" | tail -1
timeout 300 python tools/c5_sweep.py 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
