timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -4 gpurun_out/pytest_gpu.log
for ng in 3 4; do RSW_PIPE_NG=$ng timeout 300 python tools/c3_ab.py C3 5 2>&1 | tail -1; done
for v in t288n2m1 t192n3m1; do for ng in 3 4 6; do RSW_LIB=variants/$v.so RSW_PIPE_NG=$ng timeout 300 python tools/c3_ab.py C3 5 2>&1 | sed "s/^/$v NG=$ng /" | tail -1; done; done
