# triad sweeps round 2: parity suite, C3 A/B over coarse-thread / fine-group variants and NG
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -4 gpurun_out/pytest_gpu.log
for ng in 2 3 4 6; do RSW_PIPE_NG=$ng timeout 300 python tools/c3_ab.py C3 5 2>&1 | tail -1; done
for v in t288n1 t128n1; do for ng in 3 6; do RSW_LIB=variants/$v.so RSW_PIPE_NG=$ng timeout 300 python tools/c3_ab.py C3 5 2>&1 | sed "s/^/$v NG=$ng /" | tail -1; done; done
RSW_COARSE_TRIAD=0 timeout 300 python tools/c3_ab.py C3 3 2>&1 | tail -1
for c in C1 C2; do timeout 300 python tools/c3_ab.py $c 3 2>&1 | tail -1; RSW_COARSE_TRIAD=0 timeout 300 python tools/c3_ab.py $c 3 2>&1 | tail -1; done
