# cluster-mode pipelined solve: trace, bitwise check vs bulk, bench
RSW_PIPE_TRACE=1 timeout 120 python tools/pipe_check.py C3 2>&1 | grep -v "^\[rsw pipe\] fine" | tail -14
echo "== pipelined tests"
timeout 300 python -m pytest tests -m gpu -q -x -k "pipelined or parareal_c3 or divergence" 2>&1 | tail -3
