RSW_PIPE_TRACE=1 timeout 120 python tools/c3_ab.py C3 1 2>&1 | grep -E "rsw pipe\] sweep [0-9]|total"
timeout 600 python -m pytest tests -m gpu -q -x -k "pipelined" 2>&1 | tail -2
for i in 1 2; do
  timeout 300 python tools/c3_ab.py C3 7
  RSW_LIB=variants/reuse0.so timeout 300 python tools/c3_ab.py C3 7
done
