RSW_PIPE_TRACE=1 timeout 120 python tools/c3_ab.py C3 1 2>&1 | grep -E "rsw pipe\] sweep|total"
timeout 900 python -m pytest tests -m gpu -q -x -k "pipelined or pipe" 2>&1 | tail -2
for i in 1 2; do
  timeout 300 python tools/c3_ab.py C3 7
  RSW_LIB=variants/prering.so timeout 300 python tools/c3_ab.py C3 7
done
