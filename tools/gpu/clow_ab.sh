RSW_LIB=variants/clow.so timeout 600 python -m pytest tests -m gpu -q -x -k "pipelined" 2>&1 | tail -2
for i in 1 2; do
  timeout 300 python tools/c3_ab.py C3 5
  RSW_LIB=variants/clow.so timeout 300 python tools/c3_ab.py C3 5
done
