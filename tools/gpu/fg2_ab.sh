RSW_LIB=variants/fg2.so RSW_PIPE_TRACE=1 timeout 120 python tools/c3_ab.py C3 1 2>&1 | grep -E "rsw pipe\] (n=|grid|sweep [0-9])|total"
for i in 1 2; do
  timeout 300 python tools/c3_ab.py C3 5
  RSW_LIB=variants/fg2.so timeout 300 python tools/c3_ab.py C3 5
done
