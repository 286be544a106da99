timeout 120 python tools/c4_time.py 2>&1 | tail -1
for v in m2 b2m2; do RSW_LIB=variants/$v.so timeout 120 python tools/c4_time.py 2>&1 | tail -1; done
