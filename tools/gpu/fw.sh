timeout 300 python tools/c3_ab.py C3 5 2>&1 | tail -1
for v in c256t3 c256t2; do RSW_LIB=variants/$v.so timeout 300 python tools/c3_ab.py C3 5 2>&1 | tail -1; done
