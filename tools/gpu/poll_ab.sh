for i in 1 2; do
  timeout 300 python tools/c3_ab.py C3 5
  RSW_LIB=variants/poll200.so timeout 300 python tools/c3_ab.py C3 5
  RSW_LIB=variants/poll500.so timeout 300 python tools/c3_ab.py C3 5
  RSW_LIB=variants/prering.so timeout 300 python tools/c3_ab.py C3 5
done
