for i in 1 2; do
  timeout 300 python tools/c3_ab.py C3 5
  for ns in 20 50 100; do RSW_LIB=variants/sleep$ns.so timeout 300 python tools/c3_ab.py C3 5; done
done
