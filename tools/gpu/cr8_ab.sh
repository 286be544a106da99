RSW_LIB=variants/cr8.so timeout 900 python -m pytest tests -m gpu -q -x -k "coarse or parity or c5 or C5" 2>&1 | tail -2
for i in 1 2; do
  timeout 300 python tools/bulk_ab.py C5 3 256
  RSW_LIB=variants/cr8.so timeout 300 python tools/bulk_ab.py C5 3 256
done
