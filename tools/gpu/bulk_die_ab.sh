timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for w in C3 C5; do
  timeout 300 python tools/bulk_ab.py $w 3 512
  RSW_NO_DIE_AWARE=1 timeout 300 python tools/bulk_ab.py $w 3 512
done
timeout 300 python tools/c3_ab.py C3 5
