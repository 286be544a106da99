./tools/micro/warp_slots
for i in 1 2; do
  timeout 300 python tools/c3_ab.py C3 7
  RSW_LIB=variants/wswap.so timeout 300 python tools/c3_ab.py C3 7
done
