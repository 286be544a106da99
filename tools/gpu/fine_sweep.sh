# parity + fine-kernel timing per radix (RSW_FINE_RADIX) on C3 and C5
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for r in 0 4 8 32; do
  echo "== radix $r"
  RSW_FINE_RADIX=$r timeout 300 python tools/run_kernel.py --config C3 --what fine --reps 3 2>&1 | tail -1
  RSW_FINE_RADIX=$r timeout 300 python tools/run_kernel.py --config C5 --what fine --reps 3 --slices 1184 2>&1 | tail -1
done
