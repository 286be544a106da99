# die-homed coarse exchange arrays: probe result, correctness, A/B
RSW_PIPE_TRACE=1 timeout 120 python tools/c3_ab.py C3 1 2>&1 | grep -E "rsw pipe\] grid|total"
timeout 900 python -m pytest tests -m gpu -q -x -k "pipelined or pipe or multigpu or coarse or parity" 2>&1 | tail -3
for i in 1 2; do
  timeout 300 python tools/c3_ab.py C3 7
  RSW_NO_DIE_AWARE=1 timeout 300 python tools/c3_ab.py C3 7
  RSW_NO_DIE_PROBE=1 timeout 300 python tools/c3_ab.py C3 7
done
