timeout 300 python tools/pipe_check.py C1 C2 C3 2>&1 | tail -12
