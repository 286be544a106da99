RSW_PIPE_TRACE=1 timeout 120 python tools/pipe_check.py C3 2>&1 | grep "rsw pipe" | tail -14
