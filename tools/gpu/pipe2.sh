RSW_PIPE_TRACE=1 timeout 300 python tools/pipe_check.py C3 2>&1 | tail -25
