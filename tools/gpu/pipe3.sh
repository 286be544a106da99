RSW_PIPE_GRID=296 RSW_PIPE_TRACE=1 timeout 120 python tools/pipe_check.py C3 2>&1 | grep -v "dyn " | tail -16
