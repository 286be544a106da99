timeout 300 python tools/c3_ab.py C3 7 2>&1 | tail -1
RSW_PIPE_EXTRA_YOUNG=1 timeout 300 python tools/c3_ab.py C3 7 2>&1 | tail -1
timeout 300 python tools/c3_ab.py C3 7 2>&1 | tail -1
RSW_PIPE_EXTRA_YOUNG=1 timeout 300 python tools/c3_ab.py C3 7 2>&1 | tail -1
