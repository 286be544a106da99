RSW_PIPE_TRACE=1 timeout 120 python tools/pipe_check.py C3 2>&1 | grep "stage\|identical\|schedule=2\|grid" | tail -4
RSW_PIPE_NG=1 RSW_PIPE_GC=64 RSW_PIPE_TRACE=1 timeout 120 python tools/pipe_check.py C3 2>&1 | grep "stage\|schedule=2" | tail -2
RSW_PROFILE_COARSE=1 timeout 300 python tools/coarse_timing.py C3 2>&1 | tail -3
