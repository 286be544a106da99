# pipelined C3: trace of sweeps / stage phases, and the bulk coarse stage profile
RSW_PIPE_TRACE=1 timeout 120 python tools/pipe_check.py C3 2>&1 | grep -v "^\[rsw pipe\] n=" | tail -22
RSW_PROFILE_COARSE=1 timeout 300 python tools/coarse_timing.py C3 2>&1 | tail -4
