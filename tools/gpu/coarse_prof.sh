RSW_PROFILE_COARSE=1 timeout 300 python tools/coarse_timing.py C3 2>&1 | tail -6
timeout 300 python tools/coarse_timing.py C2 C3 2>&1 | tail -3
