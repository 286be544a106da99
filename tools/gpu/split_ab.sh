RSW_PROFILE_COARSE=1 timeout 200 python tools/c3_bulk_prof.py 2>&1 | grep "triad phase" | tail -1
RSW_LIB=variants/split0.so RSW_PROFILE_COARSE=1 timeout 200 python tools/c3_bulk_prof.py 2>&1 | grep "triad phase" | tail -1
RSW_PIPE_TRACE=1 timeout 120 python tools/pipe_check.py C3 2>&1 | grep -E "sweep 0 stage" | tail -1
RSW_LIB=variants/split0.so RSW_PIPE_TRACE=1 timeout 120 python tools/pipe_check.py C3 2>&1 | grep -E "sweep 0 stage" | tail -1
timeout 300 python tools/c3_ab.py C3 7 2>&1 | tail -1
RSW_LIB=variants/split0.so timeout 300 python tools/c3_ab.py C3 7 2>&1 | tail -1
timeout 300 python tools/c5_sweep.py 2>&1 | head -1
RSW_LIB=variants/split0.so timeout 300 python tools/c5_sweep.py 2>&1 | head -1
