timeout 300 python tools/c3_ab.py C3 5 2>&1 | sed "s/^/base /" | tail -1
for o in 4 5 6; do RSW_PIPE_COARSE_SOLO=1 RSW_PIPE_TRIAD_NOWN=$o timeout 300 python tools/c3_ab.py C3 5 2>&1 | sed "s/^/solo NOWN=$o /" | tail -1; done
RSW_PIPE_COARSE_SOLO=1 RSW_PIPE_TRACE=1 timeout 120 python tools/pipe_check.py C3 2>&1 | grep -E "sweep 0 stage" | tail -1
