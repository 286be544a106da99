for cfg in "3 4" "2 2" "2 3" "3 3" "2 4" "4 4"; do set -- $cfg; RSW_PIPE_NG=$1 RSW_PIPE_TRIAD_NOWN=$2 timeout 300 python tools/c3_ab.py C3 5 2>&1 | sed "s/^/NG=$1 NOWN=$2 /" | tail -1; done
RSW_PIPE_NG=2 RSW_PIPE_TRIAD_NOWN=2 RSW_PIPE_TRACE=1 timeout 120 python tools/pipe_check.py C3 2>&1 | grep -E "sweep 0 stage|grid" | tail -2
