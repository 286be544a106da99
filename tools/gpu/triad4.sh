# triad pipelined layouts: stage trace + (GC, NG) scan on C3
RSW_PIPE_TRACE=1 timeout 120 python tools/pipe_check.py C3 2>&1 | grep -E "stage|sweep [0-9]|fine k|triad|C3" | tail -16
for cfg in "24 3" "24 2" "30 3" "37 3" "37 2" "20 3" "16 2" "43 2"; do set -- $cfg; RSW_PIPE_GC=$1 RSW_PIPE_NG=$2 timeout 300 python tools/c3_ab.py C3 5 2>&1 | sed "s/^/GC=$1 NG=$2 /" | tail -1; done
