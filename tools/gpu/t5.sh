RSW_PIPE_TRACE=1 timeout 120 python tools/pipe_check.py C1 C2 C3 2>&1 | grep "identical\|schedule=2\|grid"
for cfg in "16 9" "32 4"; do set -- $cfg; echo "== GC=$1 NG=$2"; RSW_PIPE_GC=$1 RSW_PIPE_NG=$2 timeout 120 python tools/pipe_check.py C2 2>&1 | grep "schedule=2"; done
