timeout 900 python -m pytest tests -m gpu -q -x -k "pipelined or parareal" 2>&1 | tail -2
RSW_PIPE_TRACE=1 timeout 120 python tools/pipe_check.py C2 C3 2>&1 | grep "stage (us)\|identical\|schedule=2\|grid\|threads" | tail -8
for cfg in "32 4" "22 6"; do set -- $cfg; echo "== GC=$1 NG=$2"; RSW_PIPE_TRACE=1 RSW_PIPE_GC=$1 RSW_PIPE_NG=$2 timeout 120 python tools/pipe_check.py C3 2>&1 | grep "stage (us)\|identical\|schedule=2" | tail -3; done
