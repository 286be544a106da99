timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python tools/pipe_check.py C1 C2 C3 2>&1 | grep "identical\|schedule=2"
for cfg in "64 2" "32 4" "16 6"; do set -- $cfg; echo "== GC=$1 NG=$2"; RSW_PIPE_TRACE=1 RSW_PIPE_GC=$1 RSW_PIPE_NG=$2 timeout 120 python tools/pipe_check.py C3 2>&1 | grep "identical\|schedule=2\|sweep 0\|sweep 5\|fine k=0"; done
