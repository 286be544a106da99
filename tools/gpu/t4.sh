timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 120 python tools/pipe_check.py C2 C3 2>&1 | grep "identical\|schedule=2"
for cfg in "64 2" "16 6" "24 6"; do set -- $cfg; echo "== GC=$1 NG=$2"; RSW_PIPE_GC=$1 RSW_PIPE_NG=$2 timeout 120 python tools/pipe_check.py C3 2>&1 | grep "identical\|schedule=2"; done
