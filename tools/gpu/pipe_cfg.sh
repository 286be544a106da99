# pipelined C3 solve under several coarse-group layouts (GC sub-CTAs per sweep, NG concurrent sweeps)
for cfg in "24 6" "32 4" "22 6" "28 5" "48 3"; do set -- $cfg; echo "== GC=$1 NG=$2"; RSW_PIPE_GC=$1 RSW_PIPE_NG=$2 timeout 120 python tools/pipe_check.py C3 2>&1 | grep "identical\|schedule=2"; done
