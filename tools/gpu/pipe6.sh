timeout 120 python tools/pipe_check.py C2 C3 2>&1 | grep -v "dyn \|sweep\|fine k"
RSW_PROFILE_COARSE=1 timeout 300 python tools/coarse_timing.py C3 2>&1 | tail -3
for cfg in "32 4" "16 6"; do set -- $cfg; echo "== GC=$1 NG=$2"; RSW_PIPE_TRACE=1 RSW_PIPE_GC=$1 RSW_PIPE_NG=$2 timeout 120 python tools/pipe_check.py C3 2>&1 | grep "identical\|schedule=2\|sweep\|fine k"; done
