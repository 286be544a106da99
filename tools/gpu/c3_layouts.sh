# C3 pipelined solve under coarse-group layouts (GC CTAs per sweep, NG sweeps in flight)
timeout 300 python tools/c3_ab.py C3 5
for l in "32 3" "32 4" "22 6" "43 3" "64 2" "21 7" "16 6"; do set -- $l
  echo "GC=$1 NG=$2"; RSW_PIPE_GC=$1 RSW_PIPE_NG=$2 timeout 300 python tools/c3_ab.py C3 5
done
