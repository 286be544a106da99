for v in 0 1 2 3 4 5; do echo "== variant $v"; RSW_COARSE_VARIANT=$v RSW_PROFILE_COARSE=1 timeout 300 python tools/coarse_timing.py C3 2>&1 | tail -3; done
