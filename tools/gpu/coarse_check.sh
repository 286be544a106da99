timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for v in 0 4; do echo "== variant $v"; RSW_COARSE_VARIANT=$v RSW_PROFILE_COARSE=1 timeout 300 python tools/coarse_timing.py C3 2>&1 | tail -3; done
