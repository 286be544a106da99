for o in 2 3; do for ng in 3 4; do RSW_LIB=variants/tm3c192.so RSW_PIPE_TRIAD_NOWN=$o RSW_PIPE_NG=$ng timeout 300 python tools/c3_ab.py C3 5 2>&1 | sed "s/^/NOWN=$o NG=$ng /" | tail -1; done; done
