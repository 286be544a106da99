for w in C3 C5; do
timeout 300 python tools/bulk_ab.py $w 3 512
RSW_NO_DIE_AWARE=1 timeout 300 python tools/bulk_ab.py $w 3 512
done
RSW_DIE_PROBE_DEBUG=1 timeout 300 python tools/bulk_ab.py C3 1 64 2>&1 | grep -v "pairs (smid" | cut -c1-300
