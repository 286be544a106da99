# triad coarse sweeps: parity first, then C3 A/B (quadrature vs triad, NG variants), bulk sweep alone
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/pytest_gpu.log
RSW_COARSE_TRIAD=0 timeout 300 python tools/c3_ab.py C3 5 2>&1 | tail -1
for ng in 2 3 6; do RSW_PIPE_NG=$ng timeout 300 python tools/c3_ab.py C3 5 2>&1 | tail -1; done
timeout 300 python tools/c3_sweep0.py 2>&1 | tail -3
RSW_COARSE_TRIAD=0 timeout 300 python tools/c3_sweep0.py 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; echo "bench exit $?"
python - <<'PY'
import json
l=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1])
print({k:l[k] for k in ['value','ms_per_step']}, 'pipe frac', round(l['roofline']['frac'],4), l.get('phases_ms'), l['clocks'])
PY
