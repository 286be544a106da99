# parity, coarse stage profile, fine timing, bench (C3)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
RSW_PROFILE_COARSE=1 timeout 300 python tools/coarse_timing.py C3 2>&1 | tail -3
timeout 300 python tools/run_kernel.py --config C3 --what fine --reps 3 2>&1 | tail -1
timeout 300 python tools/run_kernel.py --config C5 --what fine --reps 3 --slices 1184 2>&1 | tail -1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?"
python - <<'PY'
import json
l=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print({k:l[k] for k in ['value','ms_per_step','phases_ms','fine_kernel_slice_steps_per_s']}, l['roofline']['achieved'], l['roofline']['frac'], l['clocks'])
PY
