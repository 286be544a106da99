# quick check: parity, kernel timings, bench (no cpu baseline)
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/run_kernel.py --config C5 --what fine --reps 3 --slices 1184 2>&1 | tail -1
timeout 300 python tools/run_kernel.py --config C3 --what fine --reps 3 2>&1 | tail -1
timeout 300 python tools/run_kernel.py --config C3 --what fine --reps 3 --slices 4736 2>&1 | tail -1
timeout 300 python tools/run_kernel.py --what avg --reps 3 2>&1 | tail -1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; echo "bench exit $?"
python - <<'PY'
import json
l=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1])
print({k:l[k] for k in ['value','ms_per_step']}, 'pipe frac', round(l['roofline']['frac'],4), 'fine', round(l['roofline_fine']['achieved'],3), l['clocks'])
PY
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine -c 1 -o gpurun_out/q_fine_c5 python tools/run_kernel.py --config C5 --what fine --reps 1 --slices 592 > gpurun_out/ncu_q.log 2>&1; echo "ncu c5 $?"
fi
for r in $RADICES; do
RSW_FINE_R=$r timeout 300 python tools/run_kernel.py --config C3 --what fine --reps 3 2>&1 | tail -1
RSW_FINE_R=$r timeout 300 python tools/run_kernel.py --config C3 --what fine --reps 3 --slices 4736 2>&1 | tail -1
done
