# C3 focus: parity, C3 fine kernel timing, pipelined trace, bench line
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python tools/run_kernel.py --config C3 --what fine --reps 3 2>&1 | tail -1
timeout 300 python tools/run_kernel.py --config C5 --what fine --reps 3 --slices 1184 2>&1 | tail -1
timeout 300 python tools/run_kernel.py --what avg --reps 3 2>&1 | tail -1
RSW_PIPE_TRACE=1 timeout 120 python tools/pipe_check.py C3 2>&1 | grep -v "^\[rsw pipe\] n=" | tail -22
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; echo "bench exit $?"
python - <<'PY'
import json
l=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1])
print({k:l[k] for k in ['value','ms_per_step']}, 'pipe frac', round(l['roofline']['frac'],4), 'fine', round(l['roofline_fine']['achieved'],3), 'c5', round(l['fine_c5']['achieved_tflops'],2), 'c4', round(l['avg_c4']['achieved_tflops'],2), l['clocks'])
PY
