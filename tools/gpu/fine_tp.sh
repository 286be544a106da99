for s in 296 592 1184 2368 4736; do timeout 300 python tools/run_kernel.py --config C3 --what fine --reps 3 --slices $s 2>&1 | tail -1; done
for s in 296 1184 4736; do RSW_FINE_RADIX=16 timeout 300 python tools/run_kernel.py --config C3 --what fine --reps 3 --slices $s 2>&1 | tail -1; done
