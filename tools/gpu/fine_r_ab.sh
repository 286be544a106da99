for r in 8 4 82; do echo "R=$r"; RSW_FINE_R=$r timeout 300 python tools/run_kernel.py --config C3 --what fine --reps 5 2>&1 | tail -1; done
for r in 8 4; do echo "phase R=$r"; RSW_LIB=variants/phase.so RSW_FINE_R=$r timeout 300 python tools/run_kernel.py --config C3 --what fine --reps 1 2>&1 | grep cycles | head -2; done
