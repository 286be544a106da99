# C3 fine kernel (the pipelined solve's per-iteration lag): radix A/B and an ncu capture with source lines
for r in 8 4 82; do RSW_FINE_R=$r timeout 300 python tools/run_kernel.py --config C3 --what fine --reps 3 2>&1 | tail -1; done
timeout 300 python tools/run_kernel.py --config C3 --what fine --reps 3 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine -c 1 -o gpurun_out/fine_c3 python tools/run_kernel.py --config C3 --what fine --reps 1 > gpurun_out/ncu_fc3.log 2>&1; echo "ncu $?"
python tools/ncu_summary.py gpurun_out/fine_c3.ncu-rep
