timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine -c 1 -o gpurun_out/n_fine_c5 python tools/run_kernel.py --config C5 --what fine --reps 1 --slices 592 > gpurun_out/ncu_n1.log 2>&1; echo "ncu c5 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_avg -c 1 -o gpurun_out/n_avg_c4 python tools/run_kernel.py --what avg --reps 1 --slices 1184 > gpurun_out/ncu_n2.log 2>&1; echo "ncu c4 $?"
for r in n_fine_c5 n_avg_c4; do python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.txt 2>&1; done
