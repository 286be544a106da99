# DRAM traffic (ncu --set full) of the bench's dominant kernel: k_parareal_pipe on C3 with 5 iterations
timeout 900 ncu --set full --clock-control none -k regex:k_parareal_pipe -c 1 -o gpurun_out/t_pipe_c3 python tools/run_kernel.py --config C3 --what parareal --reps 1 --iters 5 > gpurun_out/ncu_t1.log 2>&1; echo "ncu pipe $?"
python tools/ncu_summary.py gpurun_out/t_pipe_c3.ncu-rep > gpurun_out/t_pipe_c3.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_fine -c 1 -o gpurun_out/t_fine_c5 python tools/run_kernel.py --config C5 --what fine --reps 1 --slices 4096 > gpurun_out/ncu_t2.log 2>&1; echo "ncu c5 $?"
python tools/ncu_summary.py gpurun_out/t_fine_c5.ncu-rep > gpurun_out/t_fine_c5.txt 2>&1
rm -f gpurun_out/t_pipe_c3.ncu-rep gpurun_out/t_fine_c5.ncu-rep
