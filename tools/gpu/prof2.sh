python tools/run_kernel.py --config C3 --what parareal --reps 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_parareal -c 1 -o gpurun_out/pipe_c3 python tools/run_kernel.py --config C3 --what parareal --reps 1 > gpurun_out/ncu_pipe.log 2>&1; echo "ncu pipe $?"
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_v3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fine -c 1 -o gpurun_out/fine6_c5 python tools/run_kernel.py --config C5 --what fine --reps 1 --slices 296 > gpurun_out/ncu_f5.log 2>&1; echo "ncu fine c5 $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fine -c 1 -o gpurun_out/fine6_c3 python tools/run_kernel.py --config C3 --what fine --reps 1 > gpurun_out/ncu_f3.log 2>&1; echo "ncu fine c3 $?"
