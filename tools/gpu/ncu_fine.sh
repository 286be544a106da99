# full ncu capture of the fine kernel, C3 (radix 8) and C5 (radix 16)
python tools/run_kernel.py --config C3 --what fine --reps 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine -c 1 -o gpurun_out/fine5_c3 python tools/run_kernel.py --config C3 --what fine --reps 1 > gpurun_out/ncu1.log 2>&1
echo "c3 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine -c 1 -o gpurun_out/fine5_c5 python tools/run_kernel.py --config C5 --what fine --reps 1 --slices 296 > gpurun_out/ncu2.log 2>&1
echo "c5 $?"
