timeout 300 python tools/pipe_check.py C1 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --section LaunchStats --section Occupancy -k regex:k_parareal -c 1 python tools/pipe_check.py C1 > gpurun_out/ncu_occ.log 2>&1; echo $?
grep -i "occupancy\|limit\|barrier\|Registers\|Shared" gpurun_out/ncu_occ.log | head -40
