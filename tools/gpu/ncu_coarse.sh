# bulk coarse sweep (C3, k = 0 only): where does the per-stage latency go?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_coarse_sweep -c 1 -o gpurun_out/coarse_c3 python tools/c3_bulk_prof.py > gpurun_out/ncu_coarse.log 2>&1; echo "ncu $?"
python tools/ncu_summary.py gpurun_out/coarse_c3.ncu-rep > gpurun_out/coarse_c3.txt 2>&1
python tools/ncu_lines.py gpurun_out/coarse_c3.ncu-rep > gpurun_out/coarse_c3_lines.txt 2>&1
cat gpurun_out/coarse_c3.txt; head -40 gpurun_out/coarse_c3_lines.txt
