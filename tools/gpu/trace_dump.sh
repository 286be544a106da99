RSW_PIPE_TRACE=1 RSW_PIPE_TRACE_DUMP=gpurun_out/c3_trace.bin timeout 120 python tools/c3_ab.py C3 1 2>&1 | grep -E "total"
python tools/trace_analysis.py gpurun_out/c3_trace.bin
