CUDA_LAUNCH_BLOCKING=1 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "test_fine_c1" 2>&1 | grep -E "Error|error|rsw" | head -20
