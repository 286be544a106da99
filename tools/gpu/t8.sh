timeout 120 python tools/pipe_check.py C3 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "Error|FAILED|assert" | head -5
