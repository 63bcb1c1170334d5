timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -s -k "full_run" 2>&1 | grep -E "C2 full run|passed|failed|assert" | cut -c1-600
