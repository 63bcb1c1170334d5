timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -s -k "3" 2>&1 | grep -E "C[345]|passed|failed" | cut -c1-250
