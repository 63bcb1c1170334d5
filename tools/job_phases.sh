timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -s --durations=5 2>&1 | grep -E "C[345] task|passed|failed|Error|assert|slowest|s call" | head -30
