timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "mixed" 2>&1 | grep -E "mixed|passed|failed|assert|Error" | cut -c1-300
