timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -s -k "config2 or config1" 2>&1 | grep -E "parity|passed|failed" | cut -c1-300
CMTCS_PHASE_LOG=1 timeout 60 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "cmtcs\] EM|value" | cut -c1-200
CMTCS_PHASE_LOG=1 timeout 100 python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "cmtcs\] EM|value|Error" | cut -c1-200
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -s 2>&1 | grep -E "C[345] task|passed|failed|Error"
