timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s 2>&1 | grep -E "parity|multiround|passed|failed|assert|Error" | cut -c1-330
CMTCS_PHASE_LOG=1 timeout 120 python bench.py --config 2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline 2>&1 | grep -E "cmtcs\]" | grep -E "EM it|update" | cut -c1-250
CMTCS_PHASE_LOG=1 timeout 120 python bench.py --config 3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline 2>&1 | grep -E "cmtcs\] EM"
