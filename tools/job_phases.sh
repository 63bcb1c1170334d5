timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
CMTCS_PHASE_LOG=1 timeout 60 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "cmtcs\] EM|value" | cut -c1-200
CMTCS_PHASE_LOG=1 timeout 100 python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "cmtcs\] EM|value|Error" | cut -c1-200
timeout 200 python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "value|Error" | cut -c1-200
