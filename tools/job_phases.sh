timeout 200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for f in 0 32; do echo "DBG=$f"; CMTCS_DBG=$f CMTCS_PHASE_LOG=1 timeout 60 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "cmtcs\] EM|value" | cut -c1-200; done
CMTCS_PHASE_LOG=1 timeout 100 python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "cmtcs\] EM|value|Error" | cut -c1-200
