timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -s 2>&1 | grep -E "multiround|mixed|C2 parity|passed|failed" | cut -c1-250
CMTCS_PHASE_LOG=1 timeout 120 python bench.py --config 3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline 2>&1 | grep -E "cmtcs\] EM|rror" | head -3
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -s 2>&1 | grep -E "C[345]|passed|failed" | cut -c1-250
echo "--- 2-MMA form off"
CMTCS_DBG=4096 timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -s 2>&1 | grep -E "C[345]|passed|failed" | cut -c1-250
