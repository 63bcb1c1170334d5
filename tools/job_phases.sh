timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
CMTCS_PHASE_LOG=1 timeout 120 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "cmtcs\]|value" | cut -c1-300
