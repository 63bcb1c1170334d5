CMTCS_PHASE_LOG=1 timeout 120 python bench.py --config 3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline 2>&1 | grep -E "cmtcs\]" | cut -c1-200
