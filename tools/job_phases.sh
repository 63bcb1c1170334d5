for i in 1 2 3; do CMTCS_PHASE_LOG=1 timeout 60 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "cmtcs\] EM" | cut -c1-200; done
