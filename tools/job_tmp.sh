timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
CMTCS_TRACE_STEP=40 CMTCS_PHASE_LOG=1 timeout 120 python bench.py --config 2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline 2>&1 | grep -E "cmtcs\]" | grep -E "EM it|update" | head -2 | cut -c1-180
CMTCS_PHASE_LOG=1 timeout 120 python bench.py --config 3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline 2>&1 | grep -E "cmtcs\] EM"
timeout 300 python bench.py --no-e2e --no-cpu-baseline 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'): j=json.loads(l); print('C2', round(j['value'],3), j['roofline']['frac'])"
