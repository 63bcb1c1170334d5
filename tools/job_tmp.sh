for pr in 1 0; do echo "PAIR=$pr"
CMTCS_PAIR=$pr timeout 300 python bench.py --no-e2e --no-cpu-baseline 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'): j=json.loads(l); print('C2', round(j['value'],3), j['roofline']['frac'])"
CMTCS_PAIR=$pr timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'): j=json.loads(l); print('C3', round(j['value'],3), j['roofline']['frac'])"
done
