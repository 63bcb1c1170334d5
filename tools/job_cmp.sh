# bench C2/C3/C4 (device value only) for A/B comparison of kernel changes
for c in 2 3; do timeout 200 python bench.py --config $c --no-e2e --no-cpu-baseline 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'): j=json.loads(l); print('C$c', round(j['value'],3), j['roofline']['frac'])"; done
timeout 300 python bench.py --config 4 --no-e2e --no-cpu-baseline 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'): j=json.loads(l); print('C4', round(j['value'],4), j['roofline']['frac'])"
