for c in 2 3; do timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline $( [ $c = 3 ] && echo "--steps 3 --warmup 3") 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'): j=json.loads(l); print('C$c', round(j['value'],4), j['roofline']['frac'])"; done
timeout 300 python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'): j=json.loads(l); print('C4', round(j['value'],4), j['roofline']['frac'], j.get('clocks',{}).get('sm_mhz'))"
