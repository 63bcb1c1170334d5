# A/B: the same bench lines for HEAD (.ab_old/) and the working tree, interleaved.
line() { python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'): j=json.loads(l); r=j['roofline']; print('$1 C$2', round(j['value'],4), round(r['frac'],4), j['ms_per_step'])"; }
for rep in 1 2; do
for c in 1 2 3 4; do
  case $c in 1|2) a="--steps 10 --warmup 5";; 3) a="--steps 3 --warmup 3";; 4) a="--steps 1 --warmup 1";; esac
  (cd .ab_old && timeout 300 python bench.py --config $c $a --no-e2e --no-cpu-baseline 2>&1 | line old $c)
  timeout 300 python bench.py --config $c $a --no-e2e --no-cpu-baseline 2>&1 | line new $c
done; done
