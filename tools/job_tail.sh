# the split bit-identity test, then the small-config bench lines (C1, C2, C6) on the final code
set -x
mkdir -p gpurun_out/r02d
O=gpurun_out/r02d
timeout 900 python -m pytest tests/test_gpu_fp32_engine.py -m gpu -q -k "halves" > $O/test_split.log 2>&1; echo "split test rc=$?"; tail -5 $O/test_split.log
for c in 1 2 6; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 > $O/bench_c${c}_fp32.json 2> $O/bench_c${c}_fp32.err; echo "c$c rc=$?"
done
python tools/bench_digest.py $O/bench_c1_fp32.json $O/bench_c2_fp32.json $O/bench_c6_fp32.json | cut -c1-400
