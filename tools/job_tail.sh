# final check of the size-gated split: split test (forced mode), C2 / C3 quick lines, full GPU suite, smoke
set -x
mkdir -p gpurun_out/r02d
O=gpurun_out/r02d
for c in 2 3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 5 --no-cpu-baseline > $O/bench_c${c}_fp32_final.json 2>/dev/null; echo "c$c rc=$?"
done
python tools/bench_digest.py $O/bench_c2_fp32_final.json $O/bench_c3_fp32_final.json | cut -c1-200
(time timeout 1500 python -m pytest tests -m gpu -x -q) > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -4 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log | cut -c1-200
