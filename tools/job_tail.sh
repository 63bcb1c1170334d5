# the split bit-identity test, then C1 / C2 with and without the two-half loops
set -x
mkdir -p gpurun_out/r02d
O=gpurun_out/r02d
timeout 900 python -m pytest tests/test_gpu_fp32_engine.py -m gpu -q -k "halves" > $O/test_split.log 2>&1; echo "split test rc=$?"; tail -3 $O/test_split.log
for c in 1 2; do for sp in 0 1 0 1; do
  echo "C$c SPLIT $sp: $(CMTCS_SIMT_SPLIT=$sp timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python tools/bench_digest.py /dev/stdin | cut -c1-140)" | tee -a $O/ab_split_small.txt
done; done
