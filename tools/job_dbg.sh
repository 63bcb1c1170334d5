# phase timings at config ${CFG:-3} with parts of the pipeline switched off (CMTCS_DBG bits:
# 1 no DMMA, 2 no tcgen05.mma, 4 no tf32 split, 64 no epilogue, 128 no TMA) — results are wrong,
# the timings show what binds
CFG=${CFG:-3}
for f in ${FLAGS:-0 7 71 135 199 255}; do
  echo "DBG=$f $EXTRA"; env $EXTRA CMTCS_DBG=$f CMTCS_PHASE_LOG=1 timeout 120 python bench.py --config $CFG --steps 1 --warmup 0 --no-e2e --no-cpu-baseline 2>&1 | grep -E "cmtcs\] EM" | head -1 | cut -c1-200
done
