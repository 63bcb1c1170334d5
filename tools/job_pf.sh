for pf in 0 2 4 8; do for f in 0 7; do
  echo "PF=$pf DBG=$f"; CMTCS_PF=$pf CMTCS_DBG=$f CMTCS_PHASE_LOG=1 timeout 120 python bench.py --config 3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline 2>&1 | grep -E "cmtcs\] EM" | head -1 | cut -c1-200
done; done
