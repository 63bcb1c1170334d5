# A/B of the update CTA width (CMTCS_SIMT_UPDW) and the two-half CG loops (CMTCS_SIMT_SPLIT) at C4
# (32 tasks) and C3, then the whole GPU suite on the defaults.
set -x
mkdir -p gpurun_out
for rep in 1 2; do for cfg in "8 1" "4 1" "4 0"; do set -- $cfg
  echo "C4/32 UPDW $1 SPLIT $2 rep $rep: $(CMTCS_SIMT_UPDW=$1 CMTCS_SIMT_SPLIT=$2 timeout 300 python tools/profile_step.py --config 4 --tasks 32 --engine fp32 --warmup 1 --steps 2 2>&1 | tail -1 | cut -c1-100)" | tee -a gpurun_out/split_ab.txt
done; done
for cfg in "8 1" "4 1" "4 0"; do set -- $cfg
  echo "C3 UPDW $1 SPLIT $2: $(CMTCS_SIMT_UPDW=$1 CMTCS_SIMT_SPLIT=$2 timeout 300 python tools/profile_step.py --config 3 --engine fp32 --warmup 2 --steps 2 2>&1 | tail -1 | cut -c1-100)" | tee -a gpurun_out/split_ab.txt
done
(time timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/gpu_tests_split.log 2>&1; echo "tests rc=$?"
tail -8 gpurun_out/gpu_tests_split.log
