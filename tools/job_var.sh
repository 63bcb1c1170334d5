# A/B of the k_simt_probe4 variants (CMTCS_SIMT_VAR): C4, 32 tasks, EM iterations 1-2 after one warm-up,
# interleaved twice; then the FP32-engine parity tests under the candidate variants.
set -x
mkdir -p gpurun_out
for rep in 1 2; do for v in ${VARS:-0 3 7 14}; do
  echo "VAR $v rep $rep: $(CMTCS_SIMT_VAR=$v timeout 300 python tools/profile_step.py --config 4 --tasks 32 --engine fp32 --warmup 1 --steps 2 2>&1 | tail -1 | cut -c1-120)" | tee -a gpurun_out/var_ab.txt
done; done
for v in ${TESTVARS:-7 14}; do
  CMTCS_SIMT_VAR=$v timeout 900 python -m pytest tests/test_gpu_midrun.py tests/test_gpu_fp32_engine.py tests/test_gpu_fullsize.py -m gpu -q -s -k "fp32 or engine" > gpurun_out/tests_var$v.log 2>&1; echo "tests VAR $v rc=$?"
  grep -E "^\.?c[345]_step" gpurun_out/tests_var$v.log; tail -2 gpurun_out/tests_var$v.log
done
