# ncu --set full of the persistent CG kernel (one EM iteration after warm-up); CFG/WARM from env
CFG=${CFG:-2}; WARM=${WARM:-2}
python tools/profile_step.py --config $CFG --warmup $WARM > gpurun_out/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_cg_persistent -s $WARM -c 1 \
    -o gpurun_out/prof_c$CFG python tools/profile_step.py --config $CFG --warmup $WARM > gpurun_out/ncu.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu.log
