# ncu --set full of the persistent CG kernel (one EM iteration of C2 after 2 warm-up iterations)
python tools/profile_step.py --config 2 --warmup 2 > gpurun_out/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_cg_persistent -s 2 -c 1 \
    -o gpurun_out/prof_c2 python tools/profile_step.py --config 2 --warmup 2 > gpurun_out/ncu.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu.log
