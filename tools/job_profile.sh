# Round evidence: bench lines (C2 default with all legs; C3/C4/C5), the ncu launch list of one C2 EM
# iteration, and ncu --set full captures of the persistent CG kernel at C2 and C3.  Outputs in gpurun_out/.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench c2 rc=$?"
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench c3 rc=$?"
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err; echo "ref rc=$?"
# launch list (plain run first, then ncu)
python tools/profile_step.py --config 2 --warmup 3 > gpurun_out/plain_c2.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python tools/profile_step.py --config 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
python tools/profile_step.py --config 3 --warmup 1 > gpurun_out/plain_c3.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_cg_persistent -s 3 -c 1 \
    -o gpurun_out/prof_c2 python tools/profile_step.py --config 2 --warmup 3 > gpurun_out/ncu_c2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_cg_persistent -s 1 -c 1 \
    -o gpurun_out/prof_c3 python tools/profile_step.py --config 3 --warmup 1 > gpurun_out/ncu_c3.log 2>&1; echo "ncu rc=$?"
timeout 900 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 rc=$?"
timeout 900 python bench.py --config 5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"
cut -c1-300 gpurun_out/bench_c*.json gpurun_out/bench_ref_c2.json
