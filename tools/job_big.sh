# C3/C4/C5 bench lines (big configs; outputs under gpurun_out/)
nproc; free -g | head -2
CMTCS_PHASE_LOG=1 timeout 600 python bench.py --config 3 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
CMTCS_PHASE_LOG=1 timeout 900 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"
CMTCS_PHASE_LOG=1 timeout 900 python bench.py --config 5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
for c in 3 4 5; do grep -E "cmtcs\] EM" gpurun_out/bench_c$c.err | cut -c1-200; tail -2 gpurun_out/bench_c$c.err | cut -c1-300; cut -c1-400 gpurun_out/bench_c$c.json; done
