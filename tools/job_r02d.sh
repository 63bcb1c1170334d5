# Round-2 final evidence (profiles/r02d): C4 bench line (default command), reference arm, ncu launch
# list of C4 EM iteration 0 and ncu --set full of one k_simt_probe4<1> / <2> launch (whole-problem
# launches: CMTCS_SIMT_SPLIT=0 for that capture only), C3 / C5 lines.
set -x
mkdir -p gpurun_out/r02d
O=gpurun_out/r02d
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python bench.py > $O/bench_c4_fp32.json 2> $O/bench_c4_fp32.err; echo "bench rc=$?"
cut -c1-400 $O/bench_c4_fp32.json
timeout 900 python bench.py --impl reference > $O/bench_reference_c4.json 2> $O/bench_reference_c4.err; echo "ref rc=$?"
python tools/profile_step.py --config 4 --warmup 0 --engine fp32 > $O/plain_c4.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4_fp32.csv \
    python tools/profile_step.py --config 4 --warmup 0 --engine fp32 > $O/ncu_launch.log 2>&1; echo "launch rc=$?"
python tools/launches.py $O/launches_c4_fp32.csv > $O/launches_c4_fp32.txt; head -8 $O/launches_c4_fp32.txt
CMTCS_SIMT_SPLIT=0 ncu --set full --clock-control none --import-source on -k regex:k_simt_probe4 -s 4 -c 2 \
    -o $O/prof_c4_fp32 python tools/profile_step.py --config 4 --warmup 0 --engine fp32 > $O/ncu_full.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py $O/prof_c4_fp32.ncu-rep > $O/ncu_full_c4_fp32.json; head -c 1500 $O/ncu_full_c4_fp32.json
ncu -i $O/prof_c4_fp32.ncu-rep --page raw --csv > $O/ncu_full_c4_fp32_raw.csv 2>/dev/null
rm -f $O/prof_c4_fp32.ncu-rep.tmp; ls -la $O
timeout 900 python bench.py --config 3 --steps 10 --warmup 5 > $O/bench_c3_fp32.json 2> $O/bench_c3_fp32.err; echo "c3 rc=$?"
timeout 1500 python bench.py --config 5 --steps 2 --warmup 3 --no-e2e > $O/bench_c5_fp32.json 2> $O/bench_c5_fp32.err; echo "c5 rc=$?"
cut -c1-300 $O/bench_c3_fp32.json $O/bench_c5_fp32.json
(time timeout 1500 python -m pytest tests -m gpu -x -q) > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -4 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
