# Build the committed HEAD into .ab_old/ (git-ignored, shipped by gpurun) for A/B timing against
# the working tree: tools/job_ab.sh runs the same bench lines in both.
set -e
rm -rf .ab_old && mkdir .ab_old
git archive HEAD | tar -x -C .ab_old
cp -f MEASURED_PEAKS.json .ab_old/ 2>/dev/null || true
python .ab_old/paper_2310_00420_b200/build.py > /dev/null
