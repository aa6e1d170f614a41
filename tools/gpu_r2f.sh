#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2f.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2f.log
tail -2 gpurun_out/pytest_r2f.log
bash tools/round_profile.sh r2f C2
python -c "
import json; d=json.load(open('gpurun_out/bench_r2f.json')); r=d['roofline']
print('ms/step %.4f' % d['ms_per_step'], 'K1a %.4f K1b %.4f extraction %.4f frac %.3f pass2 %.4f' % (r['k_scan2d']['ms'], r['k_exact2d']['ms'], r['ms'], r['frac'], d['config']['pass2_ms']))"
