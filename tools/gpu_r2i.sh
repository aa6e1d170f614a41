#!/bin/bash
# round 2, call i: spatially blocked pass-2 hash; full GPU suite, C2 and C4 benches + C4 launch list
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_slabs_gpu.py tests/test_post_gpu.py tests/test_iso_gpu.py tests/test_stream_gpu.py -x -q > gpurun_out/pytest_r2i.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_r2i.log
for cfg in C2 C4; do
  timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-stream > gpurun_out/bench_r2i_$cfg.json 2> gpurun_out/bench_r2i_$cfg.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_r2i_$cfg.json')); r=d['roofline']
print('$cfg', 'ms/step %.4f' % d['ms_per_step'], 'K1a %.4f K1b %.4f extraction %.4f frac %.3f pass2 %.4f' % (r['k_scan2d']['ms'], r['k_exact2d']['ms'], r['ms'], r['frac'], d['config']['pass2_ms']))"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv python bench.py --config C4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-stream > gpurun_out/launches_r2i_c4.csv 2> gpurun_out/launches_r2i_c4.err; echo ncu rc=$?
