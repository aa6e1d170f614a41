#!/bin/bash
# round 2, call g: 3D scan pipelining; 3D tests + C5/C3 bench
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_slabs_gpu.py tests/test_stream_gpu.py tests/test_fullsize_gpu.py tests/test_config_labels_gpu.py tests/test_sorted_gpu.py -x -q -k "3d or C5 or c5 or c3 or moving or degenerate or slab" > gpurun_out/pytest_r2g.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_r2g.log
for cfg in C5 C3; do
  timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-stream > gpurun_out/bench_r2g_$cfg.json 2> gpurun_out/bench_r2g_$cfg.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_r2g_$cfg.json')); r=d['roofline']
print('$cfg', 'ms/step %.4f' % d['ms_per_step'], 'K1a %.4f K1b %.4f extraction %.4f frac %.3f scan frac %.3f pass2 %.4f' % (r['k_scan3d']['ms'], r['k_exact3d']['ms'], r['ms'], r['frac'], r['k_scan3d']['frac'], d['config']['pass2_ms']))"
done
