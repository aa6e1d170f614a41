#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=$PWD/paper_2011_08697_b200
for v in default s3rw4 s3rw4b; do
  lib=$L/libftk_cp.so; [ $v != default ] && lib=$L/libftk_cp_$v.so
  FTK_LIB=$lib timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_slabs_gpu.py -x -q -k "3d or moving or degenerate" 2>&1 | tail -1
  for cfg in C5 C3; do
    FTK_LIB=$lib timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-stream > gpurun_out/bench_r2l_${v}_$cfg.json 2> gpurun_out/bench_r2l_${v}_$cfg.err
    python -c "
import json; d=json.load(open('gpurun_out/bench_r2l_${v}_$cfg.json')); r=d['roofline']
print('$v $cfg', 'ms/step %.4f' % d['ms_per_step'], 'K1a %.4f K1b %.4f scan frac %.3f' % (r['k_scan3d']['ms'], r['k_exact3d']['ms'], r['k_scan3d']['frac']))"
  done
done
