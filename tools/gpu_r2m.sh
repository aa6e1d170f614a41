#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=$PWD/paper_2011_08697_b200
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_slabs_gpu.py tests/test_vector_gpu.py tests/test_stream_gpu.py tests/test_config_labels_gpu.py -x -q -k "3d or moving or degenerate or c5 or c3 or abc or vector or verif" 2>&1 | tail -1
for v in default x3m6 x3m4; do
  lib=$L/libftk_cp.so; [ $v != default ] && lib=$L/libftk_cp_$v.so
  for cfg in C5 C3 V5; do
    FTK_LIB=$lib timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-stream > gpurun_out/bench_r2m_${v}_$cfg.json 2> gpurun_out/bench_r2m_${v}_$cfg.err
    python -c "
import json; d=json.load(open('gpurun_out/bench_r2m_${v}_$cfg.json')); r=d['roofline']; k=[x for x in r if x.startswith('k_scan')][0]
print('$v $cfg', 'ms/step %.4f' % d['ms_per_step'], 'K1a %.4f K1b %.4f pass2 %.4f frac %.3f' % (r[k]['ms'], r['k_exact3d']['ms'], d['config']['pass2_ms'], r['frac']))"
  done
done
