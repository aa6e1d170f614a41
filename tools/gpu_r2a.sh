#!/bin/bash
# round 2, call a: config-scale label parity + compute-sanitizer logs
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/box_r2a.txt
nproc >> gpurun_out/box_r2a.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize.py > gpurun_out/san_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/san_${tool}.log
done
timeout 1500 python -m pytest tests/test_config_labels_gpu.py -x -q -rA --durations=0 > gpurun_out/pytest_labels_r2a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_labels_r2a.log
