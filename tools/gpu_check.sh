#!/bin/bash
# usage: tools/gpu_check.sh TAG  -- GPU parity tests, C2 timing, launch list (runs on the GPU box)
tag=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_slabs_gpu.py -m gpu -x -q > gpurun_out/t_$tag.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/t_$tag.log
python tools/prof_run.py C2 3 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv python tools/prof_run.py C2 1 > gpurun_out/launch_$tag.csv 2>&1
grep "k_\|Kernel" gpurun_out/launch_$tag.csv | awk -F'","' '{print $5, $(NF)}' | cut -c1-150 | tail -8
if [ -n "$2" ]; then
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$2" -c ${3:-1} -f -o gpurun_out/full_$tag python tools/prof_run.py C2 1 > gpurun_out/ncu_$tag.log 2>&1
  tail -1 gpurun_out/ncu_$tag.log
fi
