#!/bin/bash
# usage: tools/gpu_prof.sh TAG CONFIG KERNEL_REGEX -- on the GPU box: timings of the config, then one
# ncu --set full capture (source-correlated) of the named kernels
tag=$1; cfg=$2; kre=$3
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python tools/prof_run.py $cfg 3 2>&1 | tail -3
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$kre" -c 1 -f \
  -o gpurun_out/full_${tag}_$cfg python tools/prof_run.py $cfg 1 > gpurun_out/ncu_full_${tag}_$cfg.log 2>&1
echo "ncu rc=$?"
