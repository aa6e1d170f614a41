#!/bin/bash
# usage: tools/round_profile.sh TAG [CONFIG]  -- on the GPU box: bench line, launch list of the same
# bench command, one ncu --set full capture of K1a + K1b (each after the plain command exited 0)
tag=$1; cfg=${2:-C2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/box_$tag.txt 2>&1
python bench.py --config $cfg --steps 100 --warmup 5 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
rc=$?; echo "bench rc=$rc"; tail -c 600 gpurun_out/bench_$tag.json
if [ $rc -eq 0 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
    python bench.py --config $cfg --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_$tag.csv 2> gpurun_out/launches_$tag.err
  echo "launch list rc=$?"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_scan2d|k_exact2d|k_scan3d|k_exact3d" -c 2 -f \
    -o gpurun_out/full_$tag python tools/prof_run.py $cfg 1 > gpurun_out/ncu_full_$tag.log 2>&1
  echo "ncu full rc=$?"
fi
