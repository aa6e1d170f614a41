#!/bin/bash
# usage: tools/round_final.sh TAG [CONFIG...] -- GPU box: for each of C2, C5, V2, V5 (or the configs
# given) a bench line, the launch list of the same bench command and one ncu --set full capture of the
# scan + exact kernels (each after its plain command exited 0); C3 / C4 / ref: bench lines only
tag=$1; shift
cfgs=${@:-C2 C5 V2 V5 C3 C4 ref}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/box_$tag.txt 2>&1
for cfg in $cfgs; do
  t=${tag}_$(echo $cfg | tr C c | tr V v)
  case $cfg in
    ref)
      timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err
      echo "reference rc=$?"; continue;;
    C3|C4)
      timeout 1200 python bench.py --config $cfg --steps 20 --warmup 3 > gpurun_out/bench_$t.json 2> gpurun_out/bench_$t.err
      echo "bench $cfg rc=$?"; continue;;
    C2) re="k_scan2d|k_exact2d";; C5) re="k_scan3d|k_exact3d";;
    V2) re="k_scanvec2d|k_exactvec2d";; V5) re="k_scanvec3d|k_exact3d";;
  esac
  steps=100; [ $cfg = C2 ] || steps=30
  timeout 1200 python bench.py --config $cfg --steps $steps --warmup 5 > gpurun_out/bench_$t.json 2> gpurun_out/bench_$t.err
  rc=$?; echo "bench $cfg rc=$rc"
  if [ $rc -eq 0 ]; then
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
      python bench.py --config $cfg --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_$t.csv 2> gpurun_out/launches_$t.err
    echo "launch list $cfg rc=$?"
    timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$re" -c 2 -f \
      -o gpurun_out/full_$t python tools/prof_run.py $cfg 1 > gpurun_out/ncu_full_$t.log 2>&1
    echo "ncu full $cfg rc=$?"
  fi
done
