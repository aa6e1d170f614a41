#!/bin/bash
# usage: tools/var_time.sh CONFIG name...  -- K1/pass-2 timing of variant libraries + k_scan/k_exact split
cfg=$1; shift
for n in "$@"; do
  echo "== $n"
  FTK_LIB=$PWD/paper_2011_08697_b200/libftk_cp_$n.so timeout 120 python tools/prof_run.py $cfg 3 2>&1 | tail -1
  FTK_LIB=$PWD/paper_2011_08697_b200/libftk_cp_$n.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_scan2d|k_exact2d|k_scan3d|k_exact3d" --csv python tools/prof_run.py $cfg 1 2>/dev/null | grep "k_" | awk -F'","' '{print $5, $(NF)}' | cut -c1-90 | tail -2
done
