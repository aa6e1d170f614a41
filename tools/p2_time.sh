#!/bin/bash
# usage: tools/p2_time.sh CONFIG name...  -- pass-2 kernel times of variant libraries
cfg=$1; shift
for n in "$@"; do
  echo "== $n"
  FTK_LIB=$PWD/paper_2011_08697_b200/libftk_cp_$n.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_clear|k_hash|k_edges|k_label" --csv python tools/prof_run.py $cfg 1 2>/dev/null | grep "k_" | awk -F'","' '{print $5, $(NF)}' | cut -c1-70 | tail -4
done
