#!/bin/bash
# usage: tools/run_variants.sh CONFIG name1 name2 ...
cfg=$1; shift
for n in "$@"; do
  echo "== $n"; FTK_LIB=$PWD/paper_2011_08697_b200/libftk_cp_$n.so timeout 120 python tools/prof_run.py $cfg 3 2>&1 | tail -1
done
