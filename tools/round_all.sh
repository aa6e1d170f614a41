#!/bin/bash
# usage: tools/round_all.sh TAG -- GPU box: bench lines + launch lists + full captures for C2, C5; bench lines C3, C4
tag=$1
tools/round_profile.sh ${tag} C2
tools/round_profile.sh ${tag}_c5 C5
for c in C3 C4; do
  python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_${tag}_$(echo $c | tr C c).json 2> gpurun_out/bench_${tag}_$c.err
  echo "bench $c rc=$?"
done
