#!/bin/bash
# usage: tools/quick.sh TAG -- GPU box: 2D/3D parity tests, C2/C4 timings, C2 launch list
tag=${1:-q}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_slabs_gpu.py -m gpu -x -q 2>&1 | tail -2
python tools/prof_run.py C2 5 | tail -2
python tools/prof_run.py C4 2 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv python tools/prof_run.py C2 1 > gpurun_out/launch_$tag.csv 2>&1
python - <<PY
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/launch_$tag.csv')) if len(r)>10]
h=rows[0]; acc=collections.defaultdict(list)
for r in rows[1:]:
    d=dict(zip(h,r)); acc[d['Kernel Name'][:50]].append(float(d['Metric Value'])/1e3)
for k,v in acc.items(): print(f'{k:50s} {sum(v)/len(v):8.1f} us x{len(v)}')
PY
