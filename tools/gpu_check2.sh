mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r1f.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_r1f.log
timeout 600 python bench.py > gpurun_out/bench_default_r1f.json 2> gpurun_out/bench_default_r1f.err; echo "bench default rc=$?"
for v in base s3sp2; do for c in C5 C3; do
  lib=paper_2011_08697_b200/libftk_cp.so; [ $v = base ] || lib=paper_2011_08697_b200/libftk_cp_$v.so
  echo "== $v $c"; FTK_LIB=$PWD/$lib timeout 200 python tools/prof_run.py $c 6 2>&1 | tail -3
done; done
