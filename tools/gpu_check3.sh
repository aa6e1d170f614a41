# pass-2 label experiment: K6 after FTK_LABEL_JUMP pointer-jumping passes (variants jump2, jump4)
for v in base jump2 jump4; do for c in C2 C4 C5; do
  lib=paper_2011_08697_b200/libftk_cp.so; [ $v = base ] || lib=paper_2011_08697_b200/libftk_cp_$v.so
  echo "== $v $c"; FTK_LIB=$PWD/$lib timeout 300 python tools/prof_run.py $c 5 2>&1 | tail -2
done; done
FTK_LIB=$PWD/paper_2011_08697_b200/libftk_cp_jump4.so timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_slabs_gpu.py -x -q 2>&1 | tail -2
