#!/bin/bash
# usage: tools/gpu_var.sh CONFIG "pytest -k expr" name... -- GPU box: a parity subset on the default
# library, then K1 timings + launch split of each variant library (libftk_cp_<name>.so; "cur" = default)
cd "$GRAFT_REPO_ROOT" || exit 1
cfg=$1; kexpr=$2; shift 2
cp paper_2011_08697_b200/libftk_cp.so paper_2011_08697_b200/libftk_cp_cur.so
if [ -n "$kexpr" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$kexpr" 2>&1 | tail -3
fi
bash tools/var_time.sh $cfg "$@"
