#!/bin/bash
# usage: tools/checks_run.sh TAG -- GPU box: the full GPU suite on the default build, then the suite and
# the sanitizer cases (tools/sanitize.py) on the FTK_CHECKS build (device bounds and protocol assertions;
# compute-sanitizer is not available on this pool).  Build the checks library first:
#   python tools/variants.py checks
tag=${1:-checks}
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$tag.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log; tail -2 gpurun_out/pytest_$tag.log
FTK_LIB=$PWD/paper_2011_08697_b200/libftk_cp_checks.so timeout 1500 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/pytest_checks_$tag.log 2>&1
echo "checks pytest rc=$?" >> gpurun_out/pytest_checks_$tag.log; tail -2 gpurun_out/pytest_checks_$tag.log
FTK_LIB=$PWD/paper_2011_08697_b200/libftk_cp_checks.so timeout 600 python tools/sanitize.py > gpurun_out/checks_cases_$tag.log 2>&1
echo "cases rc=$?" >> gpurun_out/checks_cases_$tag.log; tail -3 gpurun_out/checks_cases_$tag.log
