#!/bin/bash
# compute-sanitizer passes over tools/sanitize_case.py: memcheck on the
# C1/C2 case, racecheck and synccheck on the quick case; summaries to gpurun_out/.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --leak-check no python tools/sanitize_case.py \
    > gpurun_out/san_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck.log
timeout 1500 $CS --tool racecheck --racecheck-report analysis python tools/sanitize_case.py --quick \
    > gpurun_out/san_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_racecheck.log
timeout 1500 $CS --tool synccheck python tools/sanitize_case.py --quick \
    > gpurun_out/san_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_synccheck.log
