#!/bin/bash
# A/B of the leaf GEMM's epilogue hand-off variants (libspamm_b200_<name>.so built with
# _build.build_variant): C5/C3 k = 8 NS-step GEMM times, interleaved, and the consumer-cycle
# accounting of the default.  usage: tools/ab_epilogue.sh OUT name1 name2 ...  ("" = default)
O=gpurun_out/${1:-ab_epi}; shift
L=paper_1508_05856_b200
mkdir -p $O
for r in 1 2; do
  for v in "$@"; do
    lib=$L/libspamm_b200${v:+_$v}.so
    for c in C5 C3; do
      SPAMM_LIB=$lib timeout 600 python tools/gemm_probe.py --config $c -k 8 --reps 5 > $O/probe_${c}_${v:-default}_$r.txt 2>&1
    done
  done
done
timeout 600 python tools/gemm_clocks.py --config C5 -k 8 > $O/clocks_C5.txt 2>&1
for f in $O/probe_*; do echo "$(basename $f): $(grep 'NS step' $f)"; done
