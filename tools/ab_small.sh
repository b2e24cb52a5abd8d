#!/bin/bash
# A/B of library variants on the latency-bound configs (bench C1/C2 ms per run) and the
# C5/C3 k = 8 NS-step GEMM; output hashes per variant.  usage: tools/ab_small.sh OUT name1 ...
O=gpurun_out/${1:-ab_small}; shift
L=paper_1508_05856_b200
mkdir -p $O
for v in "$@"; do
  lib=$L/libspamm_b200${v:+_$v}.so
  SPAMM_LIB=$lib timeout 300 python tools/stress_determinism.py 2 0 > $O/hash_${v:-default}.txt 2>&1
done
for r in 1 2; do
  for v in "$@"; do
    lib=$L/libspamm_b200${v:+_$v}.so
    for c in C1 C2; do
      SPAMM_LIB=$lib timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_${c}_${v:-default}_$r.json 2> /dev/null
    done
    for c in C5 C3; do
      SPAMM_LIB=$lib timeout 600 python tools/gemm_probe.py --config $c -k 8 --reps 5 > $O/probe_${c}_${v:-default}_$r.txt 2>&1
    done
  done
done
for f in $O/hash_*; do echo "$(basename $f): $(cat $f | tr '\n' ' ')"; done
for f in $O/bench_*; do echo "$(basename $f): $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['ms_per_step'], d.get('phase_ms_per_step'))" 2>&1 | tail -1)"; done
for f in $O/probe_*; do echo "$(basename $f): $(grep 'NS step' $f)"; done
