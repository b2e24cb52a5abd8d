#!/bin/bash
# A/B of the small-problem cull (single-CTA query) variants: output hashes, C1/C2 bench
# lines (alternating, 2 rounds), the cull GPU tests on the default library, an ncu launch
# list of one C2 run and a --set full capture of one C2 single-CTA cull.
# usage: tools/ab_cull.sh OUT name1 ...   (empty name = the default library)
O=gpurun_out/${1:-ab_cull}; shift
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
  done
done
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > $O/gputest_cull.log 2>&1; echo "rc=$?" >> $O/gputest_cull.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2.csv python tools/ns_once.py C2 > $O/ncu_launches_C2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_cull_small -s 200 -c 1 -o $O/cull_small_C2 python tools/ns_once.py C2 > $O/ncu_cull_C2.log 2>&1
for f in $O/hash_*; do echo "$(basename $f): $(cat $f | tr '\n' ' ')"; done
for f in $O/bench_*; do echo "$(basename $f): $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['ms_per_step'], d.get('phase_ms_per_step'))" 2>&1 | tail -1)"; done
tail -3 $O/gputest_cull.log
