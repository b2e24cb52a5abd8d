#!/bin/bash
# Repeatability of the round-2 bench lines (one gpurun call): the default bench (C5) three times
# back to back, C3 / C2 / C1 twice each, then the ncu launch list of one C2 run (per-kernel share
# of a latency-bound step). Outputs under gpurun_out/${1:-repeat}/.
O=gpurun_out/${1:-repeat}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/box.txt 2>&1
for r in 1 2 3; do
  timeout 900 python bench.py > $O/bench_C5_rep$r.json 2> $O/bench_C5_rep$r.err
done
for r in 1 2; do
  timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_C3_rep$r.json 2> /dev/null
  for c in C1 C2; do
    timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_${c}_rep$r.json 2> /dev/null
  done
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2.csv python tools/ns_once.py C2 > $O/ncu_launches_C2.log 2>&1
for f in $O/bench_*.json; do
  echo "$(basename $f): $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d.get('e2e', {}).get('value'), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1)"
done | tee $O/summary.txt
