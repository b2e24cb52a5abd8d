#!/bin/bash
# Round-2 evidence run (one gpurun call): full GPU test suite, smoke(), bench lines for every
# config, the reference arm, the ncu launch list of the default bench, a --set full capture of
# the three leaf-GEMM launches of C5 iteration 8 and the GEMM consumer-cycle accounting.
# Outputs under gpurun_out/${1:-final}/.
O=gpurun_out/${1:-final}
mkdir -p $O
nvidia-smi -q > $O/nvidia_smi.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
python -m pytest tests -m gpu -q -p no:cacheprovider -s --durations=40 > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
fi
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
if [ -z "$SKIP_TESTS" ]; then
(echo "# SPAMM_LIB=libspamm_b200_debug.so (-DSPAMM_DEBUG device bounds asserts) SPAMM_POISON=1 pytest parity/dist/fullsize"
 SPAMM_LIB=paper_1508_05856_b200/libspamm_b200_debug.so SPAMM_POISON=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider) > $O/gputest_debug_poison.log 2>&1; echo "rc=$?" >> $O/gputest_debug_poison.log
fi
python bench.py --steps 20 --warmup 5 > $O/bench_C5.json 2> $O/bench_C5.err
python bench.py --config C3 --steps 10 --warmup 3 > $O/bench_C3.json 2> $O/bench_C3.err
for c in C1 C2; do python bench.py --config $c --steps 20 --warmup 5 > $O/bench_$c.json 2> $O/bench_$c.err; done
for t in 1e-4 1e-6 1e-8; do python bench.py --config C4 --tau $t --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_C4_$t.json 2> $O/bench_C4_$t.err; done
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
python tools/gemm_clocks.py --config C5 -k 8 > $O/gemm_clocks_C5.txt 2>&1
python tools/gemm_clocks.py --config C3 -k 8 > $O/gemm_clocks_C3.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C5.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_leaf_gemm -s 24 -c 3 -o $O/gemm_C5_k8 python tools/diag_ns.py --config C5 --iters 9 --tau-s 1e-9 > $O/diag_c5_k8.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_leaf_gemm -s 24 -c 3 -o $O/gemm_C3_k8 python tools/diag_ns.py --config C3 --iters 9 > $O/diag_c3_k8.log 2>&1
