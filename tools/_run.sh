ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C5.csv python bench.py --steps 1 --warmup 1 > gpurun_out/launches_C5_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_leaf_gemm -s 24 -c 3 -o gpurun_out/gemm_C5_k8 python tools/diag_ns.py --config C5 --iters 9 --tau-s 1e-9 > gpurun_out/diag_C5_k8.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_leaf_gemm -s 24 -c 3 -o gpurun_out/gemm_C3_k8 python tools/diag_ns.py --config C3 --iters 9 > gpurun_out/diag_C3_k8.log 2>&1
