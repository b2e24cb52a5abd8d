python tools/gemm_probe.py --config C3
python tools/gemm_probe.py --config C5
python tools/gemm_probe.py --dense 8192 --reps 3
