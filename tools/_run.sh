python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python bench.py --config C2 > gpurun_out/pdl_C2.json 2>&1
python bench.py --config C1 > gpurun_out/pdl_C1.json 2>&1
python bench.py --config C3 --steps 3 > gpurun_out/pdl_C3.json 2>&1
