python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_kat.py tests/test_gpu_golden.py -x -q 2>&1 | tail -3
python tools/quick_time.py cfg5 cfg4a_K2 cfg4a_K8 cfg4b_K2 cfg4b_K8 2>&1
bash tools/prof_one.sh cfg5 4096 moments cfg5_moments2
bash tools/prof_one.sh cfg5 4096 precode_q cfg5_precode_q3
