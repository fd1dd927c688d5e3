python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py -x -q -k "cfg5" 2>&1 | tail -2
python tools/quick_time.py cfg5 2>&1
bash tools/prof_one.sh cfg5 4096 precode_q cfg5_precode_q4
bash tools/prof_one.sh cfg5 4096 block32 cfg5_block32e
