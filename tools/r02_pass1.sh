#!/bin/bash
# Round-2 first GPU pass: gpu tests, default bench (cfg5), reference arm, launch list.
set -u
O=gpurun_out/p1
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/bench_ref.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg5.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu > $O/ncu_launch.log 2>&1
echo done
