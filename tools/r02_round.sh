#!/bin/bash
# Round-2 measurement pass (run under gpurun): the headline bench (cfg5, with
# cpu_baseline), the reference arm, every other config's bench line, the ncu
# launch list of the headline command and a --set full capture of each cfg5
# kernel (summaries only).
set -u
O=gpurun_out/r02
mkdir -p $O
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $O/nvsmi.csv 2>&1
timeout 900 python bench.py > $O/bench_cfg5.log 2>&1; echo "rc=$?" >> $O/bench_cfg5.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_cfg5.log 2>&1; echo "rc=$?" >> $O/bench_ref_cfg5.log
: > $O/bench_others.jsonl
for c in cfg1 cfg2 cfg3 cfg4a_K2 cfg4a_K4 cfg4a_K8 cfg4b_K2 cfg4b_K4 cfg4b_K8; do
  timeout 600 python bench.py --config $c --no-cpu --steps 20 --warmup 3 2>/dev/null | tail -1 >> $O/bench_others.jsonl
done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg5.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu > $O/ncu_launch.log 2>&1
bash tools/prof_cfg5.sh $O/prof "channel_tc moments_rows32 block32t_kernel precode_q_kernel"
rm -f $O/prof/*.ncu-rep
ls -la $O
