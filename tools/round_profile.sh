#!/bin/bash
# Round-end measurement pass (run under gpurun): bench lines for every config,
# the reference arm on the headline, the ncu launch list of the headline bench
# command, and one `ncu --set full` capture per dominant kernel.
set -u
O=gpurun_out/round
mkdir -p $O
python bench.py > $O/bench_cfg2.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_cfg2.log 2>&1
: > $O/bench_others.jsonl
for c in cfg1 cfg3 cfg4a_K2 cfg4a_K4 cfg4a_K8 cfg4b_K2 cfg4b_K4 cfg4b_K8 cfg5; do
  python bench.py --config $c --no-cpu --steps 5 --warmup 3 2>/dev/null | tail -1 >> $O/bench_others.jsonl
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launch.log 2>&1
for spec in "cfg2 channel_tc" "cfg2 solve_rows32_pairs" "cfg1 uplink_small" "cfg3 precode_small" "cfg4a_K8 basis_kernel" "cfg4a_K8 solve_rows32_exact" "cfg5 solve_rows32_kernel"; do
  set -- $spec
  ncu --set full --import-source on --clock-control none -k regex:$2 --launch-skip 3 --launch-count 1 \
      -o $O/full_$1_$2 -f python tools/quick_time.py $1 > /dev/null 2>&1
done
ls $O
# summaries (the .ncu-rep files are too large to bring back together)
for r in $O/full_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  python tools/ncu_lines.py $r 40 > $b.lines.txt 2>&1
  BY_INST=1 python tools/ncu_lines.py $r 40 > $b.lines_by_inst.txt 2>&1
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
done
mkdir -p $O/keep
mv $O/full_cfg2_channel_tc.ncu-rep $O/full_cfg2_solve_rows32_pairs.ncu-rep $O/keep/ 2>/dev/null
rm -f $O/*.ncu-rep
du -sh $O
