#!/bin/bash
# ncu --set full of every cfg5 hot-path kernel on one 8192-subcarrier chunk
# (the production chunk size); summaries only (raw / details / per-line).
set -u
O=${1:-gpurun_out/prof5}
KS=${2:-"block32_kernel precode_q_kernel moments_kernel channel_tc"}
mkdir -p $O
python tools/run_config.py --config cfg5 --n-sc 8192 --launches 2 > $O/run.log 2>&1 || { cat $O/run.log; exit 1; }
for k in $KS; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 1 --launch-count 1 \
      -o $O/full_cfg5_$k -f python tools/run_config.py --config cfg5 --n-sc 8192 --launches 2 > $O/ncu_$k.log 2>&1
  ncu -i $O/full_cfg5_$k.ncu-rep --page raw --csv > $O/full_cfg5_$k.raw.csv 2>/dev/null
  python tools/ncu_lines.py $O/full_cfg5_$k.ncu-rep 40 > $O/full_cfg5_$k.lines.txt 2>&1
  ncu -i $O/full_cfg5_$k.ncu-rep --page details --csv > $O/full_cfg5_$k.details.csv 2>/dev/null
done
ls -la $O
