set -u
O=gpurun_out/prof1
mkdir -p $O
python tools/run_config.py --config cfg5 --n-sc 4096 --launches 2 > $O/run.log 2>&1 || { cat $O/run.log; exit 1; }
for k in solve_rows32_kernel moments_kernel channel_tc; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 6 --launch-count 1 \
      -o $O/full_cfg5_$k -f python tools/run_config.py --config cfg5 --n-sc 4096 --launches 2 > $O/ncu_$k.log 2>&1
  ncu -i $O/full_cfg5_$k.ncu-rep --page raw --csv > $O/full_cfg5_$k.raw.csv 2>/dev/null
  python tools/ncu_lines.py $O/full_cfg5_$k.ncu-rep 40 > $O/full_cfg5_$k.lines.txt 2>&1
  ncu -i $O/full_cfg5_$k.ncu-rep --page details --csv > $O/full_cfg5_$k.details.csv 2>/dev/null
done
rm -f $O/*.ncu-rep
ls -la $O
