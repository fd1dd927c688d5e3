# usage: bash tools/prof_one.sh <config> <n_sc> <kernel-regex> <tag> [POLICY]
set -u
O=gpurun_out/prof
mkdir -p $O
C=$1; N=$2; K=$3; T=$4
export POLICY=${5:-}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K --launch-skip 1 --launch-count 1 \
    -o $O/$T -f python tools/run_config.py --config $C --n-sc $N --launches 3 > $O/$T.ncu.log 2>&1
ncu -i $O/$T.ncu-rep --page raw --csv > $O/$T.raw.csv 2>/dev/null
python tools/ncu_lines.py $O/$T.ncu-rep 45 > $O/$T.lines.txt 2>&1
BY_INST=1 python tools/ncu_lines.py $O/$T.ncu-rep 60 > $O/$T.byinst.txt 2>&1
python tools/ncu_opcodes.py $O/$T.ncu-rep 40 > $O/$T.opcodes.txt 2>&1
ncu -i $O/$T.ncu-rep --page details --csv > $O/$T.details.csv 2>/dev/null
rm -f $O/$T.ncu-rep
