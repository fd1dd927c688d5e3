# compute-sanitizer memcheck / racecheck / synccheck over every default
# kernel family on small batches (run under gpurun); summaries -> gpurun_out/san/
set -u
O=gpurun_out/san
mkdir -p $O
for tool in memcheck racecheck synccheck; do
  for spec in "cfg2 64" "cfg4a_K4 64" "cfg4a_K8 32" "cfg4b_K8 16" "cfg5 24" "cfg1 64" "cfg3 64"; do
    set -- $spec
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/run_config.py --config $1 --n-sc $2 --launches 1 > $O/${tool}_$1.log 2>&1
    echo "$tool $1 rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Error' $O/${tool}_$1.log | tail -1)"
  done
done
