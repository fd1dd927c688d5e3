# channel-kernel warp split sweep on the exact configs (A/B for the default choice)
for c in cfg4a_K2 cfg5; do for w in "8,0" "8,8" "4,8" "16,0"; do
 echo "$c warps=$w $(CGMIMO_TC_WARPS=$w PROBE_POLICIES=auto python tools/small_cfg_probe.py $c 2>&1 | head -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["device_us_back_to_back"],1))')"
done; done
