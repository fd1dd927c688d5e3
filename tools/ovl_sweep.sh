for w in "8,8" "8,0"; do for o in 1 2 3 4 6; do
 echo "warps=$w overlap=$o $(CGMIMO_TC_WARPS=$w CGMIMO_OVERLAP_CHUNKS=$o PROBE_POLICIES=auto python tools/small_cfg_probe.py cfg2 2>&1 | head -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["device_us_back_to_back"],1), round(d["graph_us"],1))')"
done; done
