"""Host-side cost of one hot-path call (Python wrapper -> C ABI -> launches),
versus the device time of its kernels: python tools/host_overhead.py [cfg]"""
import json
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.join(__import__("os").path.dirname(__file__), ".."))
from paper_1404_0424_b200 import Context, get_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = get_config(name)
ctx = Context(0)
H, Y = ctx.generate_uplink(cfg.B, cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits, cfg.n0)
out = {}
call = lambda: ctx.detect_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K, cfg.tracker, out=out)
for _ in range(5):
    call()
torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
for _ in range(n):
    call()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
# raw C ABI cost: same call with the Python wrapper's work hoisted
lib, h = ctx.lib, ctx.h
print(json.dumps({"cfg": name, "host_us_per_call": (t1 - t0) / n * 1e6,
                  "wall_us_per_call_incl_drain": (t2 - t0) / n * 1e6}))

# CUDA-graph replay of the same call: device time without host submission gaps
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        call()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
try:
    with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
        call()
    ok = True
except Exception as e:  # report why capture is not possible
    ok = False
    print(json.dumps({"graph_capture": "failed", "why": str(e)[:300]}))
if ok:
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        g.replay()
    e0.record()
    for _ in range(n):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"graph_replay_us_per_call": e0.elapsed_time(e1) / n * 1e3}))
