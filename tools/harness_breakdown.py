import sys, time, torch
sys.path.insert(0, '.')
from paper_1404_0424_b200 import Context, sim
ctx = Context(0)
args = (128, 32, 6, 4, "approx", 15.0)
sim.uplink_sweep_point(ctx, *args, 8, 1200, 1)
ctx.set_profiling(True); ctx.kernel_times()
for rep in range(3):
    t0 = time.perf_counter()
    keys = sim.trial_keys(1, rep, 64)
    ctx.uplink_trials(128, 32, 1200, 6, 4, "approx", 15.0, keys)
    dt = time.perf_counter() - t0
    k1, k2, n = ctx.kernel_times()
    print(f"64 trials: wall {dt*1e3:.1f} ms, channel {k1:.2f} ms, solve {k2:.2f} ms, launches {n}", flush=True)
