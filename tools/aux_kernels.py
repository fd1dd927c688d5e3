"""One call of each auxiliary path for profiling:
a 64-trial coded uplink batch at the cfg2 array (frames, channel, detection,
deinterleave, Viterbi) and the three other detectors on the cfg2 shape.
    python tools/aux_kernels.py [harness|alt|all]
Under ncu: ncu --metrics gpu__time_duration.sum python tools/aux_kernels.py"""
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.join(__import__("os").path.dirname(__file__), ".."))
from paper_1404_0424_b200 import Context, get_config, sim  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
ctx = Context(0)
if what in ("harness", "all"):
    keys = sim.trial_keys(1, 0, 64)
    ctx.uplink_trials(128, 32, 1200, 6, 4, "approx", 15.0, keys[:8])  # warm-up / pool
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e, b = ctx.uplink_trials(128, 32, 1200, 6, 4, "approx", 15.0, keys)
    print(f"harness 64 trials: {1e3 * (time.perf_counter() - t0):.2f} ms, block errors {int(e.sum())}")
if what in ("alt", "all"):
    cfg = get_config("cfg2")
    H, Y = ctx.generate_uplink(cfg.B, cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits, cfg.n0)
    for m, K in (("cholesky", 1), ("cgls", 4), ("neumann", 3)):
        ctx.detect(m, H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, K)
        torch.cuda.synchronize()
        ctx.set_profiling(True)
        ctx.kernel_times()
        for _ in range(5):
            ctx.detect(m, H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, K)
        _, ms, n = ctx.kernel_times()
        ctx.set_profiling(False)
        print(f"{m} K={K} cfg2 ({cfg.n_sc} sc x {cfg.S}): {1e3 * ms / 5:.1f} us per call")
