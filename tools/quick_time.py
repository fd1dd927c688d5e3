"""Device time of one hot-path call per config (inputs resident on the GPU): python tools/quick_time.py cfg2 cfg5 ..."""
import sys, time, json
import torch, numpy as np
sys.path.insert(0, __import__('os').path.join(__import__('os').path.dirname(__file__), '..'))
from paper_1404_0424_b200 import Context, get_config
ctx = Context(0)
import os as _os
if _os.environ.get('POLICY'):
    ctx.set_kernel_policy(_os.environ['POLICY'])
def timeit(fn, reps=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
for name in sys.argv[1:]:
    # name or name:n_sc (e.g. cfg1:16384 -- 16 frames of cfg1 in one call)
    cfg = get_config(name.split(":")[0])
    if ":" in name:
        cfg = cfg.scaled(int(name.split(":")[1]))
    rs = cfg.rsqrt(); rs = None if rs is None else torch.tensor(rs)
    t0 = time.time()
    if cfg.kind == "downlink":
        Hd, T = ctx.generate_downlink(cfg.B, cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits)
        out = {}
        fn = lambda: ctx.precode_cg(Hd, T, cfg.rho_d, cfg.K, out=out)
    else:
        H, Y = ctx.generate_uplink(cfg.B, cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits, cfg.n0, rsqrt=rs)
        out = {}
        if cfg.kind == "both":
            T = ctx.generate_symbols(cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits)
            fn = lambda: ctx.detect_precode_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K, cfg.tracker, T, cfg.rho_d, cfg.K, out=out)
        else:
            fn = lambda: ctx.detect_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K, cfg.tracker, out=out)
    torch.cuda.synchronize()
    fn(); torch.cuda.synchronize()
    ms = timeit(fn, reps=5 if cfg.n_sc > 10000 else 20)
    print(json.dumps(dict(cfg=name, ms=round(ms, 4), vec_per_s=cfg.vectors/ms*1e3, gen_s=round(time.time()-t0, 2))), flush=True)
    # per-kernel split (CUDA events around each launch on the launch stream)
    ctx.set_profiling(True)
    ctx.kernel_times()
    reps = 5 if cfg.n_sc > 10000 else 20
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    k1, k2, n = ctx.kernel_times()
    ctx.set_profiling(False)
    print(json.dumps(dict(cfg=name, channel_ms=round(k1 / reps, 4), solve_ms=round(k2 / reps, 4),
                          launches_per_call=n / reps)), flush=True)
