import sys, json, torch
sys.path.insert(0, '.')
from paper_1404_0424_b200 import Context, get_config
ctx = Context(0)
for n in (148, 444, 888, 1200, 2400):
    cfg = get_config("cfg2").scaled(n)
    H, Y = ctx.generate_uplink(cfg.B, cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits, cfg.n0)
    out = {}
    fn = lambda: ctx.detect_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K, cfg.tracker, out=out)
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ctx.set_profiling(True); ctx.kernel_times()
    for _ in range(20): fn()
    k1, k2, l = ctx.kernel_times(); ctx.set_profiling(False)
    print(n, round(k1/20*1e3, 2), round(k2/20*1e3, 2))
