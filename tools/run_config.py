"""Minimal driver for profiling: generate one config's inputs on cuda:0 and
launch the fused kernel `--launches` times (no host work in between).

    python tools/run_config.py --config cfg2 --launches 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1404_0424_b200 import Context, get_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--launches", type=int, default=3)
    ap.add_argument("--n-sc", type=int, default=None)
    a = ap.parse_args()
    cfg = get_config(a.config)
    if a.n_sc:
        cfg = cfg.scaled(a.n_sc)
    ctx = Context(0)
    if os.environ.get('POLICY'):
        ctx.set_kernel_policy(os.environ['POLICY'])
    rs = cfg.rsqrt()
    rs = None if rs is None else torch.tensor(rs)
    if cfg.kind == "downlink":
        Hd, T = ctx.generate_downlink(cfg.B, cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits)
        fn = lambda: ctx.precode_cg(Hd, T, cfg.rho_d, cfg.K, out=out)  # noqa: E731
    else:
        H, Y = ctx.generate_uplink(cfg.B, cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits, cfg.n0,
                                   rsqrt=rs)
        if cfg.kind == "both":
            T = ctx.generate_symbols(cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits)
            fn = lambda: ctx.detect_precode_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits,  # noqa: E731
                                               cfg.K, cfg.tracker, T, cfg.rho_d, cfg.K, out=out)
        else:
            fn = lambda: ctx.detect_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,  # noqa: E731
                                       cfg.tracker, out=out)
    out = {}
    for _ in range(a.launches):
        fn()
    torch.cuda.synchronize()
    print(f"{a.config}: {a.launches} launches ok, {ctx.kernel_launches} kernels")


if __name__ == "__main__":
    main()
