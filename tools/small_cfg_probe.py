"""Per config and kernel policy: host cost of one call, device time per call
when launched back to back, CUDA-graph replay time, per-kernel event times.

    python tools/small_cfg_probe.py cfg1 cfg3 cfg2
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1404_0424_b200 import Context, get_config  # noqa: E402


def make_call(ctx, cfg):
    out = {}
    if cfg.kind == "downlink":
        Hd, T = ctx.generate_downlink(cfg.B, cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits)
        return lambda: ctx.precode_cg(Hd, T, cfg.rho_d, cfg.K, out=out)
    rs = cfg.rsqrt()
    rs = None if rs is None else torch.tensor(rs)
    H, Y = ctx.generate_uplink(cfg.B, cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits, cfg.n0, rsqrt=rs)
    if cfg.kind == "both":
        T = ctx.generate_symbols(cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits)
        return lambda: ctx.detect_precode_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,
                                             cfg.tracker, T, cfg.rho_d, cfg.K, out=out)
    return lambda: ctx.detect_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K, cfg.tracker,
                                 out=out)


def probe(ctx, cfg, policy):
    ctx.set_kernel_policy(policy)
    call = make_call(ctx, cfg)
    for _ in range(5):
        call()
    torch.cuda.synchronize()
    n = 100
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        call()
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    res = {"cfg": cfg.name, "policy": policy, "host_us": (t1 - t0) / n * 1e6,
           "device_us_back_to_back": e0.elapsed_time(e1) / n * 1e3}
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
        for _ in range(5):
            g.replay()
        e0.record()
        for _ in range(n):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res["graph_us"] = e0.elapsed_time(e1) / n * 1e3
    except Exception as ex:
        res["graph"] = str(ex)[:200]
    ctx.set_profiling(True)
    ctx.kernel_times()
    for _ in range(20):
        call()
    torch.cuda.synchronize()
    k1, k2, nl = ctx.kernel_times()
    ctx.set_profiling(False)
    res.update(k1_us=k1 / 20 * 1e3, k2_us=k2 / 20 * 1e3, launches=nl / 20)
    return res


def main():
    ctx = Context(0)
    policies = os.environ.get("PROBE_POLICIES", "auto,generic").split(",")
    for name in sys.argv[1:]:
        cfg = get_config(name)
        for pol in policies:
            try:
                print(json.dumps(probe(ctx, cfg, pol)), flush=True)
            except Exception as ex:
                print(json.dumps({"cfg": name, "policy": pol, "error": str(ex)[:300]}), flush=True)
    ctx.set_kernel_policy("auto")


if __name__ == "__main__":
    main()
