"""e2e (host-buffer) time of the public API per config, as bench.py's e2e
step: pinned host H/Y in, pinned outputs out.  python tools/e2e_time.py cfg2"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1404_0424_b200 import Context, get_config  # noqa: E402

ctx = Context(0)
for name in sys.argv[1:]:
    cfg = get_config(name)
    pin = lambda t: torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True).numpy()
    if cfg.kind == "downlink":  # precode_cg with host buffers
        Hd, T = ctx.generate_downlink(cfg.B, cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits)
        hHd, hT = pin(Hd), pin(T)
        hHd[...] = Hd.cpu().numpy()
        hT[...] = T.cpu().numpy()
        out = {"q": pin(torch.empty((cfg.n_sc, cfg.S, cfg.B), dtype=torch.complex64)),
               "s": pin(torch.empty((cfg.n_sc, cfg.S, cfg.B), dtype=torch.complex64)),
               "gain": pin(torch.empty((cfg.n_sc, cfg.S))),
               "status": pin(torch.empty((cfg.n_sc, cfg.S), dtype=torch.uint8))}
        call = lambda: ctx.precode_cg(hHd, hT, cfg.rho_d, cfg.K, out=out)
        for _ in range(3):
            call()
        n = 20
        t0 = time.perf_counter()
        for _ in range(n):
            call()
        dt = (time.perf_counter() - t0) / n
        print(json.dumps({"cfg": name, "e2e_ms": round(dt * 1e3, 4), "e2e_vec_per_s": cfg.vectors / dt}),
              flush=True)
        continue
    H, Y = ctx.generate_uplink(cfg.B, cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits, cfg.n0)
    hH, hY = pin(H), pin(Y)
    hH[...] = H.cpu().numpy()
    hY[...] = Y.cpu().numpy()
    S, U, bits = cfg.S, cfg.U, cfg.qam_bits
    out = {"xhat": pin(torch.empty((cfg.n_sc, S, U), dtype=torch.complex64)),
           "mu": pin(torch.empty((cfg.n_sc, S, U))), "rho": pin(torch.empty((cfg.n_sc, S, U))),
           "llr": pin(torch.empty((cfg.n_sc, S, U, bits))),
           "status": pin(torch.empty((cfg.n_sc, S), dtype=torch.uint8))}
    call = lambda: ctx.detect_cg(hH, hY, cfg.rho_u, cfg.n0, cfg.es, bits, cfg.K, cfg.tracker, out=out)
    for _ in range(3):
        call()
    n = 20
    t0 = time.perf_counter()
    for _ in range(n):
        call()
    dt = (time.perf_counter() - t0) / n
    print(json.dumps({"cfg": name, "chunks": os.environ.get("CGMIMO_HOST_CHUNKS", "8"),
                      "e2e_ms": round(dt * 1e3, 4), "e2e_vec_per_s": cfg.vectors / dt}), flush=True)
