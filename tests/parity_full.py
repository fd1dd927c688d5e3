"""Full-configuration parity report -- TEST INFRASTRUCTURE (the checker).

Every instance of cfg1, cfg2 and cfg3, and the first N_BIG subcarriers (all
their vectors) of cfg4a / cfg4b (K = 2, 4, 8) and cfg5, run through the CUDA
path (C ABI, device buffers) and through the unmodified reference
(oracle/_ref: detect::detect_cg detect.cpp:182-237, precode::precode_cg
precode.cpp:56-71) on the same complex64 inputs.  Per config and output:
the worst err/tol, the count outside the north_star tolerance
(|got - want| <= 1e-4 + 1e-3 |want|) and the hard-bit flips where
|LLR_ref| >= 1e-4.

For cfg4a / cfg4b it also states BASELINE configs[3]'s "exact MMSE error
comparison": the error of CG-K against the exact MMSE detector, computed on
the GPU (cgm_detect CHOLESKY, csrc/cgm_alt.cuh) and on the reference
(detect_explicit, detect.cpp:94-126), side by side.

    python tests/parity_full.py [--out profiles/r02_parity.json] [--big 4096]
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

RTOL, ATOL = 1e-3, 1e-4
N_BIG = 4096
THREADS = os.cpu_count() or 8


def _report(got, want):
    got = np.asarray(got)
    want = np.asarray(want)
    err = np.abs(got.astype(np.complex128) - want.astype(np.complex128))
    tol = ATOL + RTOL * np.abs(want)
    return {"n": int(err.size), "outside_tol": int((err > tol).sum()),
            "worst_err_over_tol": float(np.max(err / tol)) if err.size else 0.0}


def _flips(llr_got, llr_want):
    mask = np.abs(llr_want) >= ATOL
    return {"decided": int(mask.sum()),
            "hard_bit_flips": int((((llr_got > 0) != (llr_want > 0)) & mask).sum()),
            "undecided_ref_abs_lt_1e-4": int((~mask).sum())}


def _np(t):
    return t.detach().cpu().numpy()


def _gen(ctx, cfg, n_sc):
    import torch

    rs = cfg.rsqrt()
    rs = None if rs is None else torch.tensor(rs)
    H, Y = ctx.generate_uplink(cfg.B, cfg.U, n_sc, cfg.S, cfg.seed, cfg.qam_bits, cfg.n0, rsqrt=rs)
    return H, Y


def detect_section(ctx, ref, cfg, n_sc):
    import torch

    H, Y = _gen(ctx, cfg, n_sc)
    got = ctx.detect_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K, cfg.tracker)
    torch.cuda.synchronize()
    got = {k: _np(v) for k, v in got.items()}
    Hn, Yn = _np(H), _np(Y)
    t0 = time.perf_counter()
    want = ref.detect(Hn, Yn, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K, cfg.tracker,
                      threads=THREADS)
    sec = {"subcarriers": n_sc, "of": cfg.n_sc, "vectors": n_sc * cfg.S,
           "status_equal": bool((got["status"] == want["status"]).all()),
           "reference_seconds": time.perf_counter() - t0}
    for k in ("xhat", "mu", "rho", "llr"):
        sec[k] = _report(got[k], want[k])
    sec["llr"].update(_flips(got["llr"], want["llr"]))
    return sec, (H, Y, got, want)


def precode_section(ctx, ref, cfg, n_sc):
    import torch

    Hd, T = ctx.generate_downlink(cfg.B, cfg.U, n_sc, cfg.S, cfg.seed, cfg.qam_bits)
    got = ctx.precode_cg(Hd, T, cfg.rho_d, cfg.K)
    torch.cuda.synchronize()
    got = {k: _np(v) for k, v in got.items()}
    want = ref.precode(_np(Hd), _np(T), cfg.rho_d, cfg.K, threads=THREADS)
    sec = {"subcarriers": n_sc, "of": cfg.n_sc, "vectors": n_sc * cfg.S,
           "status_equal": bool((got["status"] == want["status"]).all())}
    for k in ("q", "s", "gain"):
        sec[k] = _report(got[k], want[k])
    return sec


def both_section(ctx, ref, cfg, n_sc):
    import torch

    H, Y = _gen(ctx, cfg, n_sc)
    T = ctx.generate_symbols(cfg.U, n_sc, cfg.S, cfg.seed, cfg.qam_bits)
    got = ctx.detect_precode_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K, cfg.tracker,
                                T, cfg.rho_d, cfg.K)
    torch.cuda.synchronize()
    got = {k: _np(v) for k, v in got.items()}
    Hn = _np(H)
    want = ref.detect(Hn, _np(Y), cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K, cfg.tracker,
                      threads=THREADS)
    Hd = np.ascontiguousarray(np.conj(np.transpose(Hn, (0, 2, 1))))
    wantd = ref.precode(Hd, _np(T), cfg.rho_d, cfg.K, threads=THREADS)
    sec = {"subcarriers": n_sc, "of": cfg.n_sc, "vectors": n_sc * cfg.S,
           "status_equal": bool((got["status"] == want["status"]).all()),
           "pstatus_equal": bool((got["pstatus"] == wantd["status"]).all())}
    for k in ("xhat", "mu", "rho", "llr"):
        sec[k] = _report(got[k], want[k])
    sec["llr"].update(_flips(got["llr"], want["llr"]))
    for k in ("q", "s", "gain"):
        sec[k] = _report(got[k], wantd[k])
    return sec


def _mmse_errors(cg, ex, bits):
    """Error of a CG-K detector against the exact MMSE one (same inputs)."""
    dx = np.linalg.norm(cg["xhat"] - ex["xhat"], axis=-1) / np.linalg.norm(ex["xhat"], axis=-1)
    drho = np.abs(cg["rho"] - ex["rho"]) / np.abs(ex["rho"])
    dis = (cg["llr"] > 0) != (ex["llr"] > 0)
    return {"xhat_rel_err_median": float(np.median(dx)), "xhat_rel_err_p99": float(np.quantile(dx, 0.99)),
            "rho_rel_err_median": float(np.median(drho)), "rho_rel_err_p99": float(np.quantile(drho, 0.99)),
            "hard_bit_disagreement": float(dis.mean())}


def mmse_comparison(ctx, ref, cfg, H, Y, got_cg, want_cg):
    """CG-K vs exact MMSE on the GPU (Cholesky detector) and on the reference
    (detect_explicit); BASELINE configs[3]."""
    import torch

    ex_gpu = ctx.detect("cholesky", H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, 1)
    torch.cuda.synchronize()
    ex_gpu = {k: _np(v) for k, v in ex_gpu.items()}
    ex_ref = ref.detect(_np(H), _np(Y), cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, method="explicit",
                        threads=THREADS)
    g = _mmse_errors(got_cg, ex_gpu, cfg.qam_bits)
    r = _mmse_errors(want_cg, ex_ref, cfg.qam_bits)
    return {"gpu": g, "reference": r,
            "agreement": {k: abs(g[k] - r[k]) / max(abs(r[k]), 1e-12) for k in g},
            "exact_mmse_gpu_vs_reference": {k: _report(ex_gpu[k], ex_ref[k]) for k in ("xhat", "mu", "rho")}}


def run(n_big=N_BIG, names=None):
    import oracle
    from paper_1404_0424_b200 import Context, get_config

    ctx = Context(0)
    ref = oracle.Oracle("ref")
    names = names or ["cfg1", "cfg2", "cfg3", "cfg4a_K2", "cfg4a_K4", "cfg4a_K8",
                      "cfg4b_K2", "cfg4b_K4", "cfg4b_K8", "cfg5"]
    out = {"contract": "north_star: |got - want| <= 1e-4 + 1e-3 |want|; hard bits equal where "
                       "|LLR_ref| >= 1e-4", "oracle": "oracle/_ref (unmodified reference, FP64)",
           "configs": {}}
    for name in names:
        cfg = get_config(name)
        full = cfg.n_sc <= 16384 and not name.startswith("cfg4")
        n = cfg.n_sc if full else min(cfg.n_sc, n_big)
        if cfg.kind == "downlink":
            sec = precode_section(ctx, ref, cfg, n)
        elif cfg.kind == "both":
            sec = both_section(ctx, ref, cfg, n)
        else:
            sec, (H, Y, got, want) = detect_section(ctx, ref, cfg, n)
            if name.startswith("cfg4"):
                sec["vs_exact_mmse"] = mmse_comparison(ctx, ref, cfg, H, Y, got, want)
        out["configs"][name] = sec
        print(name, json.dumps({k: v for k, v in sec.items() if k != "vs_exact_mmse"})[:400],
              flush=True)
    return out


def failures(rep):
    bad = []
    for name, sec in rep["configs"].items():
        for k, v in sec.items():
            if isinstance(v, dict) and "outside_tol" in v and v["outside_tol"]:
                bad.append((name, k, v["outside_tol"]))
            if isinstance(v, dict) and v.get("hard_bit_flips"):
                bad.append((name, k + " flips", v["hard_bit_flips"]))
            if k.endswith("status_equal") and not v:
                bad.append((name, k, 1))
    return bad


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--big", type=int, default=N_BIG)
    ap.add_argument("--configs", default=None)
    a = ap.parse_args()
    rep = run(a.big, a.configs.split(",") if a.configs else None)
    rep["failures"] = failures(rep)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rep, f, indent=1)
    print("failures:", rep["failures"])
