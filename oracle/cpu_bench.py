"""CPU baseline timing of the reference hot path -- TEST INFRASTRUCTURE.

Run by bench.py (cpu_baseline leg and ``--impl reference``) in a subprocess so
the allocator protocol of SURVEY.md section 7 (hard part 7) applies from
process start:
  GLIBC_TUNABLES=glibc.malloc.mmap_threshold=33554432:glibc.malloc.trim_threshold=1073741824:glibc.malloc.top_pad=67108864
It drives the UNMODIFIED reference (oracle/_ref, per-call detect_cg /
precode_cg over a std::thread pool with an atomic work index) on a bounded
sample of the named workload (same shapes and value distributions as the
GPU run), does `warmup` untimed passes and reports the best of `passes`.

    python -m oracle.cpu_bench --config cfg2 --n-sc 1200 --threads 16
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GLIBC_TUNABLES = ("glibc.malloc.mmap_threshold=33554432:glibc.malloc.trim_threshold=1073741824:"
                  "glibc.malloc.top_pad=67108864")


def synth(cfg, n_sc, seed=7):
    """Rayleigh channels, Gray-QAM symbols and AWGN with the config's shapes."""
    import oracle

    rng = np.random.default_rng(seed)
    o = oracle.Oracle("port") if oracle.available("port") else oracle.Oracle("ref")
    pts, _, _ = o.constellation(cfg.qam_bits)

    def cn(shape, var=1.0):
        return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) * np.sqrt(var / 2)

    if cfg.kind == "downlink":
        Hd = cn((n_sc, cfg.U, cfg.B)).astype(np.complex64)
        T = pts[rng.integers(0, 1 << cfg.qam_bits, (n_sc, cfg.S, cfg.U))].astype(np.complex64)
        return dict(Hd=Hd, T=T)
    H = cn((n_sc, cfg.B, cfg.U)).astype(np.complex64)
    X = pts[rng.integers(0, 1 << cfg.qam_bits, (n_sc, cfg.S, cfg.U))]
    Y = (np.einsum("nbu,nsu->nbs", H.astype(np.complex128), X)
         + cn((n_sc, cfg.B, cfg.S), cfg.n0)).astype(np.complex64)
    out = dict(H=H, Y=Y)
    if cfg.kind == "both":
        out["T"] = pts[rng.integers(0, 1 << cfg.qam_bits, (n_sc, cfg.S, cfg.U))].astype(np.complex64)
    return out


def device_inputs(cfg, n_sc, threads):
    """The GPU arm's inputs for subcarriers [0, n_sc) of its frame 0 (rank 0):
    the same seeded streams as the device generator (csrc/cgm_generate.cu),
    drawn on the host with the reference Rng (oracle/ref_shim.cpp
    ref_gen_uplink) -- identical complex64 values up to the last ulp of the
    FP64 libm transcendentals."""
    import oracle

    o = oracle.Oracle("ref")
    if cfg.kind == "downlink":
        raise ValueError("device_inputs: uplink / both configs only")
    rs = cfg.rsqrt()
    out = o.gen_uplink(cfg.seed, cfg.B, cfg.U, 0, n_sc, cfg.S, cfg.qam_bits, cfg.n0,
                       rsqrt=None if rs is None else rs.astype(np.float32),
                       with_t=cfg.kind == "both", threads=threads)
    d = dict(H=out[0], Y=out[1])
    if cfg.kind == "both":
        d["T"] = out[2]
    return d


def run(config: str, n_sc: int, threads: int, passes: int, warmup: int,
        min_seconds: float = 0.0) -> dict:
    """Best of `passes` timed passes of the reference over n_sc subcarriers
    (all S vectors of each).  With min_seconds > 0 the sample is grown (from
    a calibration pass) until one pass takes at least that long, capped at
    the config's own size; the rate is extrapolated linearly (instances are
    independent)."""
    import oracle
    from paper_1404_0424_b200.configs import get_config

    cfg = get_config(config)
    o = oracle.Oracle("ref") if oracle.available("ref") else oracle.Oracle("port")
    kind = "reference" if o.kind == "ref" else "port"
    if kind == "port":
        threads = 1  # the C restatement is single-threaded
    same = kind == "reference" and cfg.kind != "downlink"

    def make(n):
        return device_inputs(cfg, n, threads) if same else synth(cfg, n)

    def one(d):
        if cfg.kind in ("uplink", "both"):
            o.detect(d["H"], d["Y"], cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,
                     cfg.tracker, threads=threads)
        if cfg.kind == "downlink":
            o.precode(d["Hd"], d["T"], cfg.rho_d, cfg.K, threads=threads)
        if cfg.kind == "both":
            Hd = np.ascontiguousarray(np.conj(np.transpose(d["H"], (0, 2, 1))))
            o.precode(Hd, d["T"], cfg.rho_d, cfg.K, threads=threads)

    def timed(d):
        t0 = time.perf_counter()
        one(d)
        return time.perf_counter() - t0

    n_sc = max(1, min(n_sc, cfg.n_sc))
    if min_seconds > 0:
        n_cal = max(1, min(n_sc, 4 * threads))
        dt = timed(make(n_cal))
        while dt < 0.5 and n_cal < cfg.n_sc:  # calibrate on >= 0.5 s of work
            n_cal = min(cfg.n_sc, n_cal * 4)
            dt = timed(make(n_cal))
        n_sc = min(cfg.n_sc, max(n_sc, int(np.ceil(n_cal * min_seconds * 1.25 / dt))))
    data = {k: v.astype(np.complex128) for k, v in make(n_sc).items()}
    for _ in range(warmup):
        one(data)
    best = None
    for _ in range(passes):
        dt = timed(data)
        best = dt if best is None else min(best, dt)
    vectors = n_sc * cfg.S
    src = ("the GPU arm's own complex64 inputs (subcarriers 0..%d of frame 0, rank 0; "
           "device generator streams re-drawn with the reference Rng)" % (n_sc - 1)
           if same else "numpy synthetic inputs of the config's shapes and distributions")
    return dict(value=vectors / best, unit="vectors/s", cores=threads, kind=kind,
                seconds_per_pass=best, vectors=vectors, n_sc=n_sc,
                sample=f"{config}: {n_sc} of {cfg.n_sc} subcarriers x {cfg.S} vectors "
                       f"({vectors} instances, {best:.1f} s per pass; rate extrapolated "
                       f"linearly), best of {passes} passes after {warmup} warm-up, per-call "
                       f"FP64 reference over a {threads}-thread pool, GLIBC_TUNABLES malloc "
                       f"protocol; inputs: {src}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--n-sc", type=int, default=None)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--passes", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--min-seconds", type=float, default=0.0)
    a = ap.parse_args()
    from paper_1404_0424_b200.configs import get_config

    n_sc = a.n_sc or get_config(a.config).n_sc
    print(json.dumps(run(a.config, n_sc, a.threads, a.passes, a.warmup, a.min_seconds)))


def spawn(config: str, n_sc: int, threads: int, passes: int = 3, warmup: int = 2,
          timeout: float = 600.0, min_seconds: float = 0.0) -> dict:
    """Run main() in a fresh interpreter with the allocator protocol set."""
    import subprocess

    env = dict(os.environ, GLIBC_TUNABLES=GLIBC_TUNABLES, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-m", "oracle.cpu_bench", "--config", config,
                        "--n-sc", str(n_sc), "--threads", str(threads), "--passes", str(passes),
                        "--warmup", str(warmup),
                        "--min-seconds", str(min_seconds)], capture_output=True, text=True, env=env,
                       cwd=ROOT, timeout=timeout)
    if r.returncode != 0:
        raise RuntimeError("cpu_bench failed: " + r.stderr[-2000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


if __name__ == "__main__":
    main()
