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


def run(config: str, n_sc: int, threads: int, passes: int, warmup: int) -> dict:
    import oracle
    from paper_1404_0424_b200.configs import get_config

    cfg = get_config(config)
    o = oracle.Oracle("ref") if oracle.available("ref") else oracle.Oracle("port")
    kind = "reference" if o.kind == "ref" else "port"
    if kind == "port":
        threads = 1  # the C restatement is single-threaded
    data = synth(cfg, n_sc)
    H128 = {k: v.astype(np.complex128) for k, v in data.items()}

    def one():
        if cfg.kind in ("uplink", "both"):
            o.detect(H128["H"], H128["Y"], cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,
                     cfg.tracker, threads=threads)
        if cfg.kind == "downlink":
            o.precode(H128["Hd"], H128["T"], cfg.rho_d, cfg.K, threads=threads)
        if cfg.kind == "both":
            Hd = np.ascontiguousarray(np.conj(np.transpose(H128["H"], (0, 2, 1))))
            o.precode(Hd, H128["T"], cfg.rho_d, cfg.K, threads=threads)

    for _ in range(warmup):
        one()
    best = None
    for _ in range(passes):
        t0 = time.perf_counter()
        one()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    vectors = n_sc * cfg.S
    return dict(value=vectors / best, unit="vectors/s", cores=threads, kind=kind,
                seconds_per_pass=best, vectors=vectors,
                sample=f"{config}: {n_sc} subcarriers x {cfg.S} vectors, best of {passes} passes "
                       f"after {warmup} warm-up, per-call FP64 reference over a {threads}-thread "
                       f"pool, GLIBC_TUNABLES malloc protocol")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--n-sc", type=int, default=None)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--passes", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    a = ap.parse_args()
    from paper_1404_0424_b200.configs import get_config

    n_sc = a.n_sc or get_config(a.config).n_sc
    print(json.dumps(run(a.config, n_sc, a.threads, a.passes, a.warmup)))


def spawn(config: str, n_sc: int, threads: int, passes: int = 3, warmup: int = 2,
          timeout: float = 600.0) -> dict:
    """Run main() in a fresh interpreter with the allocator protocol set."""
    import subprocess

    env = dict(os.environ, GLIBC_TUNABLES=GLIBC_TUNABLES, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-m", "oracle.cpu_bench", "--config", config,
                        "--n-sc", str(n_sc), "--threads", str(threads), "--passes", str(passes),
                        "--warmup", str(warmup)], capture_output=True, text=True, env=env,
                       cwd=ROOT, timeout=timeout)
    if r.returncode != 0:
        raise RuntimeError("cpu_bench failed: " + r.stderr[-2000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


if __name__ == "__main__":
    main()
