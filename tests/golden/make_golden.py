"""Generate tests/golden/*.npz from the UNMODIFIED reference library.

Runs the reference (oracle/_ref/libcgmimo_ref.so, built by `make -C oracle`
from /root/reference/proj/src) on small seeded complex64 inputs of every
BASELINE shape family plus the known-answer cases of the reference's own
tests, and stores inputs and FP64 outputs.  The fixtures travel with the repo
(the GPU box has no /root/reference) and pin both the C restatement
(tests/test_oracle.py) and the CUDA path (tests/test_gpu_golden.py).

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402


def cn(rng, shape, var=1.0):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) * np.sqrt(var / 2)


# (name, B, U, S, K, tracker, qam_bits, snr_db, n_sc)
DETECT_CASES = [
    ("cfg1_like", 128, 8, 1, 3, "exact", 4, 10.0, 6),
    ("cfg2_like", 128, 32, 14, 4, "approx", 6, 15.0, 2),
    ("cfg4a_like_K8", 64, 32, 1, 8, "exact", 6, 20.0, 4),
    ("cfg4b_like_K4", 128, 64, 1, 4, "exact", 6, 20.0, 2),
    ("cfg5_like_ul", 256, 32, 4, 4, "exact", 6, 15.0, 2),
    ("small_qpsk", 16, 4, 3, 2, "approx", 2, 5.0, 3),
    ("ragged_U5", 12, 5, 2, 5, "exact", 4, 8.0, 3),
]
# (name, B, U, S, K, snr_db, n_sc)
PRECODE_CASES = [
    ("cfg3_like", 128, 16, 1, 3, 10.0, 6),
    ("cfg5_like_dl", 256, 32, 4, 4, 15.0, 2),
    ("small_dl", 16, 4, 2, 2, 5.0, 3),
]


# run_uplink_sweep points (sim.cpp:365-384) pinned for tests/test_gpu_harness.py:
# (B, U, qam_bits, K, tracker, snr_db, n_sc, trials), seed 7
SWEEP_CASES = [
    (32, 8, 6, 4, "approx", 14.0, 128, 48),   # reference SweepConfig defaults (sim.hpp)
    (32, 8, 6, 3, "exact", 12.0, 128, 32),
    (64, 16, 4, 3, "approx", 6.0, 60, 32),    # 16-QAM
    (16, 4, 2, 2, "exact", 2.0, 90, 32),      # QPSK
    (16, 4, 2, 2, "approx", 2.0, 65, 32),     # QPSK, 3 OFDM symbols per frame
    (32, 8, 4, 3, "exact", 8.0, 61, 24),      # 16-QAM, 3 OFDM symbols per frame
]

# run_downlink_sweep points (sim.cpp:386-405): (B, U, qam_bits, K, snr_db, n_sc, trials), seed 7
DL_SWEEP_CASES = [
    (32, 8, 6, 4, 13.0, 128, 48),
    (64, 16, 4, 3, 7.0, 60, 32),
    (16, 4, 2, 2, 0.0, 90, 32),
    (32, 8, 6, 1, 12.0, 128, 32),   # K = 1: matched-filter direction
    (16, 4, 2, 2, 0.0, 65, 32),     # QPSK, 3 OFDM symbols per frame
]


def coding_fixtures(ref):
    """coding.cpp: encoder outputs, soft-Viterbi decisions (incl. tie-heavy
    integer LLRs and an all-zero input) and interleavers; plus sweep points."""
    rng = np.random.default_rng(20261019)
    d = {}
    for i, n in enumerate([94, 634, 994]):  # + 6 tail = 20 / 128 / 200 periods
        info = rng.integers(0, 2, n).astype(np.uint8)
        coded = ref.conv_encode(info)
        d[f"info{i}"], d[f"coded{i}"] = info, coded
        noisy = (2.0 * coded - 1.0) * 2.0 + rng.standard_normal(len(coded)) * 2.0
        ties = rng.integers(-2, 3, len(coded)).astype(np.float64)
        d[f"llr_noisy{i}"], d[f"dec_noisy{i}"] = noisy, ref.viterbi_decode(noisy)
        d[f"llr_ties{i}"], d[f"dec_ties{i}"] = ties, ref.viterbi_decode(ties)
        d[f"dec_zero{i}"] = ref.viterbi_decode(np.zeros(len(coded)))
    d["perm_768"] = ref.make_interleaver(99, [4, 3], 768)
    d["perm_7200"] = ref.make_interleaver(12345, [1, 0, 5, 4, 31], 7200)
    sweep = np.zeros((len(SWEEP_CASES), 4), np.int64)
    for i, (B, U, bits, K, trk, snr, n_sc, trials) in enumerate(SWEEP_CASES):
        r = ref.uplink_sweep_point(B, U, bits, K, trk, snr, trials, n_sc, 7, threads=8)
        sweep[i] = [r["frames"], r["block_errors"], r["breakdowns"], r["trials_run"]]
    d["sweep"] = sweep
    dl = np.zeros((len(DL_SWEEP_CASES), 4), np.int64)
    for i, (B, U, bits, K, snr, n_sc, trials) in enumerate(DL_SWEEP_CASES):
        r = ref.downlink_sweep_point(B, U, bits, K, snr, trials, n_sc, 7, threads=8)
        dl[i] = [r["frames"], r["block_errors"], r["breakdowns"], r["trials_run"]]
    d["sweep_dl"] = dl
    return d


def alt_fixtures(ref):
    """The trade-off study's other solvers (detect.cpp:122-326,
    precode.cpp:45-93) on one small seeded uplink and downlink batch."""
    rng = np.random.default_rng(20261020)
    n_sc, B, U, S = 6, 24, 6, 2
    H = cn(rng, (n_sc, B, U)).astype(np.complex64)
    Y = cn(rng, (n_sc, B, S), 3.0).astype(np.complex64)
    Hd = cn(rng, (n_sc, U, B)).astype(np.complex64)
    T = cn(rng, (n_sc, S, U)).astype(np.complex64)
    d = dict(H=H, Y=Y, Hd=Hd, T=T)
    for m, K in (("cholesky", 1), ("cgls", 3), ("neumann", 1), ("neumann", 3)):
        r = ref.detect(H, Y, 8.0, 0.125, 1.0, 4, K, method=m)
        for k, v in r.items():
            d[f"det_{m}{K}_{k}"] = v
    for m, K in (("explicit", 1), ("cgls", 2), ("neumann", 2)):
        r = ref.precode(Hd, T, 8.0, K, method=m)
        for k, v in r.items():
            d[f"pre_{m}{K}_{k}"] = v
    return d


# the trade-off study (sim.cpp:365-516): (direction, method, iters, tracker,
# max_block_errors) on the reference SweepConfig's array / frame (32 x 8,
# 64-QAM, 128 subcarriers), SNR 10:16:2 dB, 24 trials, seed 1
TRADEOFF_SWEEPS = [
    ("uplink", "chol", 1, "approx", 0),
    ("uplink", "cg", 3, "approx", 0),
    ("uplink", "cg", 4, "exact", 0),
    ("uplink", "cgls", 3, "approx", 0),
    ("uplink", "neumann", 3, "approx", 0),
    ("uplink", "chol", 1, "approx", 40),      # early stop (sim.cpp:315-332)
    ("downlink", "chol", 1, "approx", 0),
    ("downlink", "cgls", 2, "approx", 0),
    ("downlink", "neumann", 2, "approx", 0),
]
TRADEOFF_GRID = (10.0, 16.0, 2.0)
TRADEOFF_TRIALS = 24


def tradeoff_fixtures(ref):
    d = {}
    for i, (direction, m, K, trk, mbe) in enumerate(TRADEOFF_SWEEPS):
        pts = ref.sweep(direction, m, 32, 8, 6, K, trk, *TRADEOFF_GRID, TRADEOFF_TRIALS, 128, 1,
                        max_block_errors=mbe, threads=8)
        d[f"sweep{i}"] = np.array([[p[k] for k in ("snr_db", "frames", "block_errors", "bler",
                                                   "bler_lo", "bler_hi", "real_mults_mean",
                                                   "breakdowns", "trials_run")] for p in pts])
        rm, snr = ref.tradeoff_row(m, 32, 8, K, d[f"sweep{i}"][:, 0],
                                   d[f"sweep{i}"][:, 1].astype(np.uint64),
                                   d[f"sweep{i}"][:, 2].astype(np.uint64), 0.1)
        d[f"row{i}"] = np.array([rm, np.nan if snr is None else snr])
    return d


def main():
    ref = oracle.Oracle("ref")
    only = {"--only-coding": ("coding", coding_fixtures), "--only-alt": ("alt", alt_fixtures),
            "--only-tradeoff": ("tradeoff", tradeoff_fixtures)}
    for flag, (name, fn) in only.items():
        if flag in sys.argv:
            np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **fn(ref))
            print(f"wrote {name}.npz")
            return
    rng = np.random.default_rng(20260419)
    out = {}
    for name, B, U, S, K, trk, bits, snr, n_sc in DETECT_CASES:
        n0 = U / 10 ** (snr / 10)
        rho_u = 1.0 / n0
        H = cn(rng, (n_sc, B, U)).astype(np.complex64)
        pts, _, _ = ref.constellation(bits)
        X = pts[rng.integers(0, 1 << bits, (n_sc, S, U))]
        Y = (np.einsum("nbu,nsu->nbs", H.astype(np.complex128), X)
             + cn(rng, (n_sc, B, S), n0)).astype(np.complex64)
        r = ref.detect(H, Y, rho_u, n0, 1.0, bits, K, trk)
        out[f"det_{name}"] = dict(H=H, Y=Y, meta=np.array([B, U, S, K, bits, trk == "exact"]),
                                  params=np.array([rho_u, n0, 1.0]), **r)
    for name, B, U, S, K, snr, n_sc in PRECODE_CASES:
        n0 = 1.0 / 10 ** (snr / 10)
        rho_d = 1.0 / (U * n0)
        Hd = cn(rng, (n_sc, U, B)).astype(np.complex64)
        pts, _, _ = ref.constellation(4)
        T = pts[rng.integers(0, 16, (n_sc, S, U))].astype(np.complex64)
        r = ref.precode(Hd, T, rho_d, K)
        out[f"pre_{name}"] = dict(Hd=Hd, T=T, meta=np.array([B, U, S, K]),
                                  params=np.array([rho_d]), **r)
    # known answers from the reference's tests (test_detect.cpp:71-89, :347-370,
    # :393-422; test_precode.cpp:42-53): identity channels, zero observation
    kat = {}
    I4 = np.eye(4, dtype=np.complex64)[None]
    bits = np.array([0, 1, 1, 0, 1, 1, 0, 0, 0, 0, 1, 1, 1, 0, 1, 0], np.uint8)
    pts16, _, _ = ref.constellation(4)
    labels = bits.reshape(4, 4) @ np.array([8, 4, 2, 1])
    x = pts16[labels].astype(np.complex64)
    r = ref.detect(I4, x[None, :, None], 1e12, 1e-12, 1.0, 4, 4, "exact")
    kat["noiseless_identity"] = dict(H=I4, Y=x[None, :, None], bits=bits, **r)
    y = cn(np.random.default_rng(61), 4).astype(np.complex64)
    r = ref.detect(I4, y[None, :, None], 5.0, 0.2, 1.0, 4, 1, "approx")
    kat["identity_k1"] = dict(H=I4, Y=y[None, :, None], **r)
    z = np.zeros((1, 4, 1), np.complex64)
    kat["zero_obs_qpsk"] = dict(H=I4, Y=z, **ref.detect(I4, z, 4.0, 0.25, 1.0, 2, 3, "approx"))
    kat["zero_obs_16qam"] = dict(H=I4, Y=z, **ref.detect(I4, z, 4.0, 0.25, 1.0, 4, 3, "approx"))
    tz = np.zeros((1, 1, 4), np.complex64)
    kat["zero_transmit"] = dict(Hd=I4, T=tz, **ref.precode(I4, tz, 2.0, 2))
    for k, v in kat.items():
        out[f"kat_{k}"] = v
    # LLR known answers (detect.cpp:68-86 via compute_llrs)
    llr_cases = [(0.9 + 0.9j, 1.0, 2.0, 4), (0.0 + 0.5j, 1.0, 2.0, 4), (0.9 + 0.9j, 1e-14, 10.0, 4),
                 (0.3 - 1.1j, 0.8, 40.0, 6), (-0.2 + 0.05j, 1.2, -3.0, 6), (1.0 + 0.0j, 1.0, 1.5, 2)]
    arr = np.array([[c.real, c.imag, m, r_, b] for c, m, r_, b in llr_cases])
    vals = np.zeros((len(llr_cases), 6))
    for i, (c, m, r_, b) in enumerate(llr_cases):
        vals[i, :b] = ref.compute_llrs(c, m, r_, b)
    out["llr_cases"] = dict(inputs=arr, llrs=vals)
    # RNG streams (rng.cpp): u64 draws and Rayleigh channel of a fork path
    out["rng"] = dict(u64=ref.rng_u64(12345, [2, 7], 16),
                      gauss=ref.rng_cgaussian(99, [3, 11], 0.5, 8),
                      rayleigh=ref.rayleigh(5, [2, 3], 8, 4))
    out["coding"] = coding_fixtures(ref)
    out["alt"] = alt_fixtures(ref)
    out["tradeoff"] = tradeoff_fixtures(ref)
    for name, d in out.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    print(f"wrote {len(out)} fixtures to {HERE}")


if __name__ == "__main__":
    main()
