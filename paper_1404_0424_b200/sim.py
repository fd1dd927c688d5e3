"""Coded BLER sweeps on the GPU.

The reference's run_uplink_sweep / run_downlink_sweep (sim.cpp:365-405) run
their trials one (symbol, subcarrier) solve at a time on a CPU thread pool;
here a batch of trials of an SNR point is one GPU pipeline
(cgm_uplink_trials / cgm_downlink_trials: frames, channel + noise from the
trial's streams, ONE batched CG detection or precoding, the genie demapper
downlink, deinterleaving, soft Viterbi).  Trial streams are the reference's
Rng(seed).fork(direction).fork(point).fork(trial), so block errors match the
reference trial for trial on the same seed.
"""
from __future__ import annotations

import numpy as np

from . import _lib


def trial_keys(seed: int, point: int, trials: int, direction: int = 1) -> np.ndarray:
    lib = _lib.load()
    return np.array([lib.cgm_sweep_trial_key(seed, direction, point, t) for t in range(trials)],
                    dtype=np.uint64)


def _fold(run, keys, trials, U, batch):
    errs = np.zeros(trials, np.uint32)
    brk = np.zeros(trials, np.uint8)
    for t0 in range(0, trials, batch):
        e, b = run(keys[t0:t0 + batch])
        errs[t0:t0 + batch] = e
        brk[t0:t0 + batch] = b
    ok = brk == 0
    return {"frames": int(ok.sum()) * U, "block_errors": int(errs[ok].sum()),
            "breakdowns": int((~ok).sum()), "trials_run": trials, "per_trial_errors": errs}


def uplink_sweep_point(ctx, B, U, qam_bits, K, tracker, snr_db, trials, n_sc, seed, point=0,
                       batch=64):
    """One SNR point of run_uplink_sweep with the CG detector: frames (user
    blocks), block_errors, breakdowns, trials_run -- the reference's
    SnrPointResult counters (sim.cpp:308-361, fixed trial count)."""
    keys = trial_keys(seed, point, trials, direction=1)
    return _fold(lambda k: ctx.uplink_trials(B, U, n_sc, qam_bits, K, tracker, snr_db, k),
                 keys, trials, U, batch)


def downlink_sweep_point(ctx, B, U, qam_bits, K, snr_db, trials, n_sc, seed, point=0, batch=64):
    """One SNR point of run_downlink_sweep with the CG precoder (same
    counters as uplink_sweep_point; SNR per user, N0 = 1 / SNR)."""
    keys = trial_keys(seed, point, trials, direction=2)
    return _fold(lambda k: ctx.downlink_trials(B, U, n_sc, qam_bits, K, snr_db, k),
                 keys, trials, U, batch)
