"""Coded BLER sweeps and the complexity / performance trade-off table on the
GPU.

The reference's run_uplink_sweep / run_downlink_sweep (sim.cpp:365-405) run
their trials one (symbol, subcarrier) solve at a time on a CPU thread pool;
here a batch of trials of an SNR point is one GPU pipeline
(cgm_sweep_trials: frames, channel + noise from the trial's streams, ONE
batched detection or precoding with any sim::Method, the genie demapper
downlink, deinterleaving, soft Viterbi).  Trial streams are the reference's
Rng(seed).fork(direction).fork(point).fork(trial), so block errors match the
reference trial for trial on the same seed.  The host side -- SNR grid,
early stop, Wilson interval, SNR at a target BLER, operation counts and the
trade-off table -- restates sim.cpp / opcount.cpp (cited per function).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field, replace
from typing import List, Optional

import numpy as np

from . import _lib

METHOD_NAMES = ("chol", "cg", "cgls", "neumann")  # sim::Method order (sim.hpp:34)


class ConfigError(ValueError):
    """sim::ConfigError (sim.hpp:25-27)."""


class BreakdownBudgetExceeded(RuntimeError):
    """sim::BreakdownBudgetExceeded (sim.hpp:30-32)."""


def trial_keys(seed: int, point: int, trials: int, direction: int = 1, first: int = 0) -> np.ndarray:
    lib = _lib.load()
    return np.array([lib.cgm_sweep_trial_key(seed, direction, point, t)
                     for t in range(first, first + trials)], dtype=np.uint64)


# ------------------------------------------------------------ configuration
@dataclass
class SweepConfig:
    """sim::SweepConfig (sim.hpp:53-70) with the reference's defaults."""
    bs_antennas: int = 32
    users: int = 8
    qam_bits: int = 6
    method: str = "chol"
    iterations: int = 1
    snr_start_db: float = 10.0
    snr_stop_db: float = 16.0
    snr_step_db: float = 2.0
    trials: int = 100
    subcarriers: int = 128
    seed: int = 1
    tracker: str = "approx"
    max_breakdown_fraction: float = 0.01
    max_block_errors: int = 0


@dataclass
class SnrPointResult:
    """sim::SnrPointResult (sim.hpp:75-85)."""
    snr_db: float
    frames: int = 0
    block_errors: int = 0
    bler: float = 0.0
    bler_lo: float = 0.0
    bler_hi: float = 0.0
    real_mults_mean: Optional[float] = None
    breakdowns: int = 0
    trials_run: int = 0


@dataclass
class SweepResult:
    config: SweepConfig
    direction: str
    points: List[SnrPointResult] = field(default_factory=list)


def plan_frame(subcarriers: int, qam_bits: int):
    """sim.cpp:38-51: fewest OFDM symbols whose coded length is a multiple of
    6 (the rate-5/6 output granularity); info = coded / 6 * 5 - tail."""
    for s in range(1, 7):
        if (subcarriers * qam_bits * s) % 6 == 0:
            coded = subcarriers * qam_bits * s
            info = coded // 6 * 5 - 6
            if info <= 0:
                break
            return s, coded, info
    raise ConfigError("frame does not fit the code")


def validate_config(cfg: SweepConfig):
    """sim.cpp:53-69."""
    if cfg.users < 1 or cfg.bs_antennas < cfg.users:
        raise ConfigError("need bs_antennas >= users >= 1")
    if cfg.snr_step_db <= 0.0:
        raise ConfigError("snr step must be positive")
    if cfg.snr_stop_db < cfg.snr_start_db - 1e-12:
        raise ConfigError("snr stop must not precede snr start")
    if cfg.trials < 1:
        raise ConfigError("need at least one trial")
    if cfg.subcarriers < 1:
        raise ConfigError("need at least one subcarrier")
    if cfg.iterations < 1:
        raise ConfigError("need at least one iteration")
    if not 0.0 <= cfg.max_breakdown_fraction <= 1.0:
        raise ConfigError("breakdown fraction must lie in [0, 1]")
    if cfg.method not in METHOD_NAMES:
        raise ConfigError(f"unknown method: {cfg.method}")
    if cfg.qam_bits not in (2, 4, 6):
        raise ConfigError("modulation must be QPSK, 16-QAM or 64-QAM")
    plan_frame(cfg.subcarriers, cfg.qam_bits)


def snr_grid(cfg: SweepConfig) -> List[float]:
    """sim.cpp:71-76 (accumulated steps, same rounding as the reference)."""
    grid, s = [], cfg.snr_start_db
    while s <= cfg.snr_stop_db + 1e-9:
        grid.append(s)
        s += cfg.snr_step_db
    return grid


def wilson_interval(errors: int, total: int):
    """sim.cpp:78-92: 95% Wilson score interval."""
    if total == 0:
        return 0.0, 1.0
    z = 1.959963984540054
    n = float(total)
    p = errors / n
    z2 = z * z
    denom = 1.0 + z2 / n
    center = (p + z2 / (2.0 * n)) / denom
    half = z * math.sqrt(p * (1.0 - p) / n + z2 / (4.0 * n * n)) / denom
    lo = max(0.0, center - half)
    hi = min(1.0, center + half)
    if errors == 0:
        lo = 0.0
    if errors == total:
        hi = 1.0
    return lo, hi


# ---------------------------------------------------------- operation counts
# opcount::Stage order (opcount.hpp:23-33)
STAGES = ("gram", "matched_filter", "cg_iteration", "tracker", "cholesky", "substitution",
          "neumann_term", "cgls_iteration", "other")


def count_detect_stages(method: str, B: int, U: int, K: int) -> dict:
    """opcount::count_detect_stages (opcount.cpp:69-138): real multiplications
    per detected vector by stage, closed forms (unsigned 64-bit)."""
    b, u, k = B, U, K
    c = dict.fromkeys(STAGES, 0)
    if method in ("chol", "cholesky"):
        c["gram"] = 2 * b * u * u
        c["matched_filter"] = 4 * b * u
        c["cholesky"] = u * (u - 1) + 2 * u * (u - 1) * (u - 2) // 3
        fwd = 2 * (u * u * u - u) // 3
        bwd = 2 * u * u * (u - 1)
        c["substitution"] = fwd + bwd + 4 * u * u + 6 * u * u + 2 * u
    elif method == "cg":
        c["gram"] = 2 * b * u * u
        c["matched_filter"] = 4 * b * u
        c["cg_iteration"] = 2 * u + k * (4 * u * u + 12 * u)
        c["tracker"] = k * u
    elif method == "cgls":
        c["gram"] = 2 * b * u
        c["matched_filter"] = 4 * b * u
        c["cgls_iteration"] = 2 * u + k * (8 * b * u + 4 * b + 14 * u)
        c["tracker"] = k * u
    elif method == "neumann":
        c["gram"] = 2 * b * u * u
        c["matched_filter"] = 4 * b * u
        series = 0
        if k >= 2:
            series += 4 * u * (u - 1)
        if k >= 3:
            series += (k - 2) * 2 * u * u * (u + 1)
        c["neumann_term"] = series
        apply = 2 * u if k == 1 else 4 * u * u
        extract = (u if k == 1 else 4 * u * u) + 2 * u
        c["substitution"] = apply + extract
    else:
        raise ConfigError(f"unknown method: {method}")
    return {s: v % (1 << 64) for s, v in c.items()}


def count_detect(method: str, B: int, U: int, K: int) -> int:
    """opcount::count_detect (opcount.cpp:140-143)."""
    return sum(count_detect_stages(method, B, U, K).values()) % (1 << 64)


# -------------------------------------------------------------- the sweeps
def _sharded(run, start: int, count: int, group):
    """Trials [start, start + count) split into contiguous blocks over the
    ranks of `group` (torch.distributed, one process per GPU); every rank gets
    every trial's (errors, breakdown) back in trial order.  Trials are pure
    functions of their keys, so the split does not change any result."""
    if group is None:
        return run(start, count)
    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    per = -(-count // world)
    lo = min(count, rank * per)
    n = min(count, lo + per) - lo
    e, b = run(start + lo, n) if n > 0 else (np.zeros(0, np.uint32), np.zeros(0, np.uint8))
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")
    mine = torch.full((2, per), -1, dtype=torch.int64, device=dev)
    mine[0, :n] = torch.from_numpy(e.astype(np.int64)).to(dev)
    mine[1, :n] = torch.from_numpy(b.astype(np.int64)).to(dev)
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    full = torch.cat(parts, dim=1).cpu().numpy()
    full = full[:, full[0] >= 0][:, :count]
    return full[0].astype(np.uint32), full[1].astype(np.uint8)


def _fold_point(run, cfg: SweepConfig, snr: float, batch: int, group=None) -> SnrPointResult:
    """sim.cpp:307-361 run_point: fixed trials, or waves with the in-order
    early-stop fold when max_block_errors > 0 (scheduling independent).
    run(first, count) -> (user_errors, breakdown) of trials [first, first + count)."""
    errs = np.zeros(cfg.trials, np.uint32)
    brk = np.zeros(cfg.trials, np.uint8)
    folded = 0 if cfg.max_block_errors else cfg.trials
    done, errors_so_far = 0, 0
    world = 1
    if group is not None:
        import torch.distributed as dist

        world = dist.get_world_size(group)
    while done < cfg.trials:
        end = min(cfg.trials, done + batch * world)
        errs[done:end], brk[done:end] = _sharded(run, done, end - done, group)
        if cfg.max_block_errors:
            stop = False
            for t in range(done, end):
                folded += 1
                if not brk[t]:
                    errors_so_far += int(errs[t])
                if errors_so_far >= cfg.max_block_errors:
                    stop = True
                    break
            if stop:
                break
        done = end
    ok = brk[:folded] == 0
    pt = SnrPointResult(snr_db=snr, trials_run=folded)
    pt.breakdowns = int((~ok).sum())
    pt.frames = int(ok.sum()) * cfg.users
    pt.block_errors = int(errs[:folded][ok].sum())
    if pt.breakdowns > cfg.max_breakdown_fraction * folded:
        raise BreakdownBudgetExceeded("solver breakdowns exceeded the configured budget")
    pt.bler = pt.block_errors / pt.frames if pt.frames > 0 else 0.0
    pt.bler_lo, pt.bler_hi = wilson_interval(pt.block_errors, pt.frames)
    return pt


def _run_point(ctx, cfg: SweepConfig, direction: int, pi: int, snr: float, batch: int,
               group=None):
    method = METHOD_NAMES.index(cfg.method)
    trk = 0 if cfg.tracker == "exact" else 1

    def run(first, count):
        e = np.zeros(count, np.uint32)
        b = np.zeros(count, np.uint8)
        keys = trial_keys(cfg.seed, pi, count, direction, first=first)
        ctx._check(ctx.lib.cgm_sweep_trials(
            ctx.h, direction, method, cfg.bs_antennas, cfg.users, cfg.subcarriers, cfg.qam_bits,
            cfg.iterations, trk, float(snr), count, keys.ctypes.data_as(C.c_void_p),
            e.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p)))
        return e, b

    pt = _fold_point(run, cfg, snr, batch, group)
    # per equalised vector: the closed form where the reference's opcount has
    # one (uplink, all methods except the exact tracker; sim.cpp:359)
    if direction == 1 and not (cfg.method == "cg" and cfg.tracker == "exact") and pt.frames:
        pt.real_mults_mean = float(count_detect(cfg.method, cfg.bs_antennas, cfg.users,
                                                cfg.iterations))
    return pt


def run_sweep(ctx, cfg: SweepConfig, direction: str = "uplink", batch: int = 64,
              group=None) -> SweepResult:
    """sim::run_uplink_sweep / run_downlink_sweep (sim.cpp:365-405).  With a
    torch.distributed `group` (one process per GPU) every SNR point's trials
    are sharded over the ranks and all ranks return the same result."""
    validate_config(cfg)
    d = {"uplink": 1, "downlink": 2}[direction]
    res = SweepResult(config=replace(cfg), direction=direction)
    for pi, snr in enumerate(snr_grid(cfg)):
        res.points.append(_run_point(ctx, cfg, d, pi, snr, batch, group))
    return res


def run_uplink_sweep(ctx, cfg: SweepConfig, batch: int = 64, group=None) -> SweepResult:
    return run_sweep(ctx, cfg, "uplink", batch, group)


def run_downlink_sweep(ctx, cfg: SweepConfig, batch: int = 64, group=None) -> SweepResult:
    return run_sweep(ctx, cfg, "downlink", batch, group)


def snr_at_target_bler(result: SweepResult, target: float) -> Optional[float]:
    """sim.cpp:455-473: exact hit, else log-linear interpolation between the
    first bracketing pair; an exact zero on the right is floored at half an
    error."""
    pts = result.points
    for p in pts:
        if p.bler == target:
            return p.snr_db
    for a, b in zip(pts, pts[1:]):
        if a.bler > target and b.bler < target:
            floor_b = 0.5 / max(1.0, float(b.frames))
            b_bler = max(b.bler, floor_b)
            f = (math.log(a.bler) - math.log(target)) / (math.log(a.bler) - math.log(b_bler))
            return a.snr_db + (b.snr_db - a.snr_db) * min(1.0, max(0.0, f))
    return None


@dataclass
class TradeoffRow:
    """sim::TradeoffRow (sim.hpp:104-109)."""
    method_label: str
    iterations: int
    real_mults: int
    snr_db_at_target: Optional[float]


def tradeoff_table(sweeps: List[SweepResult], target_bler: float = 0.1) -> List[TradeoffRow]:
    """sim.cpp:475-497."""
    rows = []
    for sw in sweeps:
        m = sw.config.method
        rows.append(TradeoffRow(
            method_label=m, iterations=0 if m == "chol" else sw.config.iterations,
            real_mults=count_detect(m, sw.config.bs_antennas, sw.config.users,
                                    sw.config.iterations),
            snr_db_at_target=snr_at_target_bler(sw, target_bler)))
    return rows


def write_tradeoff_csv(rows: List[TradeoffRow], target_bler: float) -> str:
    """sim.cpp:499-516 (same columns and number formats)."""
    out = [f"# cgmimo tradeoff target_bler={target_bler:.6g}\n",
           "method,iters,real_mults,snr_db_at_target\n"]
    for r in rows:
        snr = "n/a" if r.snr_db_at_target is None else f"{r.snr_db_at_target:.4f}"
        out.append(f"{r.method_label},{r.iterations},{r.real_mults},{snr}\n")
    return "".join(out)


# -------------------------------------------------- single-point shortcuts
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
