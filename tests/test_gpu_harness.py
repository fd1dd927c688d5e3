"""GPU: the coded BLER harness against the
reference library: the soft Viterbi decoder bit for bit (coding.cpp:90-147)
and whole uplink trials -- block errors, frames and breakdowns of
run_uplink_sweep (sim.cpp:365-384) on the same seeds."""
import os
import sys

import numpy as np
import pytest

from paper_1404_0424_b200 import sim

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "coding.npz")
sys.path.insert(0, os.path.join(HERE, "golden"))
from make_golden import DL_SWEEP_CASES, SWEEP_CASES  # noqa: E402

pytestmark = pytest.mark.gpu


def test_viterbi_matches_reference_fixture(gpu_ctx):
    d = np.load(GOLDEN)
    for i in range(3):
        for kind in ("noisy", "ties"):
            got = gpu_ctx.viterbi_decode(d[f"llr_{kind}{i}"][None])[0]
            assert np.array_equal(got, d[f"dec_{kind}{i}"]), (i, kind)
        zero = gpu_ctx.viterbi_decode(np.zeros((2, len(d[f"coded{i}"]))))
        assert np.array_equal(zero[1], d[f"dec_zero{i}"])


def test_viterbi_matches_oracle_decoder(gpu_ctx, oracle_port):
    rng = np.random.default_rng(0)
    n_cw, info_len = 24, 634  # the 128-subcarrier 64-QAM frame (coded 768)
    llrs, want = [], []
    for i in range(n_cw):
        info = rng.integers(0, 2, info_len).astype(np.uint8)
        coded = oracle_port.conv_encode(info)
        sigma = [0.3, 0.8, 1.2, 2.0][i % 4]  # clean .. failing codewords
        llr = (2.0 * coded - 1.0) * 2.0 + rng.standard_normal(len(coded)) * sigma * 2.0
        if i == 5:
            llr[:] = 0.0  # all-tie input: the tie rule alone decides
        llrs.append(llr)
        want.append(oracle_port.viterbi_decode(llr))
    got = gpu_ctx.viterbi_decode(np.stack(llrs))
    for i in range(n_cw):
        assert np.array_equal(got[i], want[i]), i


def test_encoder_round_trip(gpu_ctx, oracle_port):
    """Noise-free LLRs of the reference encoder decode to the info bits."""
    rng = np.random.default_rng(1)
    info = rng.integers(0, 2, (3, 94)).astype(np.uint8)  # 94 + 6 tail = 100 = 20 periods
    coded = np.stack([oracle_port.conv_encode(x) for x in info])
    got = gpu_ctx.viterbi_decode(4.0 * coded - 2.0)
    assert np.array_equal(got, info)


@pytest.mark.parametrize("case", range(len(SWEEP_CASES)))
def test_uplink_trials_match_reference_sweep(gpu_ctx, case):
    """Against run_uplink_sweep's own counts (tests/golden/coding.npz, made
    by tests/golden/make_golden.py from the reference library)."""
    B, U, bits, K, tracker, snr, n_sc, trials = SWEEP_CASES[case]
    seed = 7
    f = np.load(GOLDEN)["sweep"][case]
    want = dict(frames=int(f[0]), block_errors=int(f[1]), breakdowns=int(f[2]))
    got = sim.uplink_sweep_point(gpu_ctx, B, U, bits, K, tracker, snr, trials, n_sc, seed)
    assert got["frames"] == want["frames"]
    assert got["breakdowns"] == want["breakdowns"]
    assert got["block_errors"] == want["block_errors"], (got["block_errors"], want["block_errors"])
    # the operating points are chosen to decode some blocks and lose others
    assert 0 < want["block_errors"] < want["frames"] or tracker == "exact"


@pytest.mark.parametrize("case", range(len(DL_SWEEP_CASES)))
def test_downlink_trials_match_reference_sweep(gpu_ctx, case):
    """run_downlink_sweep's counts: CG precoding of every (symbol,
    subcarrier) in one batch, the genie demapper, Viterbi (sim.cpp:205-275)."""
    B, U, bits, K, snr, n_sc, trials = DL_SWEEP_CASES[case]
    f = np.load(GOLDEN)["sweep_dl"][case]
    got = sim.downlink_sweep_point(gpu_ctx, B, U, bits, K, snr, trials, n_sc, 7)
    assert got["frames"] == int(f[0])
    assert got["breakdowns"] == int(f[2])
    assert got["block_errors"] == int(f[1]), (got["block_errors"], int(f[1]))


def test_trial_keys_follow_reference_forks(oracle_port):
    """cgm_sweep_trial_key = Rng(seed).fork(1).fork(point).fork(trial)
    (sim.cpp:378-380): its first draw equals the restated Rng's."""
    keys = sim.trial_keys(7, 2, 3)
    for t, k in enumerate(keys):
        assert oracle_port.rng_u64(int(k), [], 1)[0] == oracle_port.rng_u64(7, [1, 2, t], 1)[0]


@pytest.mark.parametrize("case", range(9))
def test_tradeoff_sweeps_match_reference(gpu_ctx, case):
    """Whole sweeps of the trade-off study (every sim::Method, both
    directions, early stop) against run_*_sweep's SnrPointResults and the
    trade-off rows (tests/golden/tradeoff.npz)."""
    from make_golden import TRADEOFF_GRID, TRADEOFF_SWEEPS, TRADEOFF_TRIALS

    direction, m, K, trk, mbe = TRADEOFF_SWEEPS[case]
    cfg = sim.SweepConfig(bs_antennas=32, users=8, qam_bits=6, method=m, iterations=K,
                          tracker=trk, snr_start_db=TRADEOFF_GRID[0],
                          snr_stop_db=TRADEOFF_GRID[1], snr_step_db=TRADEOFF_GRID[2],
                          trials=TRADEOFF_TRIALS, subcarriers=128, seed=1,
                          max_breakdown_fraction=1.0, max_block_errors=mbe)
    res = sim.run_sweep(gpu_ctx, cfg, direction, batch=16)
    d = np.load(os.path.join(HERE, "golden", "tradeoff.npz"))
    want = d[f"sweep{case}"]
    assert len(res.points) == len(want)
    for p, w in zip(res.points, want):
        assert (p.snr_db, p.frames, p.block_errors, p.breakdowns, p.trials_run) == \
            (w[0], int(w[1]), int(w[2]), int(w[7]), int(w[8])), (p, w)
        assert (p.bler, p.bler_lo, p.bler_hi) == (w[3], w[4], w[5])
        if p.real_mults_mean is not None:
            assert p.real_mults_mean == w[6]
    row = sim.tradeoff_table([res], 0.1)[0]
    rm, snr = d[f"row{case}"]
    assert row.real_mults == int(rm)
    assert (row.snr_db_at_target is None) if np.isnan(snr) else (row.snr_db_at_target == snr)


def test_sweep_through_a_process_group_matches_reference(gpu_ctx):
    """The sharded sweep path (sim._sharded: all_gather of per-trial
    outcomes) on a one-rank group reproduces the early-stop sweep."""
    import socket

    import torch.distributed as dist
    from make_golden import TRADEOFF_GRID, TRADEOFF_SWEEPS, TRADEOFF_TRIALS

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        direction, m, K, trk, mbe = TRADEOFF_SWEEPS[5]
        cfg = sim.SweepConfig(method=m, iterations=K, tracker=trk, snr_start_db=TRADEOFF_GRID[0],
                              snr_stop_db=TRADEOFF_GRID[1], snr_step_db=TRADEOFF_GRID[2],
                              trials=TRADEOFF_TRIALS, max_breakdown_fraction=1.0,
                              max_block_errors=mbe)
        res = sim.run_sweep(gpu_ctx, cfg, direction, batch=4, group=dist.group.WORLD)
    finally:
        dist.destroy_process_group()
    want = np.load(os.path.join(HERE, "golden", "tradeoff.npz"))["sweep5"]
    assert [(p.frames, p.block_errors, p.trials_run) for p in res.points] == \
        [(int(w[1]), int(w[2]), int(w[8])) for w in want]
