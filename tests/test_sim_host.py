"""CPU: the host side of the BLER sweeps and the trade-off table
(paper_1404_0424_b200.sim) against the
reference: operation-count closed forms (opcount.cpp:69-143), the Wilson
interval (sim.cpp:78-92), SNR at a target BLER and the trade-off rows
(sim.cpp:453-497) on the reference's own sweep outputs (tests/golden/
tradeoff.npz), configuration validation (sim.cpp:53-69)."""
import os
import sys

import numpy as np
import pytest

from paper_1404_0424_b200 import sim

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from make_golden import TRADEOFF_GRID, TRADEOFF_SWEEPS  # noqa: E402

FIX = os.path.join(HERE, "golden", "tradeoff.npz")


@pytest.mark.parametrize("method", ["chol", "cg", "cgls", "neumann"])
def test_count_detect_matches_reference(oracle_ref, method):
    m = sim.METHOD_NAMES.index(method)
    for B, U, K in [(32, 8, 1), (32, 8, 4), (128, 32, 3), (64, 64, 8), (7, 1, 2), (256, 16, 12)]:
        want = oracle_ref.count_detect_stages(m, B, U, K)
        got = sim.count_detect_stages(method, B, U, K)
        assert [got[s] for s in sim.STAGES] == [int(v) for v in want], (method, B, U, K)


def test_wilson_interval_matches_reference(oracle_ref):
    for e, n in [(0, 0), (0, 10), (10, 10), (3, 17), (120, 1000), (1, 1)]:
        assert sim.wilson_interval(e, n) == oracle_ref.wilson(e, n), (e, n)


def test_tradeoff_rows_match_reference_fixture():
    d = np.load(FIX)
    sweeps = []
    for i, (direction, m, K, trk, mbe) in enumerate(TRADEOFF_SWEEPS):
        pts = d[f"sweep{i}"]
        cfg = sim.SweepConfig(method=m, iterations=K, tracker=trk)
        res = sim.SweepResult(cfg, direction, [
            sim.SnrPointResult(snr_db=p[0], frames=int(p[1]), block_errors=int(p[2]),
                               bler=p[2] / p[1] if p[1] else 0.0) for p in pts])
        # the Wilson interval of each point, as run_point computes it
        for p, row in zip(res.points, pts):
            assert sim.wilson_interval(p.block_errors, p.frames) == (row[4], row[5])
        sweeps.append(res)
    rows = sim.tradeoff_table(sweeps, 0.1)
    for i, r in enumerate(rows):
        rm, snr = d[f"row{i}"]
        assert r.real_mults == int(rm)
        if np.isnan(snr):
            assert r.snr_db_at_target is None
        else:
            assert r.snr_db_at_target == snr
    csv = sim.write_tradeoff_csv(rows, 0.1)
    assert csv.splitlines()[1] == "method,iters,real_mults,snr_db_at_target"
    assert csv.splitlines()[2].startswith("chol,0,7288,")


def test_tradeoff_rows_match_reference_on_synthetic_curves(oracle_ref):
    rng = np.random.default_rng(4)
    for _ in range(40):
        n = int(rng.integers(1, 6))
        snr = np.cumsum(rng.uniform(0.5, 3.0, n)) + 5
        frames = rng.integers(0, 300, n).astype(np.uint64)
        errs = np.array([rng.integers(0, f + 1) if f else 0 for f in frames], np.uint64)
        errs = np.sort(errs)[::-1].copy()  # mostly falling curves
        frames = np.maximum(frames, errs)
        target = float(rng.choice([0.1, 0.01, 0.5]))
        want = oracle_ref.tradeoff_row("cg", 32, 8, 4, snr, frames, errs, target)
        cfg = sim.SweepConfig(method="cg", iterations=4)
        res = sim.SweepResult(cfg, "uplink", [
            sim.SnrPointResult(snr_db=float(s), frames=int(f), block_errors=int(e),
                               bler=int(e) / int(f) if f else 0.0)
            for s, f, e in zip(snr, frames, errs)])
        got = sim.tradeoff_table([res], target)[0]
        assert (got.real_mults, got.snr_db_at_target) == want


def test_snr_grid_and_validation():
    assert sim.snr_grid(sim.SweepConfig()) == [10.0, 12.0, 14.0, 16.0]
    assert sim.snr_grid(sim.SweepConfig(snr_start_db=0.0, snr_stop_db=0.3, snr_step_db=0.1)) \
        == [0.0, 0.1, 0.2, 0.30000000000000004]
    assert list(TRADEOFF_GRID) == [10.0, 16.0, 2.0]
    for bad in (dict(users=0), dict(bs_antennas=4, users=8), dict(snr_step_db=0.0),
                dict(snr_stop_db=5.0), dict(trials=0), dict(subcarriers=0),
                dict(iterations=0), dict(max_breakdown_fraction=1.5), dict(method="qr"),
                dict(subcarriers=1, qam_bits=2)):
        with pytest.raises(sim.ConfigError):
            sim.validate_config(sim.SweepConfig(**bad))
    sim.validate_config(sim.SweepConfig())
    assert sim.plan_frame(128, 6) == (1, 768, 634)
    assert sim.plan_frame(60, 4) == (1, 240, 194)
    assert sim.plan_frame(65, 2) == (3, 390, 319)  # 3 OFDM symbols per frame
