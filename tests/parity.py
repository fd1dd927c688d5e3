"""Shared parity helpers: the north_star tolerance contract.

x-hat, SINR rho, mu and LLRs within 1e-3 relative or 1e-4 absolute
(|got - want| <= 1e-4 + 1e-3 |want|); hard bits (LLR > 0 => 1) bit-exact
except where |LLR_ref| < 1e-4; precoder q, s, gain at the same tolerance.
"""
from __future__ import annotations

import numpy as np

RTOL = 1e-3
ATOL = 1e-4


def close_report(got, want, rtol=RTOL, atol=ATOL):
    got = np.asarray(got)
    want = np.asarray(want)
    err = np.abs(got.astype(np.complex128) - want.astype(np.complex128))
    tol = atol + rtol * np.abs(want)
    bad = err > tol
    worst = float(np.max(err / tol)) if err.size else 0.0
    return int(bad.sum()), int(bad.size), worst


def assert_close(got, want, what, rtol=RTOL, atol=ATOL):
    nbad, n, worst = close_report(got, want, rtol, atol)
    assert nbad == 0, f"{what}: {nbad}/{n} outside atol={atol} rtol={rtol} (worst err/tol {worst:.3g})"


def assert_hard_bits(llr_got, llr_want, what="hard bits"):
    g = np.asarray(llr_got)
    w = np.asarray(llr_want)
    mask = np.abs(w) >= ATOL
    flips = ((g > 0) != (w > 0)) & mask
    assert not flips.any(), f"{what}: {int(flips.sum())} of {int(mask.sum())} decided bits differ"


def check_detect(got: dict, want: dict, what: str, xhat_rtol=RTOL):
    assert (np.asarray(got["status"]) == want["status"]).all(), f"{what}: status differs"
    assert_close(got["xhat"], want["xhat"], f"{what} xhat", rtol=xhat_rtol)
    assert_close(got["mu"], want["mu"], f"{what} mu")
    assert_close(got["rho"], want["rho"], f"{what} rho")
    assert_close(got["llr"], want["llr"], f"{what} llr")
    assert_hard_bits(got["llr"], want["llr"], f"{what} hard bits")


def check_precode(got: dict, want: dict, what: str):
    assert (np.asarray(got["status"]) == want["status"]).all(), f"{what}: status differs"
    assert_close(got["q"], want["q"], f"{what} q")
    assert_close(got["s"], want["s"], f"{what} s")
    assert_close(got["gain"], want["gain"], f"{what} gain")
