"""CPU: pin the C restatement (oracle/cg_oracle.c) against the reference
library itself and the committed golden fixtures, and check the reference's
own known-answer tests on the oracle.  These run without a GPU."""
import glob
import os

import numpy as np
import pytest

from conftest import cplx_randn

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def det_fixtures():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "det_*.npz")))


def pre_fixtures():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "pre_*.npz")))


@pytest.mark.parametrize("name", det_fixtures())
def test_port_reproduces_golden_detect(oracle_port, name):
    d = load(name)
    B, U, S, K, bits, exact = (int(x) for x in d["meta"])
    rho_u, n0, es = d["params"]
    got = oracle_port.detect(d["H"], d["Y"], rho_u, n0, es, bits, K, "exact" if exact else "approx")
    for k in ("xhat", "mu", "rho", "llr"):
        np.testing.assert_allclose(got[k], d[k], rtol=1e-12, atol=1e-12, err_msg=f"{name} {k}")
    assert (got["status"] == d["status"]).all()


@pytest.mark.parametrize("name", pre_fixtures())
def test_port_reproduces_golden_precode(oracle_port, name):
    d = load(name)
    B, U, S, K = (int(x) for x in d["meta"])
    got = oracle_port.precode(d["Hd"], d["T"], float(d["params"][0]), K)
    for k in ("q", "s", "gain"):
        np.testing.assert_allclose(got[k], d[k], rtol=1e-12, atol=1e-12, err_msg=f"{name} {k}")
    assert (got["status"] == d["status"]).all()


def test_port_bitwise_equals_reference_random(oracle_ref, oracle_port):
    """Same arithmetic order as the reference: the restatement is bit-exact."""
    rng = np.random.default_rng(7)
    for B, U, S, K, trk, bits in [(24, 8, 2, 3, "exact", 4), (48, 16, 3, 5, "approx", 6),
                                  (20, 7, 1, 7, "exact", 2), (64, 32, 2, 2, "exact", 6)]:
        H = cplx_randn(rng, (3, B, U)).astype(np.complex64)
        Y = cplx_randn(rng, (3, B, S), 4.0).astype(np.complex64)
        a = oracle_ref.detect(H, Y, 2.0, 0.5, 1.0, bits, K, trk)
        b = oracle_port.detect(H, Y, 2.0, 0.5, 1.0, bits, K, trk)
        for k in a:
            assert np.array_equal(a[k], b[k]), (B, U, k)
        a = oracle_ref.detect(H, Y, 2.0, 0.5, 1.0, bits, method="explicit")
        b = oracle_port.detect(H, Y, 2.0, 0.5, 1.0, bits, method="explicit")
        for k in a:
            np.testing.assert_allclose(a[k], b[k], rtol=1e-11, atol=1e-12)
    Hd = cplx_randn(rng, (4, 8, 40)).astype(np.complex64)
    T = cplx_randn(rng, (4, 3, 8)).astype(np.complex64)
    T[1, 2] = 0
    a = oracle_ref.precode(Hd, T, 0.7, 4)
    b = oracle_port.precode(Hd, T, 0.7, 4)
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    assert a["status"][1, 2] == 2  # zero_input (precode.cpp:25-31)


def test_llr_known_answers(oracle_port):
    d = load("llr_cases")
    for (xr, xi, mu, rho, bits), want in zip(d["inputs"], d["llrs"]):
        bits = int(bits)
        got = oracle_port.compute_llrs(complex(xr, xi), mu, rho, bits)
        np.testing.assert_allclose(got, want[:bits], rtol=0, atol=1e-15)


def test_llr_semantics(oracle_port):
    """test_detect.cpp:335-370: sign convention, ties, linearity, erasure."""
    pts, _, _ = oracle_port.constellation(4)
    l0 = oracle_port.compute_llrs(pts[0], 1.0, 1.5, 4)  # label 0000: all bits 0
    assert (l0 < 0).all()
    tie = oracle_port.compute_llrs(0.0 + 0.5j, 1.0, 2.0, 4)
    assert tie[0] == 0.0
    small = oracle_port.compute_llrs(0.9 + 0.9j, 1.0, 0.25, 4)
    doubled = oracle_port.compute_llrs(0.9 + 0.9j, 1.0, 0.5, 4)
    assert np.array_equal(doubled, 2 * small)
    assert (oracle_port.compute_llrs(0.9 + 0.9j, 1e-14, 10.0, 4) == 0).all()
    # clip: far away point, huge rho
    assert (np.abs(oracle_port.compute_llrs(3.0 + 3.0j, 1.0, 1e6, 6)) == 64.0).all()


def test_constellation_tables(oracle_port):
    """constellation.cpp:37-86: unit energy, Gray neighbours, axis subsets."""
    for bits in (2, 4, 6):
        pts, a0, a1 = oracle_port.constellation(bits)
        assert abs(np.mean(np.abs(pts) ** 2) - 1.0) < 1e-12
        half = bits // 2
        L = 1 << half
        scale = 1 / np.sqrt(2 * (L * L - 1) / 3)
        levels = (2 * np.arange(L) - (L - 1)) * scale
        gray = np.arange(L) ^ (np.arange(L) >> 1)
        for p in range(half):
            bit = (gray >> (half - 1 - p)) & 1
            assert sorted(a0[p]) == pytest.approx(sorted(levels[bit == 0]))
            assert sorted(a1[p]) == pytest.approx(sorted(levels[bit == 1]))


def test_kat_noiseless_identity():
    d = load("kat_noiseless_identity")
    llr = d["llr"][0]
    bits = d["bits"].reshape(4, 4)
    assert ((llr > 0) == (bits == 1)).all()
    assert (np.abs(llr) == 64.0).all()


def test_kat_identity_k1_and_zero_obs():
    d = load("kat_identity_k1")
    y = d["Y"][0, :, 0]
    alpha = 1.0 / (1.0 + 1.0 / 5.0)
    np.testing.assert_allclose(d["xhat"][0, 0], alpha * y.astype(np.complex128), rtol=1e-7)
    q = load("kat_zero_obs_qpsk")
    assert (q["xhat"] == 0).all() and (q["llr"] == 0).all()
    s16 = load("kat_zero_obs_16qam")
    assert (s16["llr"][0, 0, :, 0] == 0).all() and (s16["llr"][0, 0, :, 2] == 0).all()
    z = load("kat_zero_transmit")
    assert z["status"][0, 0] == 2 and z["gain"][0, 0] == 0.0 and (z["q"] == 0).all()


def test_exact_cg_at_full_rank_equals_explicit(oracle_port):
    """test_detect.cpp:373-391 / acceptance.cpp:47-76 (K = U)."""
    rng = np.random.default_rng(60)
    H = cplx_randn(rng, (4, 32, 8)).astype(np.complex64)
    Y = cplx_randn(rng, (4, 32, 1)).astype(np.complex64)
    n0 = 0.08
    a = oracle_port.detect(H, Y, 1 / n0, n0, 1.0, 6, 8, "exact")
    b = oracle_port.detect(H, Y, 1 / n0, n0, 1.0, 6, method="explicit")
    np.testing.assert_allclose(a["xhat"], b["xhat"], rtol=1e-6)
    np.testing.assert_allclose(a["mu"], b["mu"], rtol=1e-6)
    np.testing.assert_allclose(a["rho"], b["rho"], rtol=1e-6)
    np.testing.assert_allclose(a["llr"], b["llr"], atol=1e-5)


def test_precoder_mf_limit_and_full_rank(oracle_port):
    """test_precode.cpp:55-79: K = 1 is collinear with H^H t, K = U exact."""
    rng = np.random.default_rng(73)
    Hd = cplx_randn(rng, (3, 8, 32)).astype(np.complex64)
    T = cplx_randn(rng, (3, 1, 8)).astype(np.complex64)
    mf = oracle_port.precode(Hd, T, 4.0, 1)
    for n in range(3):
        d = np.conj(Hd[n].astype(np.complex128)).T @ T[n, 0].astype(np.complex128)
        q = mf["q"][n, 0]
        proj = np.vdot(d, q) / np.vdot(d, d)
        assert np.linalg.norm(q - proj * d) / np.linalg.norm(q) < 1e-10
        assert proj.real > 0 and abs(proj.imag) < 1e-9 * abs(proj)
    full = oracle_port.precode(Hd, T, 4.0, 8)
    ref = oracle_port.precode(Hd, T, 4.0, method="explicit")
    np.testing.assert_allclose(full["q"], ref["q"], rtol=1e-7, atol=1e-12)
    assert np.allclose(np.linalg.norm(full["s"], axis=-1), 1.0, atol=1e-12)


def test_rng_streams_match_reference_fixture(oracle_port):
    d = load("rng")
    assert np.array_equal(oracle_port.rng_u64(12345, [2, 7], 16), d["u64"])
    np.testing.assert_array_equal(oracle_port.rng_cgaussian(99, [3, 11], 0.5, 8), d["gauss"])
    np.testing.assert_array_equal(oracle_port.rayleigh(5, [2, 3], 8, 4), d["rayleigh"])


def test_splitmix_restatement_in_python(oracle_port):
    """rng.cpp:12-31 restated once more, independently, in Python integers."""
    M = (1 << 64) - 1
    G = 0x9E3779B97F4A7C15

    def mix(z):
        z = (z + G) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    def fork(k, s):
        return mix((mix(k ^ 0x8BB84B93962EACC9) + s) & M)

    k = fork(fork(777, 4), 9)
    want = [mix((k + G * c) & M) for c in range(1, 6)]
    assert list(oracle_port.rng_u64(777, [4, 9], 5)) == want


# ------------------------------------------------------- coding (coding.cpp)
def test_port_coding_matches_reference_fixture(oracle_port):
    d = load("coding")
    for i in range(3):
        assert np.array_equal(oracle_port.conv_encode(d[f"info{i}"]), d[f"coded{i}"])
        for kind in ("noisy", "ties"):
            got = oracle_port.viterbi_decode(d[f"llr_{kind}{i}"])
            assert np.array_equal(got, d[f"dec_{kind}{i}"]), (i, kind)
        assert np.array_equal(oracle_port.viterbi_decode(np.zeros(len(d[f"coded{i}"]))),
                              d[f"dec_zero{i}"])
    assert np.array_equal(oracle_port.make_interleaver(99, [4, 3], 768), d["perm_768"])
    assert np.array_equal(oracle_port.make_interleaver(12345, [1, 0, 5, 4, 31], 7200),
                          d["perm_7200"])


def test_port_coding_equals_reference_random(oracle_ref, oracle_port):
    rng = np.random.default_rng(5)
    for n in (4, 34, 289):  # + 6 = multiples of the puncture period 5
        info = rng.integers(0, 2, n).astype(np.uint8)
        coded = oracle_ref.conv_encode(info)
        assert np.array_equal(oracle_port.conv_encode(info), coded)
        llr = np.round(rng.standard_normal(len(coded)) * 3) / 2  # many ties
        assert np.array_equal(oracle_port.viterbi_decode(llr), oracle_ref.viterbi_decode(llr))
    perm = oracle_port.make_interleaver(3, [9], 1000)
    assert np.array_equal(np.sort(perm), np.arange(1000))
    assert np.array_equal(perm, oracle_ref.make_interleaver(3, [9], 1000))


def test_port_coding_rejects_reference_bad_lengths(oracle_port):
    with pytest.raises(ValueError):
        oracle_port.conv_encode(np.zeros(5, np.uint8))  # 11 not a multiple of 5
    with pytest.raises(ValueError):
        oracle_port.viterbi_decode(np.zeros(7))  # not whole periods
    with pytest.raises(ValueError):
        oracle_port.viterbi_decode(np.zeros(6))  # 5 steps < tail 6


# ------------------------------------- trade-off study solvers (section 8(f) row 4)
ALT_DETECT = (("cholesky", 1), ("cgls", 3), ("neumann", 1), ("neumann", 3))
ALT_PRECODE = (("explicit", 1), ("cgls", 2), ("neumann", 2))


def test_port_alt_solvers_match_reference_fixture(oracle_port):
    d = load("alt")
    for m, K in ALT_DETECT:
        got = oracle_port.detect(d["H"], d["Y"], 8.0, 0.125, 1.0, 4, K, method=m)
        for k, v in got.items():
            assert np.array_equal(v, d[f"det_{m}{K}_{k}"]), (m, K, k)
    for m, K in ALT_PRECODE:
        got = oracle_port.precode(d["Hd"], d["T"], 8.0, K, method=m)
        for k, v in got.items():
            assert np.array_equal(v, d[f"pre_{m}{K}_{k}"]), (m, K, k)


@pytest.mark.parametrize("B,U,S", [(32, 8, 2), (12, 12, 1), (20, 7, 3)])
def test_port_alt_solvers_bitwise_equal_reference(oracle_ref, oracle_port, B, U, S):
    rng = np.random.default_rng(B + U)
    n_sc = 4
    H = cplx_randn(rng, (n_sc, B, U)).astype(np.complex64)
    Y = (cplx_randn(rng, (n_sc, B, S)) * 2).astype(np.complex64)
    for m, K in ALT_DETECT + (("cgls", U + 2), ("neumann", 5)):
        a = oracle_ref.detect(H, Y, 5.0, 0.2, 1.0, 6, K, method=m)
        b = oracle_port.detect(H, Y, 5.0, 0.2, 1.0, 6, K, method=m)
        for k in a:
            assert np.array_equal(a[k], b[k]), (m, K, k)
    Hd = np.ascontiguousarray(np.conj(np.transpose(H, (0, 2, 1))))
    T = cplx_randn(rng, (n_sc, S, U)).astype(np.complex64)
    for m, K in ALT_PRECODE + (("cgls", U + 2), ("neumann", 4)):
        a = oracle_ref.precode(Hd, T, 5.0, K, method=m)
        b = oracle_port.precode(Hd, T, 5.0, K, method=m)
        for k in a:
            assert np.array_equal(a[k], b[k]), (m, K, k)


def test_port_alt_solver_identities(oracle_port):
    """Cholesky detection == explicit MMSE (detect.cpp:88-120 vs :122-181);
    min-norm CGLS precoding == CG precoding (same Krylov iterates,
    precode.cpp:56-82); Neumann with 1 term is the diagonal inverse."""
    rng = np.random.default_rng(3)
    H = cplx_randn(rng, (3, 32, 8))
    Y = cplx_randn(rng, (3, 32, 2)) * 2
    a = oracle_port.detect(H, Y, 5.0, 0.2, 1.0, 4, method="cholesky")
    b = oracle_port.detect(H, Y, 5.0, 0.2, 1.0, 4, method="explicit")
    for k in ("xhat", "mu", "rho"):
        np.testing.assert_allclose(a[k], b[k], rtol=1e-9, atol=1e-12)
    Hd = np.conj(np.transpose(H, (0, 2, 1)))
    T = cplx_randn(rng, (3, 2, 8))
    c = oracle_port.precode(Hd, T, 5.0, 3, method="cgls")
    g = oracle_port.precode(Hd, T, 5.0, 3, method="cg")
    np.testing.assert_allclose(c["q"], g["q"], rtol=1e-9, atol=1e-12)
    n1 = oracle_port.detect(H, Y, 5.0, 0.2, 1.0, 4, 1, method="neumann")
    G = np.einsum("nbi,nbj->nij", H.conj(), H)
    d = np.real(np.diagonal(G, axis1=1, axis2=2)) + 0.2
    mf = np.einsum("nbi,nbs->nsi", H.conj(), Y)
    np.testing.assert_allclose(n1["xhat"], mf / d[:, None, :], rtol=1e-12)
