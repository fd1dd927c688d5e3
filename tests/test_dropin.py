"""The C++ drop-in: a program written against the reference's API compiles
against include/cgmimo/ and links libcgmimo_b200.so (CPU); on a GPU its
per-call detect_cg / precode_cg results and opcount tallies match the
reference (gpu)."""
import os
import struct
import subprocess

import numpy as np
import pytest

from conftest import cplx_randn
from parity import assert_close, assert_hard_bits

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "dropin", "dropin_main.cpp")
PKG = os.path.join(ROOT, "paper_1404_0424_b200")


@pytest.fixture(scope="module")
def dropin_exe(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("dropin") / "dropin_main")
    r = subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-I" + os.path.join(ROOT, "include"),
                        SRC, "-L" + PKG, "-lcgmimo_b200", "-Wl,-rpath," + PKG, "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_dropin_host_behaviour(dropin_exe, oracle_port):
    r = subprocess.run([dropin_exe, "host"], capture_output=True, text=True)
    assert r.returncode == 0, (r.returncode, r.stderr)
    lines = r.stdout.splitlines()
    assert lines[-1] == "host ok"
    for line in lines:
        if line.startswith("constellation"):
            f = line.split()
            bits = int(f[1])
            vals = np.array([float(x) for x in f[2:]])
            pts = vals[0::2] + 1j * vals[1::2]
            want, _, _ = oracle_port.constellation(bits)
            assert np.array_equal(pts, want)
    herm = [line for line in lines if line.startswith("hermitian ")][0].split()[1:]
    v = np.array([float(x) for x in herm])
    full = (v[0:18:2] + 1j * v[1:18:2]).reshape(3, 3)
    want = np.array([[2, 1 + 0.5j, 0.25 - 0.75j], [1 - 0.5j, 3, -1.5 - 2j],
                     [0.25 + 0.75j, -1.5 + 2j, 4]])
    np.testing.assert_array_equal(full, want)  # exact conjugate mirror, real diagonal
    assert np.array_equal(full, full.conj().T)
    assert v[18] == 2.0 and v[19] == 4.0
    assert "hermitian_upper_set_throws 1" in lines
    llrs = [np.array([float(x) for x in line.split()[1:]]) for line in lines if line.startswith("llr")]
    cases = [(0.9 + 0.9j, 1.0, 2.0, 4), (0.0 + 0.5j, 1.0, 2.0, 4), (0.9 + 0.9j, 1e-14, 10.0, 4),
             (0.3 - 1.1j, 0.8, 40.0, 6), (-0.2 + 0.05j, 1.2, -3.0, 6), (1.0 + 0.0j, 1.0, 1.5, 2)]
    for got, (x, mu, rho, bits) in zip(llrs, cases):
        np.testing.assert_allclose(got, oracle_port.compute_llrs(x, mu, rho, bits), atol=1e-14)


@pytest.mark.gpu
def test_dropin_per_call_on_gpu(dropin_exe, checker, tmp_path):
    rng = np.random.default_rng(5)
    B, U, K, bits, n = 32, 8, 3, 6, 5
    n0 = 0.1
    H = [cplx_randn(rng, (B, U)).astype(np.complex64).astype(np.complex128) for _ in range(n)]
    y = [cplx_randn(rng, B, 3.0).astype(np.complex64).astype(np.complex128) for _ in range(n)]
    Bd, Ud, Kd, nd = 48, 8, 4, 3
    Hd = [cplx_randn(rng, (Ud, Bd)).astype(np.complex64).astype(np.complex128) for _ in range(nd)]
    t = [cplx_randn(rng, Ud).astype(np.complex64).astype(np.complex128) for _ in range(nd)]
    t[1][:] = 0
    rho_d = 2.0
    with open(tmp_path / "in.bin", "wb") as f:
        f.write(struct.pack("6i", B, U, K, bits, 0, n))
        for h, v in zip(H, y):
            f.write(h.tobytes())
            f.write(v.tobytes())
        f.write(struct.pack("4i", Bd, Ud, Kd, nd))
        for h, v in zip(Hd, t):
            f.write(h.tobytes())
            f.write(v.tobytes())
        f.write(struct.pack("3d", 1 / n0, n0, rho_d))
    r = subprocess.run([dropin_exe, "gpu", str(tmp_path / "in.bin"), str(tmp_path / "out.bin")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    data = open(tmp_path / "out.bin", "rb").read()
    off = 0

    def take(count, dt):
        nonlocal off
        a = np.frombuffer(data, dt, count, off)
        off += a.nbytes
        return a

    want = checker.detect(np.stack(H), np.stack(y)[:, :, None], 1 / n0, n0, 1.0, bits, K, "exact")
    tallies = []
    for i in range(n):
        xh = take(U, np.complex128)
        mu = take(U, np.float64)
        rho = take(U, np.float64)
        llr = take(U * bits, np.float64).reshape(U, bits)
        tallies.append(take(9, np.uint64))
        assert_close(xh, want["xhat"][i, 0], "dropin xhat")
        assert_close(mu, want["mu"][i, 0], "dropin mu")
        assert_close(rho, want["rho"][i, 0], "dropin rho")
        assert_close(llr, want["llr"][i, 0], "dropin llr")
        assert_hard_bits(llr, want["llr"][i, 0])
    if hasattr(checker, "tally_detect_cg") and checker.kind == "ref":
        # opcount parity: the drop-in records what the reference's
        # instrumented path records (test_opcount.cpp:74-98)
        ref_t = checker.tally_detect_cg(B, U, K, "exact", 1)
        assert np.array_equal(tallies[0], ref_t)
    wantp = checker.precode(np.stack(Hd), np.stack(t)[:, None, :], rho_d, Kd)
    for i in range(nd):
        q = take(Bd, np.complex128)
        s = take(Bd, np.complex128)
        gain, zero = take(2, np.float64)
        trace = take(Kd * Bd, np.complex128).reshape(Kd, Bd)
        assert_close(q, wantp["q"][i, 0], "dropin q")
        assert_close(s, wantp["s"][i, 0], "dropin s")
        assert bool(zero) == bool(wantp["status"][i, 0] & 2)
        assert_close(trace[-1], wantp["q"][i, 0], "dropin q_trace[K-1]")
    broke = take(1, np.int32)[0]
    assert broke == 1


@pytest.mark.gpu
def test_dropin_other_solvers_on_gpu(dropin_exe, checker, tmp_path):
    """detect_cholesky / detect_cgls / detect_neumann and precode_explicit /
    precode_cgls / precode_neumann through the reference's C++ signatures."""
    rng = np.random.default_rng(9)
    B, U, bits, n, K = 32, 8, 4, 3, 3
    n0 = 0.1
    H = [cplx_randn(rng, (B, U)).astype(np.complex64).astype(np.complex128) for _ in range(n)]
    y = [cplx_randn(rng, B, 3.0).astype(np.complex64).astype(np.complex128) for _ in range(n)]
    Bd, Ud, nd, Kd = 48, 6, 2, 2
    Hd = [cplx_randn(rng, (Ud, Bd)).astype(np.complex64).astype(np.complex128) for _ in range(nd)]
    t = [cplx_randn(rng, Ud).astype(np.complex64).astype(np.complex128) for _ in range(nd)]
    rho_d = 4.0
    with open(tmp_path / "in.bin", "wb") as f:
        f.write(struct.pack("5i", B, U, bits, n, K))
        for h, v in zip(H, y):
            f.write(h.tobytes())
            f.write(v.tobytes())
        f.write(struct.pack("4i", Bd, Ud, nd, Kd))
        for h, v in zip(Hd, t):
            f.write(h.tobytes())
            f.write(v.tobytes())
        f.write(struct.pack("3d", 1 / n0, n0, rho_d))
    r = subprocess.run([dropin_exe, "alt", str(tmp_path / "in.bin"), str(tmp_path / "out.bin")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    data = open(tmp_path / "out.bin", "rb").read()
    off = 0

    def take(count, dt):
        nonlocal off
        a = np.frombuffer(data, dt, count, off)
        off += a.nbytes
        return a

    methods = [("cholesky", 1), ("cgls", K), ("neumann", K)]
    want = {m: checker.detect(np.stack(H), np.stack(y)[:, :, None], 1 / n0, n0, 1.0, bits, k,
                              method=m) for m, k in methods}
    from paper_1404_0424_b200 import sim
    for i in range(n):
        for m, k in methods:
            w = want[m]
            xh = take(U, np.complex128)
            mu = take(U, np.float64)
            rho = take(U, np.float64)
            llr = take(U * bits, np.float64).reshape(U, bits)
            tally = take(9, np.uint64)
            assert_close(xh, w["xhat"][i, 0], f"dropin {m} xhat")
            assert_close(mu, w["mu"][i, 0], f"dropin {m} mu")
            assert_close(rho, w["rho"][i, 0], f"dropin {m} rho", rtol=2e-3)
            assert_hard_bits(llr, w["llr"][i, 0], f"dropin {m} hard bits")
            # the reference's closed forms (opcount.cpp:69-138)
            stages = sim.count_detect_stages("chol" if m == "cholesky" else m, B, U, k)
            assert [int(v) for v in tally] == [stages[s] for s in sim.STAGES], m
    for i in range(nd):
        for m, k in [("explicit", 1), ("cgls", Kd), ("neumann", Kd)]:
            wp = checker.precode(np.stack(Hd)[i:i + 1], np.stack(t)[i:i + 1, None, :], rho_d, k,
                                 method=m)
            q = take(Bd, np.complex128)
            s = take(Bd, np.complex128)
            gain = take(1, np.float64)[0]
            assert_close(q, wp["q"][0, 0], f"dropin precode {m} q")
            assert_close(s, wp["s"][0, 0], f"dropin precode {m} s")
            assert_close(gain, wp["gain"][0, 0], f"dropin precode {m} gain")
    assert take(1, np.int32)[0] == 1


RELINK = os.path.join(ROOT, "oracle", "_ref", "relink_sim")
REFSIM = os.path.join(ROOT, "oracle", "_ref", "reference_sim")


@pytest.mark.gpu
@pytest.mark.parametrize("tracker", ["1", "0"])
def test_reference_sim_relinked_against_dropin(tracker):
    """The reference's own caller, unmodified: sim.cpp's run_uplink_sweep /
    run_downlink_sweep (equalize / run_precoder call detect::detect_cg and
    precode::precode_cg per subcarrier, sim.cpp:120-145) compiled from the
    reference sources and linked against libcgmimo_b200.so for every
    detect:: / precode:: / constellation / opcount symbol (oracle/Makefile
    `relink`), reproduces the block-error counts of the same driver linked
    against the reference's own implementations, at every sweep point, for
    the approximate (1) and exact (0) trackers."""
    if not (os.path.exists(RELINK) and os.path.exists(REFSIM)):
        pytest.skip("relinked reference driver not built (oracle/Makefile relink)")
    want = subprocess.run([REFSIM, tracker], capture_output=True, text=True, timeout=600)
    got = subprocess.run([RELINK, tracker], capture_output=True, text=True, timeout=600)
    assert want.returncode == 0 and got.returncode == 0, (want.stderr, got.stderr)
    assert got.stdout.split() == want.stdout.split(), (got.stdout, want.stdout)
    assert len(got.stdout.splitlines()) == 4
