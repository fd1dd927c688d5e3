"""GPU: the reference's known-answer tests through the
CUDA path (C ABI, host buffers), each citing the reference test it mirrors.
Exact-in-FP32 cases are asserted exactly; the others at the BASELINE
tolerance (repo:tests/parity.py) or against the oracle."""
import numpy as np
import pytest

from conftest import cplx_randn
from parity import assert_close, check_detect, check_precode

pytestmark = pytest.mark.gpu


def c64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex64))


def test_approx_extraction_known_answer(gpu_ctx):
    """test_detect.cpp:279-296: G = 1, rho_u = 1 (alpha_1 = 1/(1+1) = 0.5),
    N0 = 0.5 -> mu = alpha_1 G = 0.5, rho = G / N0 = 2, exactly."""
    H = c64(np.ones((1, 1, 1)))
    Y = c64(np.full((1, 1, 1), 0.3 + 0.2j))
    got = gpu_ctx.detect_cg(H, Y, 1.0, 0.5, 1.0, 4, 1, "approx")
    assert got["mu"][0, 0, 0] == np.float32(0.5)
    assert got["rho"][0, 0, 0] == np.float32(2.0)
    assert_close(got["xhat"], c64([[[0.15 + 0.1j]]]), "xhat = alpha_1 y")


def test_llr_fixture_16qam_against_exhaustive(gpu_ctx, oracle_port):
    """test_detect.cpp:351-355 (oracle oracles.hpp:116-130): z = 0.9 + 0.9i,
    rho = 2 on 16-QAM.  Built as U = B = 1, G = 1, K = 1, huge rho_u (so
    xhat / mu = y) and N0 = 0.5 (rho = G / N0 = 2)."""
    H = c64(np.ones((1, 1, 1)))
    Y = c64(np.full((1, 1, 1), 0.9 + 0.9j))
    got = gpu_ctx.detect_cg(H, Y, 1e12, 0.5, 1.0, 4, 1, "approx")
    z = complex(got["xhat"][0, 0, 0]) / float(got["mu"][0, 0, 0])
    assert abs(z - (0.9 + 0.9j)) < 1e-6
    want = oracle_port.compute_llrs(0.9 + 0.9j, 1.0, 2.0, 4)
    assert_close(got["llr"][0, 0, 0], want.astype(np.float32), "16-QAM fixture LLRs")


def test_erasure_below_gain_floor(gpu_ctx, oracle_port):
    """test_detect.cpp:368-370 / detect.cpp:72-74: |mu| < 1e-12 erases all
    LLRs to exactly 0.  H = 1e-7 I gives G_ii = 1e-14 and, with rho_u = 1,
    mu = alpha G_ii ~ 1e-14."""
    U = 4
    H = c64(np.eye(U)[None] * 1e-7)
    Y = c64(cplx_randn(np.random.default_rng(3), (1, U, 2)))
    got = gpu_ctx.detect_cg(H, Y, 1.0, 0.3, 1.0, 6, 2, "approx")
    assert (np.abs(got["mu"]) < 1e-12).all()
    assert (got["llr"] == 0).all()
    want = oracle_port.detect(H, Y, 1.0, 0.3, 1.0, 6, 2, "approx")
    assert (want["llr"] == 0).all()


def test_rho_doubling_doubles_llrs(gpu_ctx):
    """test_detect.cpp:357-360: LLR = rho (d0 - d1).  With the approximate
    tracker N0 enters only rho = G_ii / N0, so halving N0 doubles every
    unclipped LLR exactly (power-of-two scaling) and leaves xhat, mu alone."""
    rng = np.random.default_rng(4)
    H = c64(cplx_randn(rng, (16, 64, 8)) * 0.125)
    Y = c64(cplx_randn(rng, (16, 64, 3)) * 0.05)
    a = gpu_ctx.detect_cg(H, Y, 10.0, 4.0, 1.0, 6, 3, "approx")
    b = gpu_ctx.detect_cg(H, Y, 10.0, 2.0, 1.0, 6, 3, "approx")
    assert np.array_equal(a["xhat"], b["xhat"]) and np.array_equal(a["mu"], b["mu"])
    assert np.array_equal(b["rho"], 2 * a["rho"])
    free = np.abs(a["llr"]) < 32.0  # neither side clipped
    assert free.mean() > 0.5
    assert np.array_equal(b["llr"][free], 2 * a["llr"][free])


def test_approx_equals_exact_on_diagonal_gram(gpu_ctx):
    """test_detect.cpp:222-245: for diagonal A the approximate tracker is the
    exact one restricted to the diagonal, so mu agree; rho agrees with the
    exact mu^2 / nu^2 when the interference term vanishes (Es = 0+)."""
    U, B = 8, 8
    d = np.linspace(0.5, 2.0, U)
    H = c64(np.diag(d)[None])  # G = diag(d^2)
    Y = c64(cplx_randn(np.random.default_rng(5), (1, B, 2)))
    ap = gpu_ctx.detect_cg(H, Y, 4.0, 0.25, 1.0, 4, 3, "approx")
    ex = gpu_ctx.detect_cg(H, Y, 4.0, 0.25, 1.0, 4, 3, "exact")
    assert_close(ap["mu"], ex["mu"], "mu approx vs exact (diagonal A)")
    assert_close(ap["xhat"], ex["xhat"], "xhat approx vs exact (diagonal A)")


def test_approx_equals_exact_on_orthogonal_equal_norm_columns(gpu_ctx):
    """test_detect.cpp:298-333: orthogonal columns of equal norm make A a
    multiple of I; both trackers then give the same mu."""
    U, B = 4, 16
    rng = np.random.default_rng(6)
    Q, _ = np.linalg.qr(cplx_randn(rng, (B, U)))
    H = c64((Q * 1.5)[None])
    Y = c64(cplx_randn(rng, (1, B, 3)))
    ap = gpu_ctx.detect_cg(H, Y, 2.0, 0.5, 1.0, 6, 2, "approx")
    ex = gpu_ctx.detect_cg(H, Y, 2.0, 0.5, 1.0, 6, 2, "exact")
    assert_close(ap["mu"], ex["mu"], "mu approx vs exact (A = c I)")


def test_approx_vs_exact_median_error_128x8(gpu_ctx):
    """test_detect.cpp:247-277: at 128 x 8 the approximate tracker's SINR is
    within 15% (median relative error) of the exact tracker's."""
    rng = np.random.default_rng(7)
    H = c64(cplx_randn(rng, (64, 128, 8)))
    Y = c64(cplx_randn(rng, (64, 128, 1)) * 3)
    n0 = 0.8
    ap = gpu_ctx.detect_cg(H, Y, 1 / n0, n0, 1.0, 4, 3, "approx")
    ex = gpu_ctx.detect_cg(H, Y, 1 / n0, n0, 1.0, 4, 3, "exact")
    rel = np.abs(ap["rho"] - ex["rho"]) / np.abs(ex["rho"])
    assert np.median(rel) < 0.15


def test_precoder_k1_collinear_with_matched_filter(gpu_ctx):
    """test_precode.cpp:55-73: after one iteration v_1 = alpha_1 t with
    alpha_1 > 0, so q = H_d^H v_1 is collinear with H_d^H t."""
    rng = np.random.default_rng(8)
    Hd = c64(cplx_randn(rng, (8, 6, 40)))
    T = c64(cplx_randn(rng, (8, 2, 6)))
    got = gpu_ctx.precode_cg(Hd, T, 3.0, 1)
    mf = np.einsum("nub,nsu->nsb", np.conj(Hd).astype(np.complex128), T.astype(np.complex128))
    q = got["q"].astype(np.complex128)
    cos = np.abs(np.sum(np.conj(mf) * q, -1)) / (np.linalg.norm(mf, axis=-1) * np.linalg.norm(q, axis=-1))
    assert (cos > 1 - 1e-5).all()
    ratio = np.sum(np.conj(mf) * q, -1) / np.sum(np.abs(mf) ** 2, -1)  # alpha_1
    assert (ratio.real > 0).all() and (np.abs(ratio.imag) < 1e-5 * ratio.real).all()


def test_precoder_full_rank_equals_explicit(gpu_ctx, checker):
    """test_precode.cpp:75-79: K = U CG precoding equals the explicit
    regularised inverse (FP32 tolerance, well-conditioned H_d)."""
    rng = np.random.default_rng(9)
    U, B = 6, 48
    Hd = c64(cplx_randn(rng, (6, U, B)))
    T = c64(cplx_randn(rng, (6, 2, U)))
    got = gpu_ctx.precode_cg(Hd, T, 5.0, U)
    want = checker.precode(Hd, T, 5.0, U, method="explicit")
    assert_close(got["q"], want["q"], "q vs explicit", rtol=2e-3)
    assert_close(got["gain"], want["gain"], "gain vs explicit", rtol=2e-3)


def test_maximum_sizes(gpu_ctx, checker):
    """Largest supported shapes: U = 64 users, 64 vectors per subcarrier
    (kMaxSys), exact tracker, at the BASELINE U = 64 operating point
    (config 4b: 20 dB, N0 = U / 100, rho_u = 1 / N0) with K = 8 under the
    full contract; the precoder at U = 64, St = 64, K = 16 (kMaxK)."""
    rng = np.random.default_rng(10)
    n0 = 0.64
    Hg, Yg = gpu_ctx.generate_uplink(128, 64, 2, 64, 10, 6, n0)  # y = H x + n, 64-QAM
    H, Y = Hg.cpu().numpy(), Yg.cpu().numpy()
    got = gpu_ctx.detect_cg(H, Y, 1 / n0, n0, 1.0, 6, 8, "exact")
    want = checker.detect(H, Y, 1 / n0, n0, 1.0, 6, 8, "exact", threads=8)
    check_detect(got, want, "max sizes U=64 S=64 K=8")
    Hd = c64(cplx_randn(rng, (2, 64, 96)))
    T = c64(cplx_randn(rng, (2, 64, 64)))
    gotp = gpu_ctx.precode_cg(Hd, T, 3.0, 16)
    wantp = checker.precode(Hd, T, 3.0, 16, threads=8)
    check_precode(gotp, wantp, "max sizes precode U=64 St=64 K=16")


def test_exact_tracker_weak_regularisation_high_k(gpu_ctx, checker):
    """U = 64 at high SNR / weak regularisation (28 dB: N0 = 0.1, rho_u = 10;
    y = H x + n with 64-QAM x), K = 8 and K = 16 (kMaxK).  x-hat, mu, rho
    under the contract, hard bits under the |LLR| >= 1e-4 rule; LLRs within
    1e-3 relative / 1e-2 absolute: with rho ~ 600, an LLR next to a decision
    boundary carries rho x (FP32 relative error of x-hat/mu, ~1e-6) of
    absolute error, above the contract's 1e-4 floor for any FP32 CG
    (DESIGN.md section 5).  This case drove the Chebyshev interval [rho^-1,
    1.1 lambda_max]: round 1's tr/Frobenius interval
    lost ~1% in mu at K = 16 and flipped hard bits."""
    from parity import assert_hard_bits

    Hg, Yg = gpu_ctx.generate_uplink(128, 64, 2, 64, 11, 6, 0.1)
    H, Y = Hg.cpu().numpy(), Yg.cpu().numpy()
    for K in (8, 16):
        got = gpu_ctx.detect_cg(H, Y, 10.0, 0.1, 1.0, 6, K, "exact")
        want = checker.detect(H, Y, 10.0, 0.1, 1.0, 6, K, "exact", threads=8)
        for k in ("xhat", "mu", "rho"):
            assert_close(got[k], want[k], f"U=64 rho_u=10 K={K} {k}")
        assert_close(got["llr"], want["llr"], f"U=64 rho_u=10 K={K} llr", atol=1e-2)
        assert_hard_bits(got["llr"], want["llr"])
        assert (got["status"] == want["status"]).all()


def test_empty_batch_is_a_no_op(gpu_ctx):
    """n_sc = 0: nothing to do, status OK, no launches."""
    before = gpu_ctx.kernel_launches
    H = np.zeros((0, 16, 4), np.complex64)
    Y = np.zeros((0, 16, 2), np.complex64)
    got = gpu_ctx.detect_cg(H, Y, 1.0, 1.0, 1.0, 4, 2, "approx")
    assert got["llr"].shape == (0, 2, 4, 4)
    assert gpu_ctx.kernel_launches == before


def test_unsupported_sizes_fail_loudly(gpu_ctx):
    """Beyond the supported maxima the call fails with EINVAL -> ValueError
    (no silent fallback): U = 65, K = 17, 65 vectors per subcarrier."""
    with pytest.raises(ValueError):
        gpu_ctx.detect_cg(np.zeros((1, 8, 65), np.complex64), np.zeros((1, 8, 1), np.complex64),
                          1.0, 1.0, 1.0, 4, 2, "approx")
    with pytest.raises(ValueError):
        gpu_ctx.detect_cg(np.zeros((1, 8, 4), np.complex64), np.zeros((1, 8, 1), np.complex64),
                          1.0, 1.0, 1.0, 4, 17, "exact")
    with pytest.raises(ValueError):
        gpu_ctx.detect_cg(np.zeros((1, 8, 4), np.complex64), np.zeros((1, 8, 65), np.complex64),
                          1.0, 1.0, 1.0, 4, 2, "approx")


def test_c_abi_nccl_gather_single_rank(gpu_ctx):
    """cgm_comm_create / cgm_gather (the C ABI's multi-GPU gather, NCCL via
    dlopen) on a one-rank communicator: the root's own shard lands in recv.
    Multi-rank behaviour is covered by tests/test_multiproc.py (gloo) and the
    torchrun bench; one GPU here cannot host two NCCL ranks."""
    import torch

    from paper_1404_0424_b200.parallel import Comm

    comm = Comm(gpu_ctx, 1, 0, Comm.unique_id())
    send = torch.arange(1000, dtype=torch.float32, device="cuda")
    recv = torch.zeros(1000, dtype=torch.float32, device="cuda")
    comm.gather(send, [send.numel() * 4], recv, root=0)
    torch.cuda.synchronize()
    assert torch.equal(recv, send)
    comm.close()


def test_sharded_pipeline_nccl_single_rank_equals_direct_call(gpu_ctx):
    """parallel.ShardedPipeline through the product C ABI (NcclTransport ->
    cgm_gatherv on a one-rank communicator) on a cfg5-shaped job, 3 chunks:
    the chunked compute + in-place gather gives bitwise the one-call result
    (the root's own chunks are computed straight into the whole-job buffers,
    so cgm_gatherv's self-displacement path is exercised)."""
    import torch

    from paper_1404_0424_b200 import Context, get_config
    from paper_1404_0424_b200.parallel import (Comm, NcclTransport, ShardedPipeline,
                                               detect_precode_outputs)

    cfg = get_config("cfg5").scaled(300)
    rs = torch.tensor(cfg.rsqrt())
    H, Y = gpu_ctx.generate_uplink(cfg.B, cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits, cfg.n0,
                                   rsqrt=rs)
    T = gpu_ctx.generate_symbols(cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits)
    want = gpu_ctx.detect_precode_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,
                                     cfg.tracker, T, cfg.rho_d, cfg.K)
    comm = Comm(Context(0), 1, 0, Comm.unique_id())
    spec = detect_precode_outputs(cfg)
    pipe = ShardedPipeline(cfg.n_sc, 0, 1, spec, NcclTransport(comm), n_chunks=3,
                           device=torch.device("cuda", 0))

    def compute(a, b, views):
        o = dict(views)
        gpu_ctx.detect_precode_cg(H[a:b], Y[a:b], cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,
                                  cfg.tracker, T[a:b], cfg.rho_d, cfg.K, out=o,
                                  want=tuple(views))

    got = pipe.run(compute)
    torch.cuda.synchronize()
    for k in spec:
        assert torch.equal(got[k], want[k]), k
    comm.close()
