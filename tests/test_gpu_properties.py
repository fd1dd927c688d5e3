"""GPU: full-size BASELINE configs, checked through size-independent
properties (the oracle is too slow at these sizes): completion, value
ranges, run-to-run determinism, shard invariance (results do not depend on
how subcarriers are split across launches / GPUs), exact power-of-two
linearity, host-buffer == device-buffer results, and a random subsample of
full-size instances against the oracle."""
import numpy as np
import pytest
import torch

from paper_1404_0424_b200 import get_config
from parity import check_detect, check_precode

pytestmark = pytest.mark.gpu


def gen(ctx, cfg, sc0=0, n_sc=None):
    n = cfg.n_sc if n_sc is None else n_sc
    rs = cfg.rsqrt()
    rs = None if rs is None else torch.tensor(rs)
    H, Y = ctx.generate_uplink(cfg.B, cfg.U, n, cfg.S, cfg.seed, cfg.qam_bits, cfg.n0, sc0=sc0,
                               rsqrt=rs)
    return H, Y


def assert_contract(a, b, what):
    """Two GPU variants' outputs agree within the north_star contract,
    elementwise: |a - b| <= 1e-4 + 1e-3 |b|; status bytes equal; hard LLR
    bits equal wherever |LLR| >= 1e-4."""
    for k in a:
        if a[k] is None or k not in b:
            continue
        x, y = a[k], b[k]
        if x.dtype == torch.uint8:
            assert torch.equal(x, y), (what, k)
            continue
        if x.is_complex():
            x, y = torch.view_as_real(x), torch.view_as_real(y)
        bad = (x - y).abs() > 1e-4 + 1e-3 * y.abs()
        assert int(bad.sum()) == 0, (what, k, float((x - y).abs().max()), int(bad.sum()))
        if k == "llr":
            flip = ((x > 0) != (y > 0)) & (y.abs() >= 1e-4)
            assert int(flip.sum()) == 0, (what, "hard bits", int(flip.sum()))


def run(ctx, cfg, H, Y):
    out = ctx.detect_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K, cfg.tracker)
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg4a_K8", "cfg4b_K2"])
def test_full_size_uplink_properties(gpu_ctx, checker, name):
    cfg = get_config(name)
    if cfg.n_sc > 16384:
        cfg = cfg.scaled(16384)
    H, Y = gen(gpu_ctx, cfg)
    a = run(gpu_ctx, cfg, H, Y)
    b = run(gpu_ctx, cfg, H, Y)
    assert int(a["status"].sum()) == 0
    for k in a:  # bitwise deterministic
        assert torch.equal(a[k], b[k]), k
    llr = a["llr"]
    assert torch.isfinite(llr).all() and float(llr.abs().max()) <= 64.0
    assert torch.isfinite(a["rho"]).all() and float(a["mu"].min()) > 0
    # shard invariance: regenerate + detect a middle slice on its own
    s0, n = cfg.n_sc // 3, cfg.n_sc // 4
    Hs, Ys = gen(gpu_ctx, cfg, sc0=s0, n_sc=n)
    assert torch.equal(Hs, H[s0:s0 + n]) and torch.equal(Ys, Y[s0:s0 + n])
    c = run(gpu_ctx, cfg, Hs, Ys)
    for k in a:
        assert torch.equal(c[k], a[k][s0:s0 + n]), k
    # random subsample of full-size instances against the oracle
    idx = np.random.default_rng(0).choice(cfg.n_sc, size=16, replace=False)
    Hn, Yn = H[idx].cpu().numpy(), Y[idx].cpu().numpy()
    want = checker.detect(Hn, Yn, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K, cfg.tracker,
                          threads=8)
    check_detect({k: v[idx].cpu().numpy() for k, v in a.items()}, want, name + " subsample")


def test_linearity_power_of_two(gpu_ctx):
    """Scaling the received vectors by 2 is exact in binary FP: CG scalars
    are unchanged, x-hat doubles bitwise, mu is unchanged bitwise."""
    cfg = get_config("cfg2").scaled(256)
    H, Y = gen(gpu_ctx, cfg)
    a = run(gpu_ctx, cfg, H, Y)
    b = run(gpu_ctx, cfg, H, Y * 2)
    assert torch.equal(b["xhat"], a["xhat"] * 2)
    assert torch.equal(b["mu"], a["mu"]) and torch.equal(b["rho"], a["rho"])


def test_host_and_device_buffers_agree_bitwise(gpu_ctx):
    cfg = get_config("cfg2").scaled(700)
    H, Y = gen(gpu_ctx, cfg)
    dev = run(gpu_ctx, cfg, H, Y)
    host = gpu_ctx.detect_cg(H.cpu().numpy(), Y.cpu().numpy(), cfg.rho_u, cfg.n0, cfg.es,
                             cfg.qam_bits, cfg.K, cfg.tracker)
    for k in host:
        assert np.array_equal(host[k], dev[k].cpu().numpy()), k


def test_cfg5_full_size_fused(gpu_ctx, checker):
    cfg = get_config("cfg5").scaled(8192)
    H, Y = gen(gpu_ctx, cfg)
    T = gpu_ctx.generate_symbols(cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits)
    a = gpu_ctx.detect_precode_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,
                                  cfg.tracker, T, cfg.rho_d, cfg.K)
    b = gpu_ctx.detect_precode_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,
                                  cfg.tracker, T * 2, cfg.rho_d, cfg.K)
    torch.cuda.synchronize()
    assert int(a["status"].sum()) == 0 and int(a["pstatus"].sum()) == 0
    assert torch.equal(b["q"], a["q"] * 2) and torch.equal(b["s"], a["s"])  # linearity
    nrm = torch.linalg.vector_norm(a["s"], dim=-1)
    assert float((nrm - 1).abs().max()) < 1e-5  # ||s|| = 1 (test_precode.cpp:104-120)
    idx = np.random.default_rng(1).choice(cfg.n_sc, size=8, replace=False)
    Hn, Yn, Tn = H[idx].cpu().numpy(), Y[idx].cpu().numpy(), T[idx].cpu().numpy()
    want = checker.detect(Hn, Yn, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K, cfg.tracker,
                          threads=8)
    check_detect({k: a[k][idx].cpu().numpy() for k in ("xhat", "mu", "rho", "llr", "status")},
                 want, "cfg5 subsample uplink")
    Hd = np.ascontiguousarray(np.conj(np.transpose(Hn, (0, 2, 1))))
    wantd = checker.precode(Hd, Tn, cfg.rho_d, cfg.K, threads=8)
    check_precode({"q": a["q"][idx].cpu().numpy(), "s": a["s"][idx].cpu().numpy(),
                   "gain": a["gain"][idx].cpu().numpy(), "status": a["pstatus"][idx].cpu().numpy()},
                  wantd, "cfg5 subsample downlink")


def test_generator_matches_reference_streams(gpu_ctx, oracle_port):
    """GPU seeded generator vs the reference Rng streams (rng.cpp): channel
    entries agree to the last complex64 ulp, labels exactly."""
    H, Y, L = gpu_ctx.generate_uplink(16, 4, 3, 2, 77, 4, 0.1, sc0=5, labels=True)
    torch.cuda.synchronize()
    Hn = H.cpu().numpy()
    for i in range(3):
        want = oracle_port.rayleigh(77, [2, 5 + i], 16, 4).astype(np.complex64)
        np.testing.assert_array_max_ulp(Hn[i].view(np.float32), want.view(np.float32), maxulp=1)
    # labels: bits drawn as next_u64() & 1 from root.fork(1).fork(instance)
    Ln = L.cpu().numpy()
    for i in range(3):
        for s in range(2):
            draws = oracle_port.rng_u64(77, [1, (5 + i) * 2 + s], 4 * 4)
            for u in range(4):
                lab = 0
                for b in range(4):
                    lab = (lab << 1) | int(draws[u * 4 + b] & 1)
                assert Ln[i, s, u] == lab


def test_kernel_launch_accounting(gpu_ctx):
    before = gpu_ctx.kernel_launches
    cfg = get_config("cfg2").scaled(64)
    H, Y = gen(gpu_ctx, cfg)
    mid = gpu_ctx.kernel_launches
    run(gpu_ctx, cfg, H, Y)
    assert mid > before  # generator kernels
    assert gpu_ctx.kernel_launches - mid >= 1  # the hot path ran native kernels


@pytest.mark.parametrize("name", ["cfg2", "cfg4a_K8", "cfg5", "cfg4b_K2", "cfg4b_K8"])
def test_tensor_core_channel_matches_ffma_channel(gpu_ctx, checker, name):
    """The tcgen05 channel kernels (bf16 x3 split: cgm_tc.cuh for U = 32,
    cgm_tc64.cuh for U = 64) and the FP32 FFMA channel kernel agree to FP32
    rounding, and the default matches the oracle on a subsample."""
    cfg = get_config(name).scaled(600)
    H, Y = gen(gpu_ctx, cfg)
    tc = run(gpu_ctx, cfg, H, Y)
    gpu_ctx.set_kernel_policy("ffma_channel")
    try:
        ff = run(gpu_ctx, cfg, H, Y)
    finally:
        gpu_ctx.set_kernel_policy("auto")
    assert_contract(tc, ff, "tcgen05 vs FFMA channel")
    assert int(tc["status"].sum()) == 0
    idx = np.random.default_rng(2).choice(cfg.n_sc, size=8, replace=False)
    want = checker.detect(H[idx].cpu().numpy(), Y[idx].cpu().numpy(), cfg.rho_u, cfg.n0, cfg.es,
                          cfg.qam_bits, cfg.K, cfg.tracker, threads=8)
    check_detect({k: v[idx].cpu().numpy() for k, v in tc.items()}, want, name + " tensor-core")


@pytest.mark.parametrize("U,B,K", [(4, 16, 2), (8, 32, 4), (16, 64, 3), (32, 128, 4)])
def test_precode_uplink_layout_equals_downlink_layout(gpu_ctx, U, B, K):
    """precode_cg given H_u with CGM_HD_UPLINK_LAYOUT == precode_cg given
    H_d = H_u^H explicitly (sim.cpp:223 builds H_d exactly so)."""
    g = torch.Generator().manual_seed(U)
    n_sc, S = 37, 3
    H = torch.complex(torch.randn(n_sc, B, U, generator=g), torch.randn(n_sc, B, U, generator=g))
    T = torch.complex(torch.randn(n_sc, S, U, generator=g), torch.randn(n_sc, S, U, generator=g))
    H, T = (H / 2 ** 0.5).cuda(), (T / 2 ** 0.5).cuda()
    Hd = H.conj().transpose(1, 2).contiguous()
    a = gpu_ctx.precode_cg(H, T, 3.0, K, uplink_layout=True)
    b = gpu_ctx.precode_cg(Hd, T, 3.0, K)
    torch.cuda.synchronize()
    for k in ("q", "s"):
        d = float((a[k] - b[k]).abs().max() / b[k].abs().max())
        assert d < 1e-5, (k, d)


@pytest.mark.parametrize("name,policy", [
    ("cfg2", "lane_solve"),        # default: register-tiled block CG, approximate tracker
    ("cfg2", "pairs_cg"),          # the warp-per-pair kernel (Gram row in registers, single-reduction CG)
    ("cfg4a_K2", "lane_solve"),    # default: exact pairs kernel, one system per warp (S = 1)
    ("cfg4a_K8", "lane_solve"),
    ("cfg4a_K8", "ffma_channel"),  # default: tcgen05 channel kernel
    ("cfg5", "lane_solve"),        # default: 8-warp row CTA with the precoder tail
    ("cfg5", "ffma_channel"),
    ("cfg5", "tile_moments"),      # default: warp-per-subcarrier moments kernel
    ("cfg5", "untiled_cg"),        # default: register-tiled block CG (8 systems per warp)
    ("cfg1", "split_small"),       # default: fused U <= 16 detector, one warp per subcarrier
])
def test_kernel_variants_agree(gpu_ctx, checker, name, policy):
    """Every kernel variant gives the default's results within the north_star
    contract elementwise (|a - b| <= 1e-4 + 1e-3 |b|, hard bits equal where
    |LLR| >= 1e-4), and the default matches the oracle on a subsample."""
    cfg = get_config(name).scaled(400)
    H, Y = gen(gpu_ctx, cfg)
    if cfg.kind == "both":
        T = gpu_ctx.generate_symbols(cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits)
        call = lambda: gpu_ctx.detect_precode_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits,
                                                 cfg.K, cfg.tracker, T, cfg.rho_d, cfg.K)
    else:
        call = lambda: gpu_ctx.detect_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,
                                         cfg.tracker)
    a = call()
    torch.cuda.synchronize()
    l0 = gpu_ctx.kernel_launches
    gpu_ctx.set_kernel_policy(policy)
    try:
        b = call()
        torch.cuda.synchronize()
    finally:
        gpu_ctx.set_kernel_policy("auto")
    assert gpu_ctx.kernel_launches > l0
    assert_contract(a, b, f"{name} {policy}")
    idx = np.random.default_rng(5).choice(cfg.n_sc, size=6, replace=False)
    want = checker.detect(H[idx].cpu().numpy(), Y[idx].cpu().numpy(), cfg.rho_u, cfg.n0, cfg.es,
                          cfg.qam_bits, cfg.K, cfg.tracker, threads=8)
    got = {k: v[idx].cpu().numpy() for k, v in a.items() if k in ("xhat", "mu", "rho", "llr", "status")}
    check_detect(got, want, name + " default")


@pytest.mark.parametrize("U,B,S,K,misalign", [
    (16, 128, 1, 3, False), (8, 64, 3, 4, False), (5, 30, 2, 2, False), (13, 96, 4, 5, False),
    (12, 200, 2, 3, False),  # B > 128: four 64-antenna chunks (the last one short), q held 16 per lane
    (16, 512, 1, 2, False),  # the largest B of the fused kernel
    (16, 128, 2, 3, True),   # H_d 8 bytes off 16-byte alignment: plain copies instead of cp.async
    (7, 70, 3, 4, True),
])
def test_fused_small_precoder_matches_split_and_oracle(gpu_ctx, checker, U, B, S, K, misalign):
    """The fused U <= 16 precoder (cgm_precode_small.cuh: H_d streamed in
    64-antenna chunks, one HBM read) agrees with the channel + solve pair to
    FP32 rounding and with the oracle: ragged U and B, short last chunks,
    several transmit vectors (one streamed q pass each), misaligned H_d."""
    g = torch.Generator().manual_seed(100 + U)
    n_sc = 300
    Hd = torch.complex(torch.randn(n_sc, U, B, generator=g), torch.randn(n_sc, U, B, generator=g))
    T = torch.complex(torch.randn(n_sc, S, U, generator=g), torch.randn(n_sc, S, U, generator=g))
    Hd, T = (Hd / 2 ** 0.5).cuda(), (T / 2 ** 0.5).cuda()
    if misalign:
        flat = torch.empty(Hd.numel() + 1, dtype=Hd.dtype, device=Hd.device)
        flat[1:] = Hd.reshape(-1)
        Hd = flat[1:].view(n_sc, U, B)
        assert Hd.data_ptr() % 16 == 8
    T[7] = 0  # zero transmit vectors: zero_input status, gain 0
    l0 = gpu_ctx.kernel_launches
    a = gpu_ctx.precode_cg(Hd, T, 0.625, K)
    torch.cuda.synchronize()
    assert gpu_ctx.kernel_launches - l0 == 1  # one fused launch
    gpu_ctx.set_kernel_policy("split_small")
    try:
        b = gpu_ctx.precode_cg(Hd, T, 0.625, K)
        torch.cuda.synchronize()
    finally:
        gpu_ctx.set_kernel_policy("auto")
    assert torch.equal(a["status"], b["status"])
    assert int(a["status"][7].min()) == 2
    for k in ("q", "s", "gain"):
        d = float((a[k] - b[k]).abs().max() / b[k].abs().max())
        assert d < 2e-5, (k, d)
    idx = np.arange(0, n_sc, 37)
    want = checker.precode(Hd[idx].cpu().numpy(), T[idx].cpu().numpy(), 0.625, K, threads=8)
    check_precode({k: v[idx].cpu().numpy() for k, v in a.items()}, want, f"fused U={U} B={B}")


@pytest.mark.parametrize("B,U,S,K,tracker,bits", [
    (40, 20, 3, 3, "approx", 4),   # U in 17..31: pairs kernel with padded lanes
    (40, 20, 3, 3, "exact", 4),    # exact pairs kernel, odd S
    (64, 27, 1, 6, "exact", 6),
    (96, 31, 2, 5, "approx", 6),
    (33, 13, 5, 4, "exact", 4),    # fused U <= 16 kernel, odd B (no bulk copies)
    (48, 3, 7, 2, "exact", 2),     # several systems per warp group, QPSK
    (50, 16, 4, 8, "approx", 6),
    (96, 64, 3, 4, "exact", 4),    # U = 64 tensor-core channel: 32-antenna k-blocks, odd S
    (160, 64, 7, 3, "approx", 6),
    (64, 64, 32, 2, "approx", 2),  # the largest S of the U = 64 tensor-core path (N = 192)
    (64, 32, 2, 3, "approx", 4),   # tiled approximate block CG (block32a): one warp, 2 of 8 system slots
    (64, 32, 9, 4, "approx", 6),   # two warps, the second with one system
    (64, 32, 37, 3, "approx", 4),  # more than 32 vectors: the CTA's warps take a second round
])
def test_ragged_shapes_match_oracle(gpu_ctx, checker, B, U, S, K, tracker, bits):
    """Ragged U (between the kernels' row widths), odd B and S, several
    systems per subcarrier: the default kernels against the oracle."""
    g = torch.Generator().manual_seed(B * 100 + U)
    n_sc = 50
    H = torch.complex(torch.randn(n_sc, B, U, generator=g), torch.randn(n_sc, B, U, generator=g))
    Y = torch.complex(torch.randn(n_sc, B, S, generator=g), torch.randn(n_sc, B, S, generator=g))
    H, Y = (H / 2 ** 0.5).cuda(), (Y * 2.0).cuda()
    n0 = 0.3 * U / B
    out = gpu_ctx.detect_cg(H, Y, 1.0 / n0, n0, 1.0, bits, K, tracker)
    torch.cuda.synchronize()
    want = checker.detect(H.cpu().numpy(), Y.cpu().numpy(), 1.0 / n0, n0, 1.0, bits, K, tracker,
                          threads=8)
    check_detect({k: v.cpu().numpy() for k, v in out.items()}, want,
                 f"B={B} U={U} S={S} K={K} {tracker}")


@pytest.mark.parametrize("U,tracker", [(8, "exact"), (8, "approx"), (32, "approx"), (32, "exact"),
                                       (20, "exact"), (64, "exact")])
def test_uplink_breakdown_flagged_per_instance_every_kernel(gpu_ctx, U, tracker):
    """Curvature below 1e-30 (solvers.cpp:55-57) in one subcarrier: its
    vectors are flagged (status 1) with zeroed outputs, the neighbours are
    untouched -- through each uplink kernel family (fused U <= 16, U = 32
    pairs, U = 64 lane-per-row)."""
    g = torch.Generator().manual_seed(U)
    n_sc, B, S = 5, 2 * U + 16, 3
    H = torch.complex(torch.randn(n_sc, B, U, generator=g), torch.randn(n_sc, B, U, generator=g))
    Y = torch.complex(torch.randn(n_sc, B, S, generator=g), torch.randn(n_sc, B, S, generator=g))
    H[2] *= 1e-10  # p^H A p ~ 1e-40 with rho^-1 = 1e-35: breakdown, while r0 != 0
    H, Y = H.cuda(), Y.cuda()
    out = gpu_ctx.detect_cg(H, Y, 1e35, 1.0, 1.0, 4, 3, tracker)
    torch.cuda.synchronize()
    st = out["status"].cpu()
    assert (st[2] == 1).all(), st
    assert (st[[0, 1, 3, 4]] == 0).all(), st
    for k in ("xhat", "mu", "rho", "llr"):
        assert float(out[k][2].abs().max()) == 0.0, k
        assert float(out[k][[0, 1, 3, 4]].abs().max()) > 0.0, k


@pytest.mark.parametrize("U,tracker", [(32, "approx"), (32, "exact"), (12, "exact"), (64, "approx")])
def test_zero_observation_every_kernel(gpu_ctx, U, tracker):
    """y = 0 gives x_hat = 0 and LLR exactly 0 on the sign bits (16-QAM bits
    0 and 2; test_detect.cpp:406-422), status 0 (frozen, not broken), through
    each uplink kernel family."""
    g = torch.Generator().manual_seed(7 + U)
    n_sc, B, S = 4, 2 * U + 8, 2
    H = torch.complex(torch.randn(n_sc, B, U, generator=g), torch.randn(n_sc, B, U, generator=g))
    Y = torch.zeros(n_sc, B, S, dtype=torch.complex64)
    out = gpu_ctx.detect_cg(H.cuda(), Y.cuda(), 3.0, 0.3, 1.0, 4, 3, tracker)
    torch.cuda.synchronize()
    assert int(out["status"].sum()) == 0
    assert float(out["xhat"].abs().max()) == 0.0
    llr = out["llr"].cpu()
    assert float(llr[..., 0].abs().max()) == 0.0 and float(llr[..., 2].abs().max()) == 0.0


@pytest.mark.parametrize("name", ["cfg5", "cfg2"])
def test_host_generator_matches_device(gpu_ctx, oracle_ref, name):
    """The CPU baseline times the GPU arm's own inputs: the device generator
    and the host re-draw with the reference Rng (oracle ref_gen_uplink) give
    the same complex64 values (to the last ulp of the FP64 libm calls)."""
    cfg = get_config(name)
    n = 6
    H, Y = gen(gpu_ctx, cfg, sc0=3, n_sc=n)
    T = gpu_ctx.generate_symbols(cfg.U, n, cfg.S, cfg.seed, cfg.qam_bits, sc0=3)
    torch.cuda.synchronize()
    rs = cfg.rsqrt()
    Hh, Yh, Th = oracle_ref.gen_uplink(cfg.seed, cfg.B, cfg.U, 3, n, cfg.S, cfg.qam_bits, cfg.n0,
                                       rsqrt=None if rs is None else rs.astype(np.float32),
                                       with_t=True, threads=4)
    # FP64 sums rounded to complex64: equal up to one rounding of the sum
    h = H.cpu().numpy()
    np.testing.assert_allclose(h, Hh, rtol=0, atol=2e-7 * float(np.abs(Hh).max()))
    assert np.mean(h == Hh) > 0.99
    y, yh = Y.cpu().numpy(), Yh
    np.testing.assert_allclose(y, yh, rtol=0, atol=2e-7 * float(np.abs(yh).max()))
    assert np.mean(y == yh) > 0.99
    np.testing.assert_array_equal(T.cpu().numpy(), Th)


@pytest.mark.parametrize("name", ["cfg4a_K4", "cfg4b_K2", "cfg5", "cfg1", "cfg2"])
def test_partial_output_requests_match_full(gpu_ctx, name):
    """Any subset of the outputs may be requested (NULL pointers for the
    rest): the results do not depend on which other outputs exist -- the
    exact tracker's extraction reads v_K and the breakdown flags from its
    own state, never from the caller's buffers."""
    cfg = get_config(name).scaled(64)
    H, Y = gen(gpu_ctx, cfg)
    full = run(gpu_ctx, cfg, H, Y)
    for want in (("llr",), ("llr", "mu"), ("rho",), ("xhat", "status")):
        part = gpu_ctx.detect_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,
                                 cfg.tracker, want=want)
        torch.cuda.synchronize()
        assert set(part) == set(want)
        for k in want:
            assert torch.equal(part[k], full[k]), (name, want, k)


@pytest.mark.parametrize("name", ["cfg5", "cfg4a_K4", "cfg2"])
def test_multi_chunk_two_stream_path_bitwise(name):
    """A small workspace budget (CGMIMO_CHUNK_MB, read at context creation)
    splits the call into several chunks that alternate two streams and two
    workspace halves; the results equal the one-chunk call and the serial
    chunk order bit for bit (every subcarrier's computation is independent of
    the chunking)."""
    import os

    from paper_1404_0424_b200 import Context

    cfg = get_config(name).scaled(700)
    old = os.environ.get("CGMIMO_CHUNK_MB")
    os.environ["CGMIMO_CHUNK_MB"] = "12"
    try:
        small = Context(0)
    finally:
        if old is None:
            del os.environ["CGMIMO_CHUNK_MB"]
        else:
            os.environ["CGMIMO_CHUNK_MB"] = old
    big = Context(0)
    rs = cfg.rsqrt()
    rs = None if rs is None else torch.tensor(rs)
    H, Y = big.generate_uplink(cfg.B, cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits, cfg.n0,
                               rsqrt=rs)
    T = big.generate_symbols(cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits)

    def run(ctx):
        if cfg.kind == "both":
            return ctx.detect_precode_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,
                                         cfg.tracker, T, cfg.rho_d, cfg.K)
        return ctx.detect_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K, cfg.tracker)

    want = run(big)
    l0 = small.kernel_launches
    got = run(small)
    torch.cuda.synchronize()
    assert small.kernel_launches - l0 >= 4, "expected several chunks"
    small.set_kernel_policy("serial_chunks")
    ser = run(small)
    torch.cuda.synchronize()
    for k in want:
        assert torch.equal(got[k], want[k]), (name, k)
        assert torch.equal(ser[k], want[k]), (name, k)


def test_cfg5_path_degenerate_inputs_match_oracle(gpu_ctx, checker):
    """The headline detect + precode path (block CG, moment extraction, TMA
    precoder) on degenerate inputs, against the reference: a subcarrier whose
    transmit vectors are all zero and one zero vector elsewhere (zero_input:
    status 2, gain 0, q = s = 0; precode.cpp:22-36), a subcarrier with zero
    observations (x_hat = 0, frozen CG), and ordinary neighbours."""
    cfg = get_config("cfg5").scaled(40)
    H, Y = gen(gpu_ctx, cfg)
    T = gpu_ctx.generate_symbols(cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits)
    T[3] = 0
    T[5, 2] = 0
    Y[4] = 0
    got = gpu_ctx.detect_precode_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,
                                    cfg.tracker, T, cfg.rho_d, cfg.K)
    torch.cuda.synchronize()
    assert int(got["pstatus"][3].min()) == 2 and int(got["pstatus"][5, 2]) == 2
    assert float(got["gain"][3].abs().max()) == 0.0 and float(got["s"][3].abs().max()) == 0.0
    assert float(got["xhat"][4].abs().max()) == 0.0
    h = H.cpu().numpy()
    want = checker.detect(h, Y.cpu().numpy(), cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,
                          cfg.tracker, threads=8)
    check_detect({k: got[k].cpu().numpy() for k in ("xhat", "mu", "rho", "llr", "status")}, want,
                 "cfg5 degenerate uplink")
    wantd = checker.precode(np.conj(np.transpose(h, (0, 2, 1))), T.cpu().numpy(), cfg.rho_d,
                            cfg.K, threads=8)
    check_precode({"q": got["q"].cpu().numpy(), "s": got["s"].cpu().numpy(),
                   "gain": got["gain"].cpu().numpy(), "status": got["pstatus"].cpu().numpy()},
                  wantd, "cfg5 degenerate downlink")
