"""GPU parity: the CUDA path through the C ABI vs the FP64 oracle (the
reference library itself when built, else the C restatement) on identical
seeded complex64 inputs, for every BASELINE config at a subsampled size."""
import numpy as np
import pytest
import torch

from paper_1404_0424_b200 import get_config
from parity import check_detect, check_precode

pytestmark = pytest.mark.gpu

# (config, subcarriers checked against the oracle)
UPLINK = [("cfg1", 512), ("cfg2", 96), ("cfg4a_K2", 96), ("cfg4a_K4", 96), ("cfg4a_K8", 96),
          ("cfg4b_K2", 24), ("cfg4b_K4", 24), ("cfg4b_K8", 24)]


def to_np(t):
    return t.detach().cpu().numpy()


def gen_uplink(ctx, cfg, sc0=0):
    rs = cfg.rsqrt()
    rs = None if rs is None else torch.tensor(rs)
    H, Y = ctx.generate_uplink(cfg.B, cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits, cfg.n0,
                               sc0=sc0, rsqrt=rs)
    torch.cuda.synchronize()
    return H, Y


def run_uplink(ctx, cfg, H, Y):
    out = ctx.detect_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K, cfg.tracker)
    torch.cuda.synchronize()
    return {k: to_np(v) for k, v in out.items()}


@pytest.fixture(params=["auto", "ffma_channel+split_small+lane_solve"])
def policy_ctx(gpu_ctx, request):
    """The production kernels (auto) and every A/B alternative at once (FFMA
    channel kernel, split path for U <= 16, lane-per-row solve kernel)."""
    gpu_ctx.set_kernel_policy(request.param)
    yield gpu_ctx
    gpu_ctx.set_kernel_policy("auto")


@pytest.mark.parametrize("name,n_sc", UPLINK)
def test_uplink_parity(policy_ctx, checker, name, n_sc):
    gpu_ctx = policy_ctx
    cfg = get_config(name).scaled(n_sc)
    H, Y = gen_uplink(gpu_ctx, cfg)
    got = run_uplink(gpu_ctx, cfg, H, Y)
    want = checker.detect(to_np(H), to_np(Y), cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,
                          cfg.tracker, threads=8)
    check_detect(got, want, name)


def test_downlink_parity_cfg3(policy_ctx, checker):
    gpu_ctx = policy_ctx
    cfg = get_config("cfg3").scaled(1024)
    Hd, T = gpu_ctx.generate_downlink(cfg.B, cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits)
    out = gpu_ctx.precode_cg(Hd, T, cfg.rho_d, cfg.K)
    torch.cuda.synchronize()
    got = {k: to_np(v) for k, v in out.items()}
    want = checker.precode(to_np(Hd), to_np(T), cfg.rho_d, cfg.K, threads=8)
    check_precode(got, want, "cfg3")


def test_fused_parity_cfg5(policy_ctx, checker):
    gpu_ctx = policy_ctx
    cfg = get_config("cfg5").scaled(24)
    H, Y = gen_uplink(gpu_ctx, cfg)
    T = gpu_ctx.generate_symbols(cfg.U, cfg.n_sc, cfg.S, cfg.seed, cfg.qam_bits)
    out = gpu_ctx.detect_precode_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,
                                    cfg.tracker, T, cfg.rho_d, cfg.K)
    torch.cuda.synchronize()
    got = {k: to_np(v) for k, v in out.items()}
    Hn = to_np(H)
    want_u = checker.detect(Hn, to_np(Y), cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K,
                            cfg.tracker, threads=8)
    Hd = np.ascontiguousarray(np.conj(np.transpose(Hn, (0, 2, 1))))
    want_d = checker.precode(Hd, to_np(T), cfg.rho_d, cfg.K, threads=8)
    check_detect({k: got[k] for k in ("xhat", "mu", "rho", "llr", "status")}, want_u, "cfg5 uplink")
    check_precode({"q": got["q"], "s": got["s"], "gain": got["gain"], "status": got["pstatus"]},
                  want_d, "cfg5 downlink")


@pytest.mark.parametrize("S,St,K,Kt,B", [(16, 16, 4, 2, 256), (5, 3, 3, 4, 128), (13, 7, 4, 4, 256),
                                         (2, 9, 2, 5, 192), (16, 1, 6, 1, 256)])
@pytest.mark.parametrize("policy", ["auto", "untiled_cg"])
def test_detect_precode_ragged_systems(gpu_ctx, checker, S, St, K, Kt, B, policy):
    """The cfg5 path (block CG + moment extraction + TMA precoder) with system
    counts that do not fill the CG warps (8 systems per warp tiled, 4
    untiled), different uplink / downlink iteration counts and B below 256,
    against the reference."""
    cfg = get_config("cfg5")
    n_sc = 37
    H, Y = gpu_ctx.generate_uplink(B, cfg.U, n_sc, S, cfg.seed, cfg.qam_bits, cfg.n0)
    T = gpu_ctx.generate_symbols(cfg.U, n_sc, 16, cfg.seed + 1, cfg.qam_bits)[:, :St].contiguous()
    gpu_ctx.set_kernel_policy(policy)
    try:
        out = gpu_ctx.detect_precode_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, K,
                                        "exact", T, cfg.rho_d, Kt)
        torch.cuda.synchronize()
    finally:
        gpu_ctx.set_kernel_policy("auto")
    got = {k: to_np(v) for k, v in out.items()}
    Hn = to_np(H)
    want_u = checker.detect(Hn, to_np(Y), cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, K, "exact",
                            threads=8)
    Hd = np.ascontiguousarray(np.conj(np.transpose(Hn, (0, 2, 1))))
    want_d = checker.precode(Hd, to_np(T), cfg.rho_d, Kt, threads=8)
    tag = f"S{S} St{St} K{K} Kt{Kt} B{B} {policy}"
    check_detect({k: got[k] for k in ("xhat", "mu", "rho", "llr", "status")}, want_u, tag)
    check_precode({"q": got["q"], "s": got["s"], "gain": got["gain"], "status": got["pstatus"]},
                  want_d, tag)
