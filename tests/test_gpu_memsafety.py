"""GPU memory-safety checks (compute-sanitizer is not available on this
pool): every default kernel family on small and ragged batches must

* write nothing outside its output arrays -- each output is a view in the
  middle of a larger tensor whose guard bands hold a sentinel pattern that
  must survive the call bit for bit;
* read nothing from the split-path workspace that it did not write first --
  the workspace is NaN-filled before every chunk (policy "poison_ws") and
  the outputs must equal the unpoisoned run bit for bit;
* give the same bits run to run and match the oracle (tests elsewhere)."""
import pytest
import torch

from paper_1404_0424_b200 import get_config

pytestmark = pytest.mark.gpu

GUARD = 4096  # elements on each side


def guarded(shape, dtype, dev):
    n = 1
    for s in shape:
        n *= s
    base = torch.empty(n + 2 * GUARD, dtype=dtype, device=dev)
    if dtype == torch.uint8:
        base.fill_(0xA5)
    else:
        base.view(torch.uint8).fill_(0x7B)
    view = base[GUARD:GUARD + n].view(shape)
    return base, view


def check_guards(base, n, what):
    lo, hi = base[:GUARD], base[GUARD + n:]
    if base.dtype == torch.uint8:
        ok = bool((lo == 0xA5).all()) and bool((hi == 0xA5).all())
    else:
        ok = bool((lo.view(torch.uint8) == 0x7B).all()) and bool((hi.view(torch.uint8) == 0x7B).all())
    assert ok, f"{what}: guard band overwritten"


CASES = ["cfg1", "cfg2", "cfg4a_K4", "cfg4a_K8", "cfg4b_K2", "cfg5"]


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("n_sc", [1, 37])
def test_detect_outputs_and_workspace(gpu_ctx, name, n_sc):
    cfg = get_config(name).scaled(n_sc)
    dev = torch.device("cuda", 0)
    rs = cfg.rsqrt()
    rs = None if rs is None else torch.tensor(rs)
    H, Y = gpu_ctx.generate_uplink(cfg.B, cfg.U, n_sc, cfg.S, cfg.seed, cfg.qam_bits, cfg.n0,
                                   rsqrt=rs)
    S, U, B, bits = cfg.S, cfg.U, cfg.B, cfg.qam_bits
    specs = {"xhat": ((n_sc, S, U), torch.complex64), "mu": ((n_sc, S, U), torch.float32),
             "rho": ((n_sc, S, U), torch.float32), "llr": ((n_sc, S, U, bits), torch.float32),
             "status": ((n_sc, S), torch.uint8)}
    both = cfg.kind == "both"
    if both:
        specs.update({"q": ((n_sc, S, B), torch.complex64), "s": ((n_sc, S, B), torch.complex64),
                      "gain": ((n_sc, S), torch.float32), "pstatus": ((n_sc, S), torch.uint8)})
        T = gpu_ctx.generate_symbols(U, n_sc, S, cfg.seed, bits)

    def call(policy):
        bufs = {k: guarded(shape, dt, dev) for k, (shape, dt) in specs.items()}
        out = {k: v[1] for k, v in bufs.items()}
        gpu_ctx.set_kernel_policy(policy)
        try:
            if both:
                gpu_ctx.detect_precode_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, bits, cfg.K, cfg.tracker,
                                          T, cfg.rho_d, cfg.K, out=out)
            else:
                gpu_ctx.detect_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, bits, cfg.K, cfg.tracker, out=out)
            torch.cuda.synchronize()
        finally:
            gpu_ctx.set_kernel_policy("auto")
        for k, (base, view) in bufs.items():
            check_guards(base, view.numel(), f"{name} {k}")
        return out

    a = call("auto")
    b = call("poison_ws")
    for k in a:
        assert torch.equal(a[k].view(torch.uint8) if a[k].dtype != torch.uint8 else a[k],
                           b[k].view(torch.uint8) if b[k].dtype != torch.uint8 else b[k]), (name, k)
        if a[k].is_floating_point() or a[k].is_complex():
            x = torch.view_as_real(a[k]) if a[k].is_complex() else a[k]
            assert torch.isfinite(x).all(), (name, k)


@pytest.mark.parametrize("n_sc", [1, 37])
def test_precode_outputs_guarded(gpu_ctx, n_sc):
    cfg = get_config("cfg3").scaled(n_sc)
    dev = torch.device("cuda", 0)
    Hd, T = gpu_ctx.generate_downlink(cfg.B, cfg.U, n_sc, cfg.S, cfg.seed, cfg.qam_bits)
    specs = {"q": ((n_sc, cfg.S, cfg.B), torch.complex64), "s": ((n_sc, cfg.S, cfg.B), torch.complex64),
             "gain": ((n_sc, cfg.S), torch.float32), "status": ((n_sc, cfg.S), torch.uint8)}
    for policy in ("auto", "split_small+poison_ws"):
        bufs = {k: guarded(shape, dt, dev) for k, (shape, dt) in specs.items()}
        gpu_ctx.set_kernel_policy(policy)
        try:
            gpu_ctx.precode_cg(Hd, T, cfg.rho_d, cfg.K, out={k: v[1] for k, v in bufs.items()})
            torch.cuda.synchronize()
        finally:
            gpu_ctx.set_kernel_policy("auto")
        for k, (base, view) in bufs.items():
            check_guards(base, view.numel(), f"cfg3 {policy} {k}")
