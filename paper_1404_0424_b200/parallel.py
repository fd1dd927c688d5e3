"""Multi-GPU sharding of the detection / precoding path.

Subcarriers are independent: each rank owns a
contiguous block of subcarriers with all S vectors of a subcarrier on the
same rank (so its Gram matrix is shared) and runs the fused kernel on it
with no data-path collective.  The only exchange is the final gather of
LLRs / precoded vectors to rank 0 (NCCL over NVLink on GPUs, gloo on CPU
in the tests).  Inputs are generated from subcarrier-indexed RNG streams,
so per-instance results do not depend on the number of ranks.
"""
from __future__ import annotations


def shard_range(n_sc: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, stop) block of subcarriers for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(n_sc, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def gather_to_root(t, world: int, rank: int, sizes=None):
    """Gather every rank's tensor `t` (1-D, same dtype) to rank 0; returns the
    concatenation on rank 0 and None elsewhere.  Uneven shards are padded to
    the largest size for the collective and trimmed after."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return t
    if sizes is None:
        n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
        all_n = [torch.zeros_like(n) for _ in range(world)]
        dist.all_gather(all_n, n)
        sizes = [int(x.item()) for x in all_n]
    m = max(sizes)
    src = t if t.numel() == m else torch.cat([t, t.new_zeros(m - t.numel())])
    if rank == 0:
        bufs = [torch.empty(m, dtype=t.dtype, device=t.device) for _ in range(world)]
        dist.gather(src, gather_list=bufs, dst=0)
        return torch.cat([b[:s] for b, s in zip(bufs, sizes)])
    dist.gather(src, dst=0)
    return None


class Comm:
    """The C ABI's NCCL communicator (cgm_comm_create / cgm_gather): the same
    gather as gather_to_root, callable from any FFI without torch.distributed.
    Rank 0 makes the id with ``Comm.unique_id()`` and ships its 128 bytes to
    the other ranks out of band."""

    def __init__(self, ctx, nranks: int, rank: int, uid: bytes):
        import ctypes as C

        self.ctx, self.lib, self.rank, self.nranks = ctx, ctx.lib, rank, nranks
        h = C.c_void_p()
        ctx._check(self.lib.cgm_comm_create(ctx.h, nranks, rank, bytes(uid), C.byref(h)))
        self.h = h

    @staticmethod
    def unique_id() -> bytes:
        import ctypes as C
        from . import _lib

        buf = C.create_string_buffer(128)
        rc = _lib.load().cgm_comm_unique_id(buf)
        if rc != _lib.CGM_OK:
            raise RuntimeError(f"cgm_comm_unique_id rc={rc} (NCCL not available?)")
        return buf.raw

    def gather(self, send, counts_bytes, recv=None, root: int = 0):
        """Concatenate every rank's device buffer `send` (counts_bytes[r] bytes
        on rank r) on `root` into the device tensor `recv`, rank order."""
        import ctypes as C

        self.ctx._bind_torch_stream()
        cnt = (C.c_size_t * self.nranks)(*[int(c) for c in counts_bytes])
        self.ctx._check(self.lib.cgm_gather(self.ctx.h, self.h, C.c_void_p(send.data_ptr()), cnt,
                                            C.c_void_p(recv.data_ptr() if recv is not None else 0),
                                            root))
        return recv

    def close(self):
        if getattr(self, "h", None):
            self.lib.cgm_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


def sharded_detect(ctx, cfg, world: int, rank: int, gather: bool = True):
    """Generate this rank's shard of `cfg` on its GPU, detect it, and (optionally)
    gather LLRs to rank 0.  Returns (local outputs, gathered LLRs or None)."""
    import torch

    s0, s1 = shard_range(cfg.n_sc, rank, world)
    rs = cfg.rsqrt()
    rs = None if rs is None else torch.tensor(rs)
    H, Y = ctx.generate_uplink(cfg.B, cfg.U, s1 - s0, cfg.S, cfg.seed, cfg.qam_bits, cfg.n0,
                               sc0=s0, rsqrt=rs)
    out = ctx.detect_cg(H, Y, cfg.rho_u, cfg.n0, cfg.es, cfg.qam_bits, cfg.K, cfg.tracker)
    torch.cuda.synchronize()
    g = None
    if gather:
        sizes = [(b - a) * cfg.S * cfg.U * cfg.qam_bits
                 for a, b in (shard_range(cfg.n_sc, r, world) for r in range(world))]
        g = gather_to_root(out["llr"].reshape(-1), world, rank, sizes)
    return out, g
