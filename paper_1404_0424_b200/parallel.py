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


class NcclTransport:
    """Chunk gathers through the product C ABI (cgm_gatherv over NCCL, on the
    current torch stream of the context's device)."""

    def __init__(self, comm: "Comm"):
        self.comm = comm

    def gatherv(self, send, counts_bytes, displs_bytes, recv, root: int = 0):
        import ctypes as C

        n = self.comm.nranks
        ctx = self.comm.ctx
        ctx._bind_torch_stream()
        cnt = (C.c_size_t * n)(*[int(c) for c in counts_bytes])
        dsp = (C.c_size_t * n)(*[int(d) for d in displs_bytes])
        ctx._check(self.comm.lib.cgm_gatherv(
            ctx.h, self.comm.h, C.c_void_p(send.data_ptr() if send.numel() else 0), cnt, dsp,
            C.c_void_p(recv.data_ptr() if recv is not None else 0), root))


class TorchTransport:
    """The same chunk gathers over torch.distributed point-to-point (gloo on
    CPU for the multi-process tests; any backend works)."""

    def __init__(self, rank: int, world: int):
        self.rank, self.world = rank, world

    def gatherv(self, send, counts_bytes, displs_bytes, recv, root: int = 0):
        import torch.distributed as dist

        sb = send.reshape(-1).view(_u8())
        if self.rank == root:
            rb = recv.reshape(-1).view(_u8())
            for r in range(self.world):
                c, d = int(counts_bytes[r]), int(displs_bytes[r])
                if c == 0:
                    continue
                if r == root:
                    if rb[d:d + c].data_ptr() != sb.data_ptr():
                        rb[d:d + c].copy_(sb[:c])
                else:
                    dist.recv(rb[d:d + c], src=r)
        elif int(counts_bytes[self.rank]) > 0:
            dist.send(sb, dst=root)


def _u8():
    import torch

    return torch.uint8


class ShardedPipeline:
    """One rank's share of a strong-scaling sharded job (SURVEY.md 8(e),
    BASELINE configs[4]: n_sc subcarriers split evenly over the ranks), run
    in ``n_chunks`` chunks of its contiguous shard; chunk c's outputs are
    gathered to ``root`` while chunk c + 1 is computed.

    * ``compute(lo, hi, views)`` runs the hot path on the rank's local
      subcarriers [lo, hi) and writes into ``views`` (a dict of output
      tensors sliced to those subcarriers) -- on GPUs it launches on the
      current (compute) stream;
    * ``outputs`` maps an output name to its per-subcarrier shape and dtype;
      each gathered output is one whole-job tensor on the root, filled in
      place: the root computes its own shard straight into it (nothing to
      copy) and rank r's chunk c lands at subcarrier shard_lo(r) +
      chunk_lo(r, c) through one cgm_gatherv per output;
    * on CUDA the gathers run on a separate stream that waits on an event
      recorded after the chunk's compute, so the NVLink transfer of chunk c
      overlaps the kernels of chunk c + 1; on CPU (the gloo tests) the same
      schedule runs in program order.

    Every rank derives every other rank's chunk boundaries from (n_sc,
    world, n_chunks) alone, so the gather needs no size exchange."""

    def __init__(self, n_sc: int, rank: int, world: int, outputs: dict, transport,
                 n_chunks: int = 4, root: int = 0, device=None):
        import torch

        self.n_sc, self.rank, self.world, self.root = n_sc, rank, world, root
        self.transport = transport
        self.n_chunks = max(1, int(n_chunks))
        self.device = device
        self.lo, self.hi = shard_range(n_sc, rank, world)
        self.n_local = self.hi - self.lo
        self.specs = {k: (tuple(shape), dtype) for k, (shape, dtype) in outputs.items()}
        # whole-job buffers on the root, the local shard elsewhere
        self.full = {}
        self.local = {}
        for k, (shape, dtype) in self.specs.items():
            if rank == root:
                self.full[k] = torch.empty((n_sc, *shape), dtype=dtype, device=device)
                self.local[k] = self.full[k][self.lo:self.hi]
            else:
                self.local[k] = torch.empty((self.n_local, *shape), dtype=dtype, device=device)
        self.cuda = device is not None and torch.device(device).type == "cuda"
        if self.cuda:
            self.comm_stream = torch.cuda.Stream(device)

    def chunk_range(self, rank: int, c: int) -> tuple[int, int]:
        """Local subcarrier range [a, b) of `rank`'s chunk c."""
        lo, hi = shard_range(self.n_sc, rank, self.world)
        a, b = shard_range(hi - lo, c, self.n_chunks)
        return a, b

    def gather_layout(self, c: int, per_sc_bytes: int):
        """(counts, displs) in bytes of chunk c over all ranks for an output
        of `per_sc_bytes` per subcarrier."""
        counts, displs = [], []
        for r in range(self.world):
            lo, _ = shard_range(self.n_sc, r, self.world)
            a, b = self.chunk_range(r, c)
            counts.append((b - a) * per_sc_bytes)
            displs.append((lo + a) * per_sc_bytes)
        return counts, displs

    def _gather_chunk(self, c: int):
        import math

        a, b = self.chunk_range(self.rank, c)
        for k, (shape, dtype) in self.specs.items():
            per = math.prod(shape) * self.local[k].element_size()
            counts, displs = self.gather_layout(c, per)
            send = self.local[k][a:b]
            self.transport.gatherv(send, counts, displs,
                                   self.full.get(k) if self.rank == self.root else None, self.root)

    def run(self, compute, gather: bool = True):
        """Compute the whole shard chunk by chunk (and gather it); returns the
        whole-job outputs on the root, the local shard elsewhere."""
        import torch

        if not self.cuda:
            for c in range(self.n_chunks):
                a, b = self.chunk_range(self.rank, c)
                if b > a:
                    compute(a, b, {k: v[a:b] for k, v in self.local.items()})
                if gather and self.world > 1:
                    self._gather_chunk(c)
            return self.full if self.rank == self.root else self.local
        cs = torch.cuda.current_stream(self.device)
        self.comm_stream.wait_stream(cs)  # the previous run's readers of the buffers
        for c in range(self.n_chunks):
            a, b = self.chunk_range(self.rank, c)
            if b > a:
                compute(a, b, {k: v[a:b] for k, v in self.local.items()})
            if gather and self.world > 1:
                ev = torch.cuda.Event()
                ev.record(cs)
                with torch.cuda.stream(self.comm_stream):
                    self.comm_stream.wait_event(ev)
                    self._gather_chunk(c)
        if gather and self.world > 1:
            cs.wait_stream(self.comm_stream)  # outputs complete on the caller's stream
        return self.full if self.rank == self.root else self.local


def detect_precode_outputs(cfg, which=("llr", "q", "s", "gain", "status", "pstatus")):
    """Per-subcarrier shapes / dtypes of detect_precode_cg's outputs that the
    sharded job gathers (north_star: the LLRs and the precoded vectors)."""
    import torch

    S, U, B = cfg.S, cfg.U, cfg.B
    spec = {"xhat": ((S, U), torch.complex64), "mu": ((S, U), torch.float32),
            "rho": ((S, U), torch.float32), "llr": ((S, U, cfg.qam_bits), torch.float32),
            "status": ((S,), torch.uint8), "q": ((S, B), torch.complex64),
            "s": ((S, B), torch.complex64), "gain": ((S,), torch.float32),
            "pstatus": ((S,), torch.uint8)}
    return {k: spec[k] for k in which}


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
