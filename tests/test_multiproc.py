"""CPU, world_size 2 over gloo: the multi-GPU plumbing (subcarrier shards +
the single gather of LLRs to rank 0) reproduces the unsharded result.  The
per-rank compute here is the CPU oracle standing in for the GPU kernels."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(n_sc, B=16, U=4, S=3):
    sys.path.insert(0, ROOT)
    import oracle

    o = oracle.Oracle("port")
    H = np.stack([o.rayleigh(11, [2, sc], B, U) for sc in range(n_sc)]).astype(np.complex64)
    Y = np.stack([o.rayleigh(11, [3, sc], B, S) for sc in range(n_sc)]).astype(np.complex64)
    return o, H, Y


def _worker(rank, world, port, n_sc, outq):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1404_0424_b200.parallel import gather_to_root, shard_range

    o, H, Y = _inputs(n_sc)
    a, b = shard_range(n_sc, rank, world)
    r = o.detect(H[a:b], Y[a:b], 2.0, 0.5, 1.0, 4, 3, "exact")
    local = torch.from_numpy(r["llr"].astype(np.float32).reshape(-1))
    got = gather_to_root(local, world, rank)
    if rank == 0:
        outq.put(got.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_sc", [6, 5])
def test_two_rank_shard_and_gather_equals_single(n_sc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_sc, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    o, H, Y = _inputs(n_sc)
    want = o.detect(H, Y, 2.0, 0.5, 1.0, 4, 3, "exact")["llr"].astype(np.float32).reshape(-1)
    assert np.array_equal(got, want)


# --------------------------------------------- sharded BLER sweeps (sim.py)
def _fake_trials(first, count):
    """Deterministic stand-in for cgm_sweep_trials: errors and breakdowns as
    functions of the trial index only (as real trials are of their keys)."""
    t = np.arange(first, first + count)
    return ((t * 7919) % 5).astype(np.uint32), ((t % 13) == 4).astype(np.uint8)


def _sweep_worker(rank, world, port, cfgs, outq):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1404_0424_b200 import sim

    res = []
    for kw in cfgs:
        cfg = sim.SweepConfig(**kw)
        res.append(sim._fold_point(_fake_trials, cfg, 10.0, batch=7, group=dist.group.WORLD))
    outq.put((rank, [(p.frames, p.block_errors, p.breakdowns, p.trials_run) for p in res]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_sweep_point_equals_single():
    """Trials split over 2 ranks (contiguous blocks, all_gather, in-order fold)
    give the single-process SnrPointResult, with and without the early stop."""
    sys.path.insert(0, ROOT)
    from paper_1404_0424_b200 import sim

    cfgs = [dict(trials=50, max_breakdown_fraction=1.0), dict(trials=49, max_breakdown_fraction=1.0,
                                                            max_block_errors=33),
            dict(trials=3, max_breakdown_fraction=1.0)]
    want = []
    for kw in cfgs:
        p = sim._fold_point(_fake_trials, sim.SweepConfig(**kw), 10.0, batch=7)
        want.append((p.frames, p.block_errors, p.breakdowns, p.trials_run))
    assert want[1][3] < 49  # the early stop fired
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sweep_worker, args=(r, 2, port, cfgs, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert got[0] == want and got[1] == want


# ------------------------- chunked sharded detect + precode with the q/s gather
def _both_inputs(n_sc, B=16, U=4, S=3):
    sys.path.insert(0, ROOT)
    import oracle

    o = oracle.Oracle("port")
    H = np.stack([o.rayleigh(13, [2, sc], B, U) for sc in range(n_sc)]).astype(np.complex64)
    Y = np.stack([o.rayleigh(13, [3, sc], B, S) for sc in range(n_sc)]).astype(np.complex64)
    T = np.stack([o.rayleigh(13, [5, sc], S, U) for sc in range(n_sc)]).astype(np.complex64)
    return o, H, Y, T


def _both_compute(o, H, Y, T):
    """The per-chunk hot path (the CPU oracle standing in for the GPU kernels):
    detect_cg on (H, Y) and precode_cg on (H^H, T), as detect_precode_cg does."""
    d = o.detect(H, Y, 2.0, 0.5, 1.0, 4, 3, "exact")
    p = o.precode(np.conj(np.transpose(H, (0, 2, 1))), T, 3.0, 3)
    return {"llr": d["llr"].astype(np.float32), "status": d["status"],
            "q": p["q"].astype(np.complex64), "s": p["s"].astype(np.complex64),
            "gain": p["gain"].astype(np.float32), "pstatus": p["status"]}


_SPEC = {"llr": ((3, 4, 4), torch.float32), "status": ((3,), torch.uint8),
         "q": ((3, 16), torch.complex64), "s": ((3, 16), torch.complex64),
         "gain": ((3,), torch.float32), "pstatus": ((3,), torch.uint8)}


def _pipeline_worker(rank, world, port, n_sc, n_chunks, outq):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1404_0424_b200.parallel import ShardedPipeline, TorchTransport

    o, H, Y, T = _both_inputs(n_sc)
    pipe = ShardedPipeline(n_sc, rank, world, _SPEC, TorchTransport(rank, world),
                           n_chunks=n_chunks)
    calls = []

    def compute(a, b, views):
        lo = pipe.lo
        calls.append((a, b))
        r = _both_compute(o, H[lo + a:lo + b], Y[lo + a:lo + b], T[lo + a:lo + b])
        for k, v in views.items():
            v.copy_(torch.from_numpy(r[k]))

    res = pipe.run(compute)
    # every local subcarrier computed exactly once, in order
    assert [x for a, b in calls for x in range(a, b)] == list(range(pipe.n_local))
    if rank == 0:
        outq.put({k: v.numpy().copy() for k, v in res.items()})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_sc,n_chunks", [(7, 3), (4, 3), (9, 1)])
def test_two_rank_chunked_pipeline_gathers_llr_and_precoded_vectors(n_sc, n_chunks):
    """Strong-scaling shard (cfg5's split), chunked, with the gather of LLRs
    AND the precoded vectors q, s (and gains, status bytes) to rank 0 chunk by
    chunk: rank 0 ends with exactly the unsharded outputs.  Ragged shards
    (n_sc = 7) and empty chunks (n_sc = 4 over 2 ranks x 3 chunks) included."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pipeline_worker, args=(r, 2, port, n_sc, n_chunks, q))
             for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=180)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    o, H, Y, T = _both_inputs(n_sc)
    want = _both_compute(o, H, Y, T)
    for k in _SPEC:
        assert np.array_equal(got[k], want[k]), k


def test_gather_layout_covers_every_subcarrier_once():
    """The chunk layouts of all ranks tile [0, n_sc) exactly (pure host logic)."""
    sys.path.insert(0, ROOT)
    from paper_1404_0424_b200.parallel import ShardedPipeline

    class _Null:
        def gatherv(self, *a, **k):
            pass

    for n_sc, world, n_chunks in [(65536, 8, 4), (65536, 3, 5), (10, 4, 3), (3, 4, 2)]:
        seen = np.zeros(n_sc, np.int64)
        for r in range(world):
            p = ShardedPipeline(n_sc, r, world, {"x": ((1,), torch.uint8)}, _Null(),
                                n_chunks=n_chunks)
            for c in range(n_chunks):
                counts, displs = p.gather_layout(c, 1)
                a, b = p.chunk_range(r, c)
                assert counts[r] == b - a and displs[r] == p.lo + a
                seen[displs[r]:displs[r] + counts[r]] += 1
        assert (seen == 1).all(), (n_sc, world, n_chunks)
