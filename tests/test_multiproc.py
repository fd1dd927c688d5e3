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
