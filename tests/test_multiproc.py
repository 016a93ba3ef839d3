"""Multi-process (gloo, world size 2, CPU) coverage of the N-sharded path's host logic:
column slabs on whole samples, replicated-plan digests, max-over-ranks timing reduction,
and that the concatenation of per-rank slab results equals the unsharded oracle result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2008_11849_b200.shard import shard_columns


def test_shard_columns_cover_and_balance():
    for n, w, u in [(50176, 8, 196), (50176, 3, 196), (25088, 2, 3136), (49, 4, 49), (1000, 7, 1)]:
        ranges = [shard_columns(n, w, r, u) for r in range(w)]
        assert ranges[0][0] == 0 and ranges[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        assert all((b - a) % u == 0 for a, b in ranges)
        sizes = [(b - a) // u for a, b in ranges]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_columns(100, 2, 0, 7)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2008_11849_b200 as srt
        from synth import gen
        M, K, N, unit = 96, 200, 7 * 49, 49  # 7 samples over 2 ranks: uneven slabs
        w = gen.pruned_weights(M, K, 90, seed=5)
        X = gen.uniform_x(K, N, seed=6).astype(np.float64)
        # replicated plan: identical digests on every rank
        plan = srt.Plan.from_csr(w, n_hint=N, device=srt.SPARSE_DEVICE_HOST_ONLY)
        digs = [None] * world
        dist.all_gather_object(digs, int(plan.info["digest"]))
        # each rank computes its slab (oracle stands in for the executor on CPU)
        n0, n1 = shard_columns(N, world, rank, unit)
        y = oracle.spmm(M, K, w.row_ptr, w.col_idx, w.values.astype(np.float64),
                        np.ascontiguousarray(X[:, n0:n1]))
        parts = [None] * world
        dist.all_gather_object(parts, y)
        from paper_2008_11849_b200.shard import gather_columns
        gathered = gather_columns(torch.from_numpy(y), N, world, unit).numpy()
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            full = oracle.spmm(M, K, w.row_ptr, w.col_idx, w.values.astype(np.float64), X)
            out.put((len(set(digs)) == 1, bool(np.array_equal(np.concatenate(parts, axis=1), full))
                     and bool(np.array_equal(gathered, full)), float(t.item())))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_sharded_equals_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    same_digest, equal, tmax = q.get(timeout=10)
    assert same_digest and equal and tmax == 2.0
