"""The library in two processes on one GPU (gloo for the host-side exchange): each rank builds
its replica of the plan, runs its whole-image shard of a conv batch and its column slab of an
SpMM through the C ABI, and the gathered result equals the single-process call bitwise (the
N-sharding of SURVEY 8(e) with a real executor, not the oracle as a stand-in)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2008_11849_b200 as srt
        from paper_2008_11849_b200.shard import shard_columns, gather_columns
        from synth import gen
        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        # conv: 10 images of 14x14 over the ranks, whole images per rank
        cin, cout, B, H, W = 64, 96, 10, 14, 14
        w = gen.pruned_weights(cout, 9 * cin, 90, seed=21)
        x = gen.relu_normal_x((cin, B, H, W), seed=22)
        b0, b1 = shard_columns(B, world, rank)
        plan = srt.Plan.from_csr(w, kind=srt.SPARSE_CONV3X3, c_in=cin, h=H, w=W, n_hint=B, device=0)  # replica
        y = plan.conv3x3(torch.from_numpy(np.ascontiguousarray(x[:, b0:b1])).to(dev))
        torch.cuda.synchronize()
        ys = [None] * world
        dist.all_gather_object(ys, y.cpu().numpy())
        digs = [None] * world
        dist.all_gather_object(digs, int(plan.info["digest"]))
        # SpMM: column slabs on whole 49-column samples
        M, K, N = 512, 2048, 49 * 9
        ws = gen.pruned_weights(M, K, 90, seed=23)
        X = gen.uniform_x(K, N, seed=24)
        n0, n1 = shard_columns(N, world, rank, 49)
        ps = srt.Plan.from_csr(ws, n_hint=N, device=0)  # replica
        Yl = ps.spmm(torch.from_numpy(np.ascontiguousarray(X[:, n0:n1])).to(dev))
        torch.cuda.synchronize()
        Yg = gather_columns(Yl.cpu(), N, world, 49).numpy()
        if rank == 0:
            full = srt.Plan.from_csr(w, kind=srt.SPARSE_CONV3X3, c_in=cin, h=H, w=W, n_hint=B, device=0)
            yf = full.conv3x3(torch.from_numpy(x).to(dev)).cpu().numpy()
            fs = srt.Plan.from_csr(ws, n_hint=N, device=0)
            Yf = fs.spmm(torch.from_numpy(X).to(dev)).cpu().numpy()
            q.put((len(set(digs)) == 1, bool(np.array_equal(np.concatenate(ys, axis=1), yf)),
                   bool(np.array_equal(Yg, Yf))))
    finally:
        dist.destroy_process_group()


def test_two_processes_one_gpu_sharded_equals_unsharded():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    same_digest, conv_eq, spmm_eq = q.get(timeout=10)
    assert same_digest and conv_eq and spmm_eq
