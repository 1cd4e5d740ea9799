"""Multi-process (world_size 2, gloo, CPU) tests of the data-parallel host logic:
view-sharded batches are disjoint and cover only the rank's views, the NCCL unique id is
broadcast identically (the id comes from the library's dinr_nccl_unique_id), and averaging per-rank oracle gradients equals the gradient of the
union batch (K-invariance, R16)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        from oracle import oracle as O
        from paper_2404_19075_b200 import dist as pd
        from paper_2404_19075_b200 import synth

        # 1) unique-id broadcast of the library's own NCCL id (dinr_nccl_unique_id: ncclGetUniqueId
        #    needs no GPU), exactly as dist.init_comm does before dinr_comm_init
        from paper_2404_19075_b200 import _lib as D

        uid = pd.broadcast_unique_id(D.nccl_unique_id, rank, world)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        # 2) shards
        name = "fan512"
        idx = pd.shard_batch(name, 6, rank, world, seed=5)
        N = 512
        own_views = set((idx // N) % world)
        shards = [None] * world
        dist.all_gather_object(shards, idx.tolist())
        # 3) K-invariance with the oracle on a tiny net
        g = synth.geometry(name, n_s=32)
        th, t = synth.views(name)
        f = synth.field(name, C=4, L=2)
        B = synth.grff_matrix(4, 0.1, 0.5)
        prm = synth.init_params(4, 2)
        y = synth.synthetic_y(6, 1.0, seed=rank)
        gr, _ = O.project_and_grad(g, th, t, f, B, prm, idx, y)
        tg = torch.tensor(gr)
        dist.all_reduce(tg)
        avg = (tg / world).numpy()
        ys = [None] * world
        dist.all_gather_object(ys, y.tolist())
        out_q.put((rank, ids, own_views, shards, avg, ys))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo(O):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    # identical ids everywhere (128 bytes from rank 0's ncclGetUniqueId, not all zero)
    assert res[0][1][0] == res[0][1][1] == res[1][1][0]
    assert len(res[0][1][0]) == 128 and any(res[0][1][0])
    # each rank drew only from its own views, and the shards are disjoint
    for r in range(world):
        assert res[r][2] == {r}
    s0, s1 = set(res[0][3][0]), set(res[0][3][1])
    assert not (s0 & s1)
    # averaged per-rank gradients == gradient of the union batch (equal |Omega_k|)
    from paper_2404_19075_b200 import synth

    name = "fan512"
    g = synth.geometry(name, n_s=32)
    th, t = synth.views(name)
    f = synth.field(name, C=4, L=2)
    B = synth.grff_matrix(4, 0.1, 0.5)
    prm = synth.init_params(4, 2)
    idx = np.array(res[0][3][0] + res[0][3][1], dtype=np.int64)
    y = np.array(res[0][5][0] + res[0][5][1])
    full, _ = O.project_and_grad(g, th, t, f, B, prm, idx, y)
    assert np.allclose(res[0][4], full, rtol=1e-12, atol=1e-15)
    assert np.array_equal(res[0][4], res[1][4])
