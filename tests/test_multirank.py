"""Multi-GPU host logic on CPU (gloo, world size 2).

libsgtr splits each step's view batch over ranks (sgtr_shard_views), sums
[g | z.w | loss] with one allreduce and applies the trust-region update on
every replica.  Here two gloo ranks compute their shards' unscaled gradient
and loss sums with the CPU oracle, all-reduce them, and must reproduce the
single-process stochastic_gradient (optimizer.cpp:36-65) — the same scaling
the GPU path applies after its ncclAllReduce.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, batch, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import pyoracle as orc
    from paper_2602_00395_b200 import splat as sp

    x, cams, gts = orc.make_check_scene(6, 16, 5, 21)
    M = len(cams)
    m = 6 * 16 * 16 * M
    mine = sp.shard_views(len(batch), rank, world)
    g = np.zeros(x.size)
    loss = 0.0
    for p in mine:
        # unscaled per-view sums: stochastic_gradient with |batch| = 1 returns
        # g_v * M/m and loss_v * M/(2m)
        gv, lv = orc.stochastic_gradient(x, cams, gts, [batch[p]])
        g += gv * m / M
        loss += lv * 2 * m / M
    buf = torch.from_numpy(np.concatenate([g, [loss]]))
    dist.all_reduce(buf)
    tot = buf.numpy()
    n1 = len(batch)
    out[rank] = (tot[:-1] * M / (m * n1), tot[-1] * M / (2 * m * n1), mine)
    dist.destroy_process_group()


def test_shards_partition_the_batch():
    from paper_2602_00395_b200 import splat as sp
    for n in (1, 2, 7, 8, 32):
        for world in (1, 2, 4, 8):
            parts = [sp.shard_views(n, r, world) for r in range(world)]
            flat = sorted(p for part in parts for p in part)
            assert flat == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


@pytest.mark.parametrize("batch", [[3, 1, 4, 0], [2]])
def test_two_rank_gradient_equals_single(orc, batch):
    import __graft_entry__
    __graft_entry__.build()
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(2, port, batch, out), nprocs=2, join=True)
        res = dict(out)
    x, cams, gts = orc.make_check_scene(6, 16, 5, 21)
    g_ref, loss_ref = orc.stochastic_gradient(x, cams, gts, batch)
    for r in (0, 1):
        g, loss, _ = res[r]
        assert np.max(np.abs(g - g_ref)) <= 1e-12 * np.max(np.abs(g_ref))
        assert loss == pytest.approx(loss_ref, rel=1e-12)
    assert np.array_equal(res[0][0], res[1][0])  # replicas see identical bits
