"""The multi-rank data plane on one GPU.

The view batch is split round-robin over ranks, each rank's
[g | loss | flags | errors | z.w] buffer is summed by one allreduce per step,
refresh views are cut into tile-row bands when |S2| < ranks, and the
trust-region radii are sharded by splat range and all-gathered
(DESIGN §0(e)).  NCCL cannot put two ranks on one GPU, so these tests use
libsgtr's in-process communicator (sgtr_comm_init_loopback: one host thread
and one context per rank, collectives through device memory in rank order):
the same step code, buffers and collectives call sites as the NCCL path.
An N-rank run must agree with the 1-rank run to rounding.

test_nccl_two_gpus runs the real NCCL path with torchrun when two devices
are visible (it skips on the one-GPU boxes this project is measured on).
"""
import os
import subprocess
import sys
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


@pytest.fixture(scope="module")
def sp():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2602_00395_b200 import splat
    return splat


@pytest.fixture(scope="module")
def ds(orc):
    return orc.make_synthetic(orc.SynthConfig(gt_splats=300, init_splats=300, views=6,
                                              image_size=48, seed=5))


def run_ranks(sp, ds, nranks, steps, batch, kind="3dgs2tr", cap=None):
    views = [sp.Camera.from_c(c, g) for c, g in zip(ds.cams, ds.gts)]
    opt = sp.OptimizerOptions(schedule=sp.TrustRegionSchedule(1e-6, 1e-8, 40), batch_size=batch,
                              kind=kind, scene_extent=1.3, record_applied_step=False)
    ctxs = []
    for r in range(nranks):
        c = sp.Context()
        c.set_scene(ds.init_x)
        c.set_views(views)
        c.state_reset(11)
        if cap is not None:
            c.set_dup_capacity(cap)
        ctxs.append(c)
    group = None
    if nranks > 1:
        group = sp.LoopbackGroup(nranks)
        for r, c in enumerate(ctxs):
            c.comm_init_loopback(group, r)
    out = [None] * nranks
    errs = []

    def work(r):
        try:
            diags = [ctxs[r].step(opt) for _ in range(steps)]
            g, d, t = ctxs[r].state_get()
            out[r] = dict(g=g, d=d, t=t, x=ctxs[r].get_scene(),
                          loss=[dg.batch_loss for dg in diags],
                          refreshed=[dg.refreshed for dg in diags],
                          local=[dg.n_local_views for dg in diags],
                          reruns=[dg.reruns for dg in diags])
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    threads = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for c in ctxs:
        c.close()
    if group:
        group.close()
    assert not errs, errs
    return out


@pytest.mark.parametrize("nranks,batch", [(2, 4), (3, 4), (4, 4), (5, 4)])
def test_n_ranks_match_one_rank(sp, ds, nranks, batch):
    # refreshes at t = 1 and 11 (|S2| = 1 < ranks: row bands; at 4 and 5
    # ranks some rank has no band, at 5 one also has no gradient view)
    steps = 12
    one = run_ranks(sp, ds, 1, steps, batch)[0]
    many = run_ranks(sp, ds, nranks, steps, batch)
    for r, o in enumerate(many):
        # every rank holds the identical replica
        assert np.array_equal(o["x"], many[0]["x"]) and np.array_equal(o["g"], many[0]["g"])
        assert np.array_equal(o["d"], many[0]["d"])
        assert o["t"] == steps and o["refreshed"] == one["refreshed"]
        assert sum(m["local"][0] for m in many) == batch
    m = many[0]
    assert rel(m["g"], one["g"]) < 1e-11
    assert rel(m["d"], one["d"]) < 1e-11
    assert rel(m["x"], one["x"]) < 1e-8
    assert np.allclose(m["loss"], one["loss"], rtol=1e-12, atol=0)


def test_capacity_reruns_are_collective(sp, ds):
    """Every rank starts with a capacity its views outgrow: the overflow
    count is part of the summed tail, so all ranks rerun the step together
    and grow alike, and the result is the 1-rank run's."""
    one = run_ranks(sp, ds, 1, 4, 4)[0]
    many = run_ranks(sp, ds, 3, 4, 4, cap=16)
    for o in many:
        assert o["reruns"] == many[0]["reruns"] and o["reruns"][0] >= 1
        assert np.array_equal(o["x"], many[0]["x"])
    assert rel(many[0]["g"], one["g"]) < 1e-11
    assert rel(many[0]["x"], one["x"]) < 1e-8


def test_adam_tr_two_ranks(sp, ds):
    one = run_ranks(sp, ds, 1, 6, 4, kind="adam-tr")[0]
    two = run_ranks(sp, ds, 2, 6, 4, kind="adam-tr")
    assert np.array_equal(two[0]["x"], two[1]["x"])
    assert rel(two[0]["x"], one["x"]) < 1e-8
    assert np.allclose(two[0]["loss"], one["loss"], rtol=1e-12, atol=0)


def visible_gpus():
    # counted in a child process: importing torch here, after libsgtr brought
    # in the system libnccl, would clash with torch's bundled NCCL
    r = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True)
    n = sum(1 for line in r.stdout.splitlines() if line.startswith("GPU "))
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES")
    return n if cvd is None else min(n, len([d for d in cvd.split(",") if d.strip()]))


def test_nccl_two_gpus(tmp_path):
    if visible_gpus() < 2:
        pytest.skip("needs two visible GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", "29533", os.path.join(root, "tools", "nccl_check.py")],
                       cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "nccl_check ok" in r.stdout
