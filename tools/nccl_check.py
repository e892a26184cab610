"""Two-GPU check of the NCCL path (run by tests/test_gpu_multirank.py with
torchrun when two devices are visible): every rank steps the same scene with
its share of the views and one ncclAllReduce per step; rank 0 also runs the
1-rank step on its own device and compares."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch.distributed as dist
    from oracle import pyoracle as orc
    from paper_2602_00395_b200 import splat as sp

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    os.environ.setdefault("NCCL_ALGO", "Ring")
    os.environ.setdefault("NCCL_PROTO", "Simple")
    dist.init_process_group("gloo")
    ds = orc.make_synthetic(orc.SynthConfig(gt_splats=300, init_splats=300, views=6,
                                            image_size=48, seed=5))
    views = [sp.Camera.from_c(c, g) for c, g in zip(ds.cams, ds.gts)]
    opt = sp.OptimizerOptions(schedule=sp.TrustRegionSchedule(1e-6, 1e-8, 40), batch_size=4,
                              record_applied_step=False)

    def ctx_on(dev):
        c = sp.Context(dev)
        c.set_scene(ds.init_x)
        c.set_views(views)
        c.state_reset(11)
        return c

    ctx = ctx_on(local)
    uid = [sp.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    ctx.comm_init(uid[0], world, rank)
    for _ in range(12):
        ctx.step(opt)
    x = ctx.get_scene()
    g, d, _ = ctx.state_get()
    xs = [None] * world
    dist.all_gather_object(xs, x)
    if rank == 0:
        assert all(np.array_equal(xs[0], xr) for xr in xs)
        one = ctx_on(local)
        for _ in range(12):
            one.step(opt)
        x1 = one.get_scene()
        g1, d1, _ = one.state_get()
        rel = lambda a, b: float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))
        assert rel(g, g1) < 1e-11 and rel(d, d1) < 1e-11 and rel(x, x1) < 1e-8, \
            (rel(g, g1), rel(d, d1), rel(x, x1))
        print("nccl_check ok", rel(g, g1), rel(d, d1), rel(x, x1), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
