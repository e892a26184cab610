"""A short run of every device path for compute-sanitizer (one tool per
process): BASELINE config 1 scale scene (2K splats, 4 views at 64x64),
12 3DGS2-TR steps (two refreshes), ADAM and ADAM-TR steps, the seams
(rasterize, JVP, VJP, SSIM/residual chain, gradient, Hutchinson, radii),
binning dump, evaluation, refresh bands and sharded radii.

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import pyoracle as orc  # noqa: E402
from paper_2602_00395_b200 import splat as sp  # noqa: E402


def main():
    ds = orc.make_synthetic(orc.SynthConfig(gt_splats=1500, init_splats=2000, views=4,
                                            image_size=64, seed=2))
    views = [sp.Camera.from_c(c, g) for c, g in zip(ds.cams, ds.gts)]
    ctx = sp.Context()
    ctx.set_scene(ds.init_x)
    ctx.set_views(views)
    ctx.state_reset(3)
    opt = sp.OptimizerOptions(schedule=sp.TrustRegionSchedule(1e-6, 1e-8, 30), batch_size=2)
    for _ in range(12):
        ctx.step(opt)
    ctx.set_refresh_bands(2)
    ctx.set_tr_shards(3)
    ctx.step(sp.OptimizerOptions(schedule=sp.TrustRegionSchedule(1e-6, 1e-8, 30), batch_size=2,
                                 hess_interval=1))
    for kind in ("adam", "adam-tr"):
        ctx.step(sp.OptimizerOptions(schedule=sp.TrustRegionSchedule(1e-6, 1e-8, 30),
                                     batch_size=2, kind=kind, scene_extent=1.3))
    scene = sp.Scene(ctx.get_scene())
    rng = np.random.default_rng(0)
    v = rng.standard_normal(scene.dim())
    for cam in views[:2]:
        out = sp.rasterize(scene, cam)
        sp.rasterize_jvp(scene, cam, v)
        sp.rasterize_vjp(scene, cam, rng.standard_normal((64, 64, 3)))
        sp.ssim_map(out.color, cam.gt)
    g, _ = sp.stochastic_gradient(scene, views, [0, 3])
    z = np.where(rng.integers(0, 2, scene.dim()) == 1, 1.0, -1.0)
    sp.hutchinson_diag(scene, views, [1], 1, lambda s: z)
    sp.shd_radii(scene, 1e-6)
    ctx.set_eval_views(views[:1])
    ctx.evaluate()
    print("sanitize run ok", float(np.linalg.norm(g)))


if __name__ == "__main__":
    main()
