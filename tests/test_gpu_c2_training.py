"""BASELINE config 2 as a training run: 100K Gaussians, SH degree 3, 16 views
at 512x512 (views with id % 5 == 0 held out, split_views dataset.cpp:79-85),
|S1| = 8, 500 3DGS²-TR iterations with the refresh every 10th.

The training-view and held-out PSNR (evaluate_scene on the device:
quantize8 + psnr, harness.cpp:43-58) are recorded every 50 iterations.  The
training fit must keep improving (each 100-iteration window ends above where
it began, the reference's regression criterion, acceptance.cpp:205-212) and
gain over 15 dB; the held-out views must improve at first.  With 48 SH
coefficients per splat and 12 training views the view-dependent colour
overfits: measured, training 17.5 -> 38.1 dB while held-out rises to 20.1 dB
at iteration 50 and then slides to 18.4 dB (the same geometry at SH degree 0:
training 18.1 -> 31.8, held-out 18.1 -> 23.4 dB, monotone;
tools/c2_diag.py).  The trajectory is written to $SGTR_C2_LOG (JSON) when
set.  There is no CPU comparison at this size (a single oracle iteration takes hours); C2's
kernels are covered against the oracle on crops
(test_gpu_parity.py::test_c2_scale_crop_parity, test_gpu_sh.py)."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_c2_500_iterations():
    import __graft_entry__
    __graft_entry__.build()
    import bench
    from paper_2602_00395_b200 import splat as sp

    k, v, w, h, b, sh = bench.CONFIGS["c2"]
    ctx = sp.Context()
    gt, init, cams = bench.make_dataset(sp, ctx, "c2", 1)
    targets = [ctx.get_target(i, w, h) for i in range(v)]
    train = [i for i in range(v) if i % 5 != 0]
    held = [i for i in range(v) if i % 5 == 0]
    ctx.set_views([sp.Camera.from_c(cams[i]._c(), targets[i]) for i in train])
    ctx.set_eval_views([sp.Camera.from_c(cams[i]._c(), targets[i]) for i in held])
    ctx.set_scene(init.x, sh)
    ctx.state_reset(1)
    opt = sp.OptimizerOptions(batch_size=b, schedule=sp.TrustRegionSchedule(1e-6, 1e-8, 500),
                              record_applied_step=False)

    def point(t, loss):
        ev = ctx.evaluate()
        tr = ctx.evaluate(training_views=True)
        return (t, ev.mean_psnr, ev.mean_ssim, tr.mean_psnr, loss)

    traj = [point(0, None)]
    for t in range(1, 501):
        d = ctx.step(opt)
        assert np.isfinite(d.batch_loss)
        if t % 50 == 0:
            traj.append(point(t, d.batch_loss))
    ctx.close()
    log = os.environ.get("SGTR_C2_LOG")
    if log:
        with open(log, "w") as f:
            json.dump({"config": bench.workload_desc("c2"), "held_out_views": held,
                       "trajectory": [{"iter": t, "held_out_psnr": p, "held_out_ssim": s,
                                       "train_psnr": tp, "loss": l}
                                      for t, p, s, tp, l in traj]}, f, indent=1)
    train_psnr = [tp for _, _, _, tp, _ in traj]
    held_psnr = [p for _, p, _, _, _ in traj]
    assert train_psnr[-1] > train_psnr[0] + 15.0, train_psnr
    assert all(train_psnr[i + 2] > train_psnr[i] for i in range(0, len(train_psnr) - 2, 2))
    assert held_psnr[1] > held_psnr[0] + 1.0, held_psnr
