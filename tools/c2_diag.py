"""C2 training diagnostics: held-out and training PSNR every 50 iterations
for SH degree 3 and 0 (same geometry), 3DGS2-TR."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2602_00395_b200 import splat as sp  # noqa: E402

out = {}
for sh in (3, 0):
    bench.CONFIGS["c2x"] = (100_000, 16, 512, 512, 8, sh)
    k, v, w, h, b, _ = bench.CONFIGS["c2x"]
    ctx = sp.Context()
    gt, init, cams = bench.make_dataset(sp, ctx, "c2x", 1)
    targets = [ctx.get_target(i, w, h) for i in range(v)]
    train = [i for i in range(v) if i % 5 != 0]
    held = [i for i in range(v) if i % 5 == 0]
    ctx.set_views([sp.Camera.from_c(cams[i]._c(), targets[i]) for i in train])
    ctx.set_eval_views([sp.Camera.from_c(cams[i]._c(), targets[i]) for i in held])
    ctx.set_scene(init.x, sh)
    ctx.state_reset(1)
    opt = sp.OptimizerOptions(batch_size=b, schedule=sp.TrustRegionSchedule(1e-6, 1e-8, 500),
                              record_applied_step=False)
    rows = []
    for t in range(0, 501):
        if t:
            d = ctx.step(opt)
        if t % 50 == 0:
            rows.append((t, round(ctx.evaluate().mean_psnr, 3),
                         round(ctx.evaluate(training_views=True).mean_psnr, 3),
                         d.batch_loss if t else None, d.clip_frac if t else None))
    out[f"sh{sh}"] = rows
    print(sh, rows, flush=True)
    ctx.close()
json.dump(out, open("gpurun_out/c2_diag.json", "w"), indent=1)
