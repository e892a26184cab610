"""Print the acceptance-criterion-9 PSNR curves (tests/test_gpu_acceptance.py)."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import __graft_entry__
__graft_entry__.build()
from paper_2602_00395_b200 import splat as sp
import test_gpu_acceptance as T

gt, init, cams = sp.make_synthetic()
ctx = sp.Context()
ctx.set_scene(gt.x)
ctx.set_cameras(cams)
ctx.render_targets(quantize=True)
for i, c in enumerate(cams):
    c.gt = ctx.get_target(i, c.width, c.height)
train = [c for c in cams if c.id % 5 != 0]
held = [c for c in cams if c.id % 5 == 0]
for kind in ("3dgs2tr", "adam", "adam-tr"):
    p = T._bench_train(sp, init.x, train, held, kind)
    print(kind, " ".join(f"{p[t]:.2f}" for t in sorted(p)))
