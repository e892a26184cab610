"""Print a hash of the scene after a few training steps (A/B bit-identity
checks between builds: SGTR_LIB=<other libsgtr.so> python tools/scene_hash.py).

  python tools/scene_hash.py [config] [steps] [duplicate capacity before the steps]"""
import hashlib
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402  (dataset helpers)
from paper_2602_00395_b200 import splat as sp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = sp.Context(0)
k, v, w, h, b, sh = bench.CONFIGS[cfg]
bench.make_dataset(sp, ctx, cfg, 0)
ctx.state_reset(0)
if len(sys.argv) > 3:
    ctx.set_dup_capacity(int(sys.argv[3]))
opt = sp.OptimizerOptions(batch_size=b, schedule=sp.TrustRegionSchedule(1e-6, 1e-8, 30000),
                          record_applied_step=False)
reruns = sum(ctx.step(opt).reruns for _ in range(steps))
x = ctx.get_scene()
print("reruns", reruns)
print(cfg, steps, hashlib.sha256(x.tobytes()).hexdigest()[:16])
