"""Generates tests/golden/c1_reference.npz (the compiled reference,
oracle/_ref via oracle/pyref.py -- the default) or, with ``--oracle``, the
same run of the restatement into /tmp/c1_oracle.npz (bit-identical to the
reference's): BASELINE config 1 (10K splats, 4 views
at 128x128, id 0 held out as in split_views, dataset.cpp:79-85) trained for
100 3DGS²-TR iterations (seed 1, nu 1, |S1| = |S2| = 1, l = 10, eps 1e-6 ->
1e-8 over 100 steps) on the CPU.  Stores the per-step diagnostics, the
held-out PSNR after the last step (evaluate_scene, harness.cpp:43-58) and the
final scene.  Run:  python tests/golden/make_c1_golden.py [--oracle]
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

if "--oracle" in sys.argv:
    from oracle import pyoracle as orc  # noqa: E402
    OUT = "/tmp/c1_oracle.npz"
else:
    from oracle import pyref  # noqa: E402
    pyref.build()
    orc = pyref.ref
    OUT = "c1_reference.npz"

ITERS = 100


def main():
    orc.build()
    ds = orc.make_synthetic(orc.SynthConfig(gt_splats=10000, init_splats=10000, views=4,
                                            image_size=128, seed=1))
    train = [i for i in range(4) if i % 5 != 0]
    held = [i for i in range(4) if i % 5 == 0]
    cams = [ds.cams[i] for i in train]
    gts = [ds.gts[i] for i in train]
    x = ds.init_x.copy()
    st = orc.State(x.size, 1)
    opts = orc.TrOptions(total_steps=ITERS)
    diag = []
    t0 = time.time()
    for t in range(1, ITERS + 1):
        d = orc.step_3dgs2tr(st, x, cams, gts, opts)
        diag.append([d[k] for k in ("batch_loss", "gnorm", "step_pre", "step_post",
                                    "clip_frac", "eps", "max_step_over_radius")])
    psnr = [orc.psnr(orc.quantize8(orc.rasterize(x, ds.cams[i])[0]), ds.gts[i]) for i in held]
    np.savez_compressed(os.path.join(HERE, OUT), diag=np.array(diag),
                        psnr=np.array(psnr), final_x=x, init_x=ds.init_x)
    print(f"done in {time.time() - t0:.1f}s: held-out PSNR {psnr}")


if __name__ == "__main__":
    main()
