"""ctypes binding of the compiled REFERENCE (oracle/_ref/libsplat_ref.so).

TEST INFRASTRUCTURE ONLY, like pyoracle.  oracle/ref.mk compiles the
unmodified reference sources (/root/reference/proj/src) against the
stand-ins in oracle/refshim/ together with oracle/ref_capi.cpp, which
exports the orc_* entry points of oracle.h that the reference has a
counterpart for, implemented by calling the reference itself.  This module
is a second instance of pyoracle's wrappers bound to that library, so every
wrapper (rasterize, stochastic_gradient, step_3dgs2tr, make_synthetic, ...)
has the same signature whether it asks the restatement or the reference.

``available()`` is False when the library was not built (no
/root/reference at build time); tests skip then.  On the GPU box the
prebuilt library travels with the snapshot; the reference sources do not.
"""
from __future__ import annotations

import ctypes as C
import importlib.util
import os
import subprocess
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(_HERE, "_ref")
LIB_PATH = os.path.join(REF_DIR, "libsplat_ref.so")
UNIT_TESTS = os.path.join(REF_DIR, "unit_tests")
ACCEPTANCE_TESTS = os.path.join(REF_DIR, "acceptance_tests")
REFERENCE_SRC = os.environ.get("SGTR_REFERENCE", "/root/reference/proj")


def build() -> bool:
    """Compile oracle/_ref with oracle/ref.mk when the reference sources are
    present (this container); returns whether the library exists."""
    if os.path.isdir(os.path.join(REFERENCE_SRC, "src")):
        subprocess.run(["make", "-s", "-j", str(os.cpu_count() or 4), "-f",
                        os.path.join(_HERE, "ref.mk"), f"REF={REFERENCE_SRC}"], check=True)
    return os.path.exists(LIB_PATH)


def available() -> bool:
    return os.path.exists(LIB_PATH)


def _load():
    spec = importlib.util.spec_from_file_location("oracle._pyref_impl",
                                                  os.path.join(_HERE, "pyoracle.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["oracle._pyref_impl"] = mod
    spec.loader.exec_module(mod)
    mod._LIB_PATH = LIB_PATH
    mod.build = lambda force=False: LIB_PATH  # never rebuild the restatement here

    def _lib():
        if mod._lib is None:
            if not os.path.exists(LIB_PATH):
                raise FileNotFoundError(f"{LIB_PATH} not built (make -f oracle/ref.mk)")
            L = C.CDLL(LIB_PATH)
            mod._setup(L)
            L.ref_project.restype = C.c_int
            mod._lib = L
        return mod._lib

    mod.lib = _lib

    def project(x, cam, ro=None):
        """splat::project<double> per splat: (K, 8) culled, depth, mu_x, mu_y,
        c00, c01, c11, 0 (render.hpp:34-63)."""
        ro = ro or mod.RenderOptions()
        x = mod._f64(x)
        k = x.size // 14
        out = np.empty((k, 8))
        mod._check(_lib().ref_project(mod._p(x), C.c_int64(k), C.byref(cam), C.byref(ro.c()),
                                      mod._p(out)))
        return out

    def evaluate_scene(x, cams, gts, ro=None):
        """harness.cpp:43-58: per-view (psnr, ssim) of quantize8(render)."""
        ro = ro or mod.RenderOptions()
        x = mod._f64(x)
        n = len(cams)
        keep, ptrs = mod._gts(gts)
        ps, ss = np.empty(n), np.empty(n)
        mod._check(_lib().ref_evaluate_scene(mod._p(x), C.c_int64(x.size // 14), mod._cams(cams),
                                             ptrs, n, C.byref(ro.c()), ro.workers, mod._p(ps),
                                             mod._p(ss)))
        return ps, ss

    mod.project = project
    mod.evaluate_scene = evaluate_scene
    return mod


ref = _load()
