"""The reference's own suites running on the B200 through the drop-in.

integration/Makefile links the UNMODIFIED reference (splat_core minus
src/render.cpp and src/optimizer.cpp, which integration/b200_backend.cpp
replaces by calls into libsgtr.so) and its unmodified unit and acceptance
suites.  So every KAT of test_render.cpp, test_optimizer.cpp,
test_residuals.cpp, ... and acceptance criteria 1-10 exercise the CUDA path
through the reference's own C++ API (OptimizerState, Scene, Camera,
step_3dgs2tr, rasterize_vjp, hutchinson_diag, ...).

The binaries are built in this container (they need /root/reference) and
travel to the GPU box with the snapshot.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "integration", "_build")
UNIT = os.path.join(BUILD, "unit_tests_b200")
ACCEPT = os.path.join(BUILD, "acceptance_tests_b200")
LIB = os.path.join(BUILD, "libsplat_core_b200.so")

built = pytest.mark.skipif(not os.path.exists(UNIT), reason="integration/_build not built")


@built
def test_backend_replaces_render_and_optimizer():
    """The library defines the reference's render/optimizer entry points
    itself and takes them to libsgtr (no CPU fallback is linked in)."""
    syms = subprocess.run(["nm", "-DC", "--defined-only", LIB], capture_output=True,
                          text=True).stdout
    for name in ("splat::step_3dgs2tr(", "splat::rasterize(", "splat::rasterize_vjp(",
                 "splat::hutchinson_diag(", "splat::stochastic_gradient(",
                 "splat::optimizer_step(", "splat::view_jacobian_applyT("):
        assert name in syms, name
    undef = subprocess.run(["nm", "-DC", "--undefined-only", LIB], capture_output=True,
                           text=True).stdout
    for name in ("sgtr_step_3dgs2tr_explicit", "sgtr_rasterize_vjp", "sgtr_hutchinson_diag"):
        assert name in undef, name
    deps = subprocess.run(["ldd", LIB], capture_output=True, text=True).stdout
    assert "libsgtr.so" in deps


@built
@pytest.mark.gpu
def test_reference_unit_suite_on_b200(tmp_path):
    r = subprocess.run([UNIT], cwd=tmp_path, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-6000:]
    assert "test cases: 83 | 83 passed" in r.stdout, out[-6000:]


@built
@pytest.mark.gpu
def test_reference_acceptance_on_b200(tmp_path):
    r = subprocess.run([ACCEPT], cwd=tmp_path, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    passed = set(int(m) for m in re.findall(r"\[PASS\] criterion\s+(\d+)", r.stdout))
    assert r.returncode == 0 and passed == set(range(1, 11)), out[-6000:]
    assert "all acceptance criteria passed" in r.stdout
