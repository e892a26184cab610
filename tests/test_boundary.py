"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every entry point include/sgtr.h declares, and the Python mirror's
host logic (options, scene layout, RNG mappings) follows the reference."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def built():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2602_00395_b200 import _lib
    return _lib


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "sgtr.h")).read()
    return sorted(set(re.findall(r"\b(sgtr_[A-Za-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported(built):
    L = built.lib()
    names = declared_symbols()
    assert len(names) >= 40
    for n in names:
        assert hasattr(L, n), n
    assert sorted(built.exported_symbols()) == names


def test_no_device_fails_loudly(built):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2602_00395_b200 import splat
    with pytest.raises(splat.SgtrError):
        splat.Context(0)


def test_eps_at_host(built):  # trust_region.cpp:261-268 (no device needed)
    from paper_2602_00395_b200 import splat
    s = splat.TrustRegionSchedule(1e-6, 1e-8, 1000)
    assert splat.eps_at(s, 0) == 1e-6
    assert splat.eps_at(s, 500) == pytest.approx(1e-7, rel=1e-12)
    assert splat.eps_at(s, 2000) == 1e-8
    with pytest.raises(splat.InvalidArgument, match="bad schedule"):
        splat.eps_at(splat.TrustRegionSchedule(1e-8, 1e-6, 10), 3)


def test_rng_matches_reference_stream(built, orc):
    from paper_2602_00395_b200 import splat
    a, b = splat.Rng(123), orc.Rng(123)
    assert np.array_equal(a.raw_n(1000), b.raw(1000))
    a, b = splat.Rng(9), orc.Rng(9)
    assert [a.normal() for _ in range(7)] == b.normal(7).tolist()
    a, b = splat.Rng(4), orc.Rng(4)
    assert a.sample_without_replacement(50, 7) == b.sample_without_replacement(50, 7).tolist()
    a, b = splat.Rng(6), orc.Rng(6)
    assert np.array_equal(a.rademacher_n(333), b.rademacher(333))


def test_synthetic_generator_matches_reference(built, orc):
    # dataset.cpp:25-67: scenes and cameras bit-identical to the oracle's
    from paper_2602_00395_b200 import splat
    gt, init, cams = splat.make_synthetic(gt_splats=64, init_splats=96, views=25, width=64)
    ds = orc.make_synthetic(orc.SynthConfig(), with_gt=False)
    assert np.array_equal(gt.x, ds.gt_x) and np.array_equal(init.x, ds.init_x)
    for c, oc in zip(cams, ds.cams):
        assert c.id == oc.id and c.fx == oc.fx and c.cx == oc.cx and c.width == oc.width
        assert tuple(c.q_wc) == tuple(oc.q_wc) and tuple(c.t_wc) == tuple(oc.t_wc)


def test_host_helpers(built):
    from paper_2602_00395_b200 import splat
    d = np.array([0.5, -0.3, 0.1])
    eta = np.array([0.2, 0.4, 0.2])
    c = splat.clip_step(d, eta)
    assert c.tolist() == [0.2, -0.3, 0.1] and np.array_equal(splat.clip_step(c, eta), c)
    g = np.array([1.0, -2.0])
    assert np.all(np.isfinite(splat.newton_step(g, np.zeros(2), 1e-12)))
    assert splat.ema(np.zeros(3), np.array([1.0, 2, 3]), 0.9).tolist() == pytest.approx(
        [0.1, 0.2, 0.3], rel=1e-15)
    s = splat.Scene.from_primitives([[1, 2, 3]], [[4, 5, 6]], [[7, 8, 9, 10]], [11], [[12, 13, 14]])
    assert s.x.tolist() == list(range(1, 15))
    assert (s.scale_offset(), s.quat_offset(), s.opacity_offset(), s.color_offset()) == (3, 6, 10, 11)


def run_cpp_host():
    import subprocess
    import tempfile
    exe = os.path.join(tempfile.mkdtemp(), "cpp_host")
    libdir = os.path.join(ROOT, "paper_2602_00395_b200")
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "cpp_host.cpp"), "-L", libdir, "-lsgtr",
                    f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "host-only C-ABI ok" in r.stdout
    return r.stdout


def test_cpp_caller_of_the_c_abi(built):
    """A C++ program compiled against include/sgtr.h and linked with
    libsgtr.so exercises the boundary without Python (host-only part)."""
    run_cpp_host()


@pytest.mark.gpu
def test_cpp_caller_steps_on_the_device(built):
    """The same C++ program on a B200: synthetic targets rendered on the
    device, then three sgtr_step_3dgs2tr calls, each printing its batch loss."""
    out = run_cpp_host()
    assert "no CUDA device" not in out, out
    losses = [float(m) for m in re.findall(r"^step \d loss (\S+)", out, re.M)]
    assert len(losses) == 3 and all(np.isfinite(losses)) and min(losses) > 0, out
