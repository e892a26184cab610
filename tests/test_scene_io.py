"""Scene / camera files (scene_io.cpp), mirroring test_scene_io.cpp:43-167.

The host-buffer PLY and camera entry points of libsgtr run without a GPU;
the device path (Context.save_scene / load_scene) is covered by the gpu-marked
test at the end.
"""
import math
import os

import numpy as np
import pytest

from paper_2602_00395_b200 import splat as sp


def random_scene(k, seed):  # test_scene_io.cpp:15-28 (numpy draws)
    r = np.random.default_rng(seed)
    mu = r.uniform(-1, 1, (k, 3))
    s = r.uniform(0.05, 0.5, (k, 3))
    q = r.normal(size=(k, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    a = r.uniform(0.1, 0.9, k)
    c = r.uniform(0.1, 1.0, (k, 3))
    return sp.Scene(np.concatenate([mu.ravel(), s.ravel(), q.ravel(), a, c.ravel()]))


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()


def test_ply_round_trip_is_bitwise(tmp_path):  # :67-75
    s = random_scene(3, 33)
    p = tmp_path / "roundtrip.ply"
    sp.save_scene(s, p)
    assert np.array_equal(sp.load_scene(p).x, s.x)
    # the reference's exact header and AoS payload
    raw = p.read_bytes()
    head, payload = raw.split(b"end_header\n", 1)
    assert head.startswith(b"ply\nformat binary_little_endian 1.0\ncomment splat-tr v1\n"
                           b"element vertex 3\nproperty double x\n")
    rows = np.frombuffer(payload, "<f8").reshape(3, 14)
    assert np.array_equal(rows[1, :3], s.x[3:6])       # mu of splat 1
    assert np.array_equal(rows[2, 6:10], s.x[6 * 3 + 8:6 * 3 + 12])  # quat of splat 2
    assert rows[0, 10] == s.x[10 * 3]                  # opacity of splat 0


def test_ply_rejects_invariant_violations(tmp_path):  # :77-84
    s = random_scene(2, 5)
    s.x[10 * 2 + 1] = 1.5
    p = tmp_path / "bad_alpha.ply"
    sp.save_scene(s, p)
    with pytest.raises(sp.SgtrError, match="splat 1: opacity out of range"):
        sp.load_scene(p)


def test_empty_scene_file_is_valid(tmp_path):  # :86-91
    p = tmp_path / "empty.ply"
    sp.save_scene(sp.Scene(np.zeros(0)), p)
    assert sp.load_scene(p).size() == 0


def test_malformed_headers(tmp_path):  # :93-107
    p = tmp_path / "malformed.ply"
    p.write_text("ply\nformat binary_little_endian 1.0\nelement vertex 1\n"
                 "property double x\nend_header\n")
    with pytest.raises(sp.SgtrError, match="14"):
        sp.load_scene(p)
    p.write_text("not a ply\n")
    with pytest.raises(sp.SgtrError, match="malformed.ply:1: not a PLY file"):
        sp.load_scene(p)
    p.write_text("ply\nformat ascii 1.0\n")
    with pytest.raises(sp.SgtrError, match="unsupported format"):
        sp.load_scene(p)


def test_truncated_payload(tmp_path):
    s = random_scene(4, 9)
    p = tmp_path / "trunc.ply"
    sp.save_scene(s, p)
    raw = p.read_bytes()
    p.write_bytes(raw[:-14 * 8 - 5])
    with pytest.raises(sp.SgtrError, match="truncated payload at element 2"):
        sp.load_scene(p)


def test_ply_nonfinite_names_element(tmp_path):  # :109-116
    s = random_scene(2, 8)
    s.x[3 * 1 + 0] = np.nan
    p = tmp_path / "nan.ply"
    sp.save_scene(s, p)
    with pytest.raises(sp.SgtrError, match="splat 1"):
        sp.load_scene(p)


def test_validation_order_and_bounds(tmp_path):
    # scene.cpp:60-80 order: finite/scale/color per axis, quaternion, opacity
    s = random_scene(3, 2)
    k = 3
    s.x[3 * k + 3 * 2 + 1] = 1e-9          # scale of splat 2 below s_min
    s.x[6 * k + 4 * 2:6 * k + 4 * 2 + 4] = 0.0  # and a degenerate quaternion
    p = tmp_path / "order.ply"
    sp.save_scene(s, p)
    with pytest.raises(sp.SgtrError, match="splat 2: scale below s_min"):
        sp.load_scene(p)
    with pytest.raises(sp.SgtrError, match="splat 2: degenerate quaternion"):
        sp.load_scene(p, sp.ParamBounds(s_min=1e-12))


def test_camera_file_round_trip(tmp_path):  # :118-140
    cams = []
    for i in range(3):
        c = sp.look_at_camera((2.0 + i, -1.0, 0.8), (0.0, 0.0, 0.0), 120, 130, 32, 24)
        c.id = i * 5
        c.image_name = f"img_{i}.png"
        cams.append(c)
    p = tmp_path / "cams.txt"
    sp.save_cameras(cams, p)
    loaded = sp.load_cameras(p)
    assert len(loaded) == 3
    for a, b in zip(loaded, cams):
        assert a.id == b.id and a.fx == b.fx and a.width == b.width
        assert np.linalg.norm(np.subtract(a.t_wc, b.t_wc)) < 1e-15
        assert np.linalg.norm(a.rotation() - b.rotation()) < 1e-12
        assert a.image_name == b.image_name
    assert p.read_text().startswith("# id fx fy cx cy width height qw qx qy qz tx ty tz image\n")


def test_camera_file_comments_and_bad_lines(tmp_path):  # :142-153
    p = tmp_path / "cams_bad.txt"
    p.write_text("# header comment\n\n"
                 "0 100 100 8 8 16 16 1 0 0 0 0 0 2 a.png # trailing\n"
                 "1 100 100 8 8 16 16 1 0 0\n")
    with pytest.raises(sp.SgtrError, match="cams_bad.txt:4"):
        sp.load_cameras(p)
    p.write_text("0 -1 100 8 8 16 16 1 0 0 0 0 0 2 a.png\n")
    with pytest.raises(sp.SgtrError, match="focal lengths must be positive"):
        sp.load_cameras(p)
    p.write_text("0 100 100 8 8 16 16 2 0 0 0 0 0 2 a.png\n")
    (c,) = sp.load_cameras(p)
    assert tuple(c.q_wc) == (0.0, 0.0, 0.0, 1.0) and c.image_name == "a.png"


def test_scene_extent():  # :155-167
    assert sp.scene_extent([]) == 1.0
    cams = [sp.look_at_camera((2 * math.cos(i * math.pi / 2), 2 * math.sin(i * math.pi / 2), 0),
                              (0, 0, 0), 100, 100, 16, 16) for i in range(4)]
    assert sp.scene_extent(cams) == pytest.approx(2.0, rel=1e-12)


@pytest.mark.gpu
def test_device_ply_round_trip_and_validation(tmp_path):
    s = random_scene(1000, 4)
    ctx = sp.Context()
    ctx.set_scene(s.x)
    p = tmp_path / "dev.ply"
    ctx.save_scene(p)
    assert np.array_equal(sp.load_scene(p).x, s.x)  # host reader, same bits
    s2 = random_scene(700, 5)
    sp.save_scene(s2, tmp_path / "other.ply")
    ctx.load_scene(tmp_path / "other.ply")
    assert ctx.k == 700 and np.array_equal(ctx.get_scene(), s2.x)
    bad = random_scene(50, 6)
    bad.x[11 * 50 + 3 * 17 + 2] = 2.0  # colour of splat 17
    bad.x[11 * 50 + 3 * 31] = 2.0      # and 31: the lowest index is reported
    sp.save_scene(bad, tmp_path / "bad.ply")
    with pytest.raises(sp.SgtrError, match="splat 17: color out of range"):
        ctx.load_scene(tmp_path / "bad.ply")
    assert np.array_equal(ctx.get_scene(), s2.x)  # a failed load leaves the scene
