"""Results do not depend on scheduling knobs: the raster kernels' tile
launch order (SGTR_TILE_ORDER=0: row-major instead of longest list first)
and the number of view lanes (SGTR_LANES=1: no overlap) leave a few C2
training steps (100K splats, SH degree 3, 512x512, batch 8, through a
refresh) bit-identical.  Knobs are read once per process, so each runs in
its own process (tools/scene_hash.py)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _hash(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "tools/scene_hash.py", "c2", "11"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.strip().splitlines()[-1]


@pytest.mark.gpu
def test_scheduling_knobs_are_bit_identical():
    base = _hash({})
    for knobs in ({"SGTR_TILE_ORDER": "0"}, {"SGTR_LANES": "1"}):
        assert _hash(knobs) == base, knobs
