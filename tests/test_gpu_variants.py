"""The kernel variants DESIGN.md §4 calls bit-identical give bit-identical
scenes: a few C2 training steps (100K splats, SH degree 3, 512x512, batch 8,
through refresh) under each variant knob, compared by the scene's hash.  The
knobs are read once per process, so every variant runs in its own process
(tools/scene_hash.py)."""
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
def test_bit_identical_variants():
    base = _hash({})
    for knobs in ({"SGTR_VJP_STAGED": "2"}, {"SGTR_FWD_WARP": "2"}):
        assert _hash(knobs) == base, knobs
