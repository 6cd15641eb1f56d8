"""SURVEY §4 T8 (memory safety) without compute-sanitizer, which is closed on the GPU pool: the
bounds-checked build (libmrf_checked.so, MRF_CHECK=1: device-side checks of the belief-slot
gathers, the message slots of chunks and runs, the K6 accumulator indices, the compacted tile
positions, the DDA fill's voxel slots and the run placement; a failed check prints its site and
traps) runs scripts/sanitize_run.py through every K5 / K6 path and mode, one process per mode."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MODES = [("default", {}), ("staged", {"MRF_K5": "staged"}), ("voxel", {"MRF_K6": "voxel"}),
         ("compact", {"MRF_COMPACT": "1"}), ("runfill", {"MRF_RUN_FILL": "1"}), ("long", {}), ("kfavg", {}),
         ("sparse", {}), ("mf", {}), ("kfmf", {}), ("room", {}), ("room_tile", {"MRF_K6": "tile"}),
         ("block_fallback", {"MRF_K6": "block", "MRF_BLK_PROBE": "-1"})]


@pytest.mark.parametrize("mode,env", MODES, ids=[m for m, _ in MODES])
def test_checked_build_runs_clean(mode, env):
    from paper_2006_03512_b200 import _build
    lib = _build.build_checked()
    e = dict(os.environ, MRF_LIB=lib, **env)
    script_mode = ("default" if mode in ("staged", "voxel", "compact", "runfill") else
                   "room" if mode in ("room_tile", "block_fallback") else mode)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_run.py"), script_mode],
                       capture_output=True, text=True, timeout=900, env=e, cwd=ROOT)
    out = r.stdout + r.stderr
    assert "MRF_CHECK failed" not in out, out[-3000:]
    assert r.returncode == 0 and "done" in r.stdout, out[-3000:]
