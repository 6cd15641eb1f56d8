"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the MRFMap method (no traversal, no
messages, no marginals).  It only produces the inputs the method consumes:
posed z-depth frames rendered from a seeded room scene, and the forward sensor
model tabulated as a log-density LUT (Eq.4; A1 reading in
DESIGN.md).  Both the oracle and the CUDA path read exactly these bytes.

Recipe: SURVEY.md §8(d) "Generator spec" (DESIGN.md §Inputs restates it).
"""

from .scenes import (  # noqa: F401
    Frame,
    Workload,
    CONFIG_NAMES,
    make_workload,
    tiny,
    tiny_frames,
    single_frame,
    frames30,
    frames100,
    sweep300,
    tiny_patch,
    frame1_patch,
    PatchNoise,
    patch_noise_model,
)
from .lut import build_log_nu_lut  # noqa: F401
