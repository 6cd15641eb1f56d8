"""ctypes binding of include/mrf.h -- argument marshalling only.

Every entry point keeps the C name (mrf_create, mrf_add_frame, mrf_bp_iterate,
mrf_marginals, ...).  Every step of the hot path runs in libmrf.so's CUDA kernels;
there is no Python or CPU fallback: if the library cannot be loaded, or a call fails,
an MrfError is raised.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import _build

_lock = threading.Lock()
_lib = None

MRF_OK, MRF_ERR_INVALID_ARG, MRF_ERR_OUT_OF_MEMORY, MRF_ERR_CAPACITY, MRF_ERR_CUDA, MRF_ERR_NCCL, MRF_ERR_STATE = range(7)
STATUS_NAMES = {0: "MRF_OK", 1: "MRF_ERR_INVALID_ARG", 2: "MRF_ERR_OUT_OF_MEMORY", 3: "MRF_ERR_CAPACITY",
                4: "MRF_ERR_CUDA", 5: "MRF_ERR_NCCL", 6: "MRF_ERR_STATE"}
MRF_COMM_NCCL, MRF_COMM_EXTERNAL = 0, 1
MRF_EVAL_SIGMA_BAND, MRF_EVAL_VOXEL_BOUNDS = 0, 1
MRF_MSG_PER_RAY, MRF_MSG_KEYFRAME_AVG = 0, 1
KERNEL_NAMES = ["raygen_count", "dda_fill", "scan", "transpose", "ray_messages", "voxel_sum", "allreduce",
                "marginals"]
MRF_K_COUNT = len(KERNEL_NAMES)

# every symbol include/mrf.h declares
EXPORTS = ["mrf_create", "mrf_add_frame", "mrf_bp_iterate", "mrf_marginals", "mrf_destroy", "mrf_last_error",
           "mrf_set_stream", "mrf_reset", "mrf_reserve", "mrf_graph_sizes", "mrf_layout_sizes", "mrf_k6_path", "mrf_export_graph", "mrf_export_rays", "mrf_evaluate",
           "mrf_export_transpose", "mrf_export_messages", "mrf_import_messages", "mrf_export_beliefs",
           "mrf_bp_partial", "mrf_bp_finish", "mrf_belief_slots", "mrf_nccl_unique_id", "mrf_set_profiling",
           "mrf_profile_read", "mrf_launch_count", "mrf_set_message_mode", "mrf_export_keyframe_average", "mrf_set_sparse_bricks", "mrf_export_bricks", "mrf_set_matrix_free",
           "mrf_set_patch_noise"]


class MrfError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class NoiseDesc(ctypes.Structure):
    _fields_ = [("log_nu", ctypes.POINTER(ctypes.c_float)), ("n_z", ctypes.c_int32), ("n_off", ctypes.c_int32),
                ("z_lo", ctypes.c_double), ("z_hi", ctypes.c_double), ("off_lo", ctypes.c_double),
                ("off_hi", ctypes.c_double), ("margin_min", ctypes.c_double), ("margin_k", ctypes.c_double),
                ("sigma_c", ctypes.c_double * 3)]


class DistDesc(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("comm", ctypes.c_int32),
                ("nccl_id", ctypes.c_ubyte * 128)]


def load(build: bool = True):
    """Load (building first if the sources are newer) the in-tree libmrf.so."""
    global _lib
    with _lock:
        if _lib is None:
            if build:
                _build.build()
            path = os.environ.get("MRF_LIB") or _build.LIB  # MRF_LIB: an in-tree build variant (kernel experiments)
            if not os.path.exists(path):
                raise MrfError(-1, f"{path} missing: run paper_2006_03512_b200._build")
            L = ctypes.CDLL(path)
            P = ctypes.POINTER
            vp, i32, i64, f32, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_double
            st = ctypes.c_int
            sig = {
                "mrf_create": (st, [P(i32), f64, P(f64), f32, P(NoiseDesc), P(DistDesc), P(vp)]),
                "mrf_add_frame": (st, [vp, vp, i32, i32, P(f64), P(f64), P(i64)]),
                "mrf_bp_iterate": (st, [vp, i32]),
                "mrf_marginals": (st, [vp, vp, i32]),
                "mrf_destroy": (st, [vp]),
                "mrf_last_error": (ctypes.c_char_p, [vp]),
                "mrf_set_stream": (st, [vp, vp]),
                "mrf_reset": (st, [vp]),
                "mrf_reserve": (st, [vp, i64, i64]),
                "mrf_graph_sizes": (st, [vp, P(i64), P(i64), P(i64), P(i64), P(i64)]),
                "mrf_layout_sizes": (st, [vp, P(i64), P(i64), P(i64)]),
                "mrf_k6_path": (st, [vp, P(i32)]),
                "mrf_export_rays": (st, [vp, i64, vp, vp, i64, vp, vp, vp, vp]),
                "mrf_evaluate": (st, [vp, vp, i32, i32, P(f64), P(f64), i32, f64, f64, vp, P(i64), P(i64)]),
                "mrf_set_message_mode": (st, [vp, i32]),
                "mrf_export_keyframe_average": (st, [vp, i64, vp]),
                "mrf_set_sparse_bricks": (st, [vp, i32]),
                "mrf_set_matrix_free": (st, [vp, i32]),
                "mrf_set_patch_noise": (st, [vp, i32, i32, i32, P(f64), f64]),
                "mrf_export_bricks": (st, [vp, vp, P(i64)]),
                "mrf_export_graph": (st, [vp, vp, vp, vp, vp]),
                "mrf_export_transpose": (st, [vp, vp, vp]),
                "mrf_export_messages": (st, [vp, vp]),
                "mrf_import_messages": (st, [vp, vp]),
                "mrf_export_beliefs": (st, [vp, vp]),
                "mrf_bp_partial": (st, [vp, i32, vp]),
                "mrf_bp_finish": (st, [vp, vp]),
                "mrf_belief_slots": (i64, [vp]),
                "mrf_nccl_unique_id": (st, [P(ctypes.c_ubyte)]),
                "mrf_set_profiling": (st, [vp, i32]),
                "mrf_profile_read": (st, [vp, P(i64), P(f64)]),
                "mrf_launch_count": (i64, [vp]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def check(status, ctx=None):
    if status != MRF_OK:
        msg = load().mrf_last_error(ctx)
        raise MrfError(status, msg.decode() if msg else "")
