"""B200-native MRFMap hot path (arxiv 2006.03512): ray-voxel factor graph + loopy BP.

Thin Python layer over the C ABI in include/mrf.h (libmrf.so, CUDA for sm_100a).  The
functions of `_lib` keep the C names; `MRFMap` only marshals numpy arrays / torch tensors
to pointers.  PyTorch is used for device memory, streams and process groups only.

    m = MRFMap(dims, res, origin, prior, log_nu, z_lo, z_hi, off_lo, off_hi, margin_min, margin_k, sigma_c)
    m.add_frame(depth, K, T_wc)      # mrf_add_frame
    m.bp_iterate(n)                  # mrf_bp_iterate  (Eq.13/14 + Eq.6)
    p = m.marginals()                # mrf_marginals   (Eq.8)
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import MrfError, KERNEL_NAMES, MRF_COMM_NCCL, MRF_COMM_EXTERNAL  # noqa: F401
from ._lib import MRF_MSG_PER_RAY, MRF_MSG_KEYFRAME_AVG  # noqa: F401

__all__ = ["MRFMap", "MrfError", "nccl_unique_id", "load"]


def load():
    return _lib.load()


def _ptr(a):
    """Pointer of a numpy array (host) or torch tensor (host/device)."""
    if isinstance(a, np.ndarray):
        assert a.flags.c_contiguous
        return ctypes.c_void_p(a.ctypes.data)
    if hasattr(a, "data_ptr"):
        assert a.is_contiguous()
        return ctypes.c_void_p(a.data_ptr())
    raise TypeError(type(a))


def _is_device(a):
    return hasattr(a, "is_cuda") and a.is_cuda


def nccl_unique_id() -> bytes:
    L = _lib.load()
    buf = (ctypes.c_ubyte * 128)()
    _lib.check(L.mrf_nccl_unique_id(buf))
    return bytes(buf)


class MRFMap:
    """One rank's share of the map (the whole map when world == 1)."""

    def __init__(self, dims, res, origin, prior, log_nu, z_lo, z_hi, off_lo, off_hi, margin_min=0.1,
                 margin_k=3.0, sigma_c=(0.0, 0.0, 0.0012), rank=0, world=1, comm=MRF_COMM_NCCL, nccl_id=None):
        self._L = _lib.load()
        self._brick = 0
        self.dims = tuple(int(d) for d in dims)
        self.V = self.dims[0] * self.dims[1] * self.dims[2]
        self.prior = float(prior)
        self._lut = np.ascontiguousarray(log_nu, dtype=np.float32)
        nd = _lib.NoiseDesc()
        nd.log_nu = self._lut.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        nd.n_z, nd.n_off = self._lut.shape
        nd.z_lo, nd.z_hi, nd.off_lo, nd.off_hi = z_lo, z_hi, off_lo, off_hi
        nd.margin_min, nd.margin_k = margin_min, margin_k
        nd.sigma_c[0], nd.sigma_c[1], nd.sigma_c[2] = sigma_c
        dims_a = (ctypes.c_int32 * 3)(*self.dims)
        org = (ctypes.c_double * 3)(*origin)
        dist = None
        self.rank, self.world = int(rank), int(world)
        if world > 1 or comm != MRF_COMM_NCCL:
            dd = _lib.DistDesc()
            dd.rank, dd.world, dd.comm = rank, world, comm
            if nccl_id is not None:
                ctypes.memmove(dd.nccl_id, bytes(nccl_id), 128)
            dist = ctypes.byref(dd)
        h = ctypes.c_void_p()
        st = self._L.mrf_create(dims_a, float(res), org, float(prior), ctypes.byref(nd), dist, ctypes.byref(h))
        if st != 0:
            msg = self._L.mrf_last_error(None)
            raise MrfError(st, msg.decode() if msg else "")
        self._h = h

    @classmethod
    def from_workload(cls, w, **kw):
        m = cls(w.dims, w.res, w.origin, w.prior, w.log_nu, w.z_lo, w.z_hi, w.off_lo, w.off_hi,
                w.margin_min, w.margin_k, w.sigma_c, **kw)
        if getattr(w, "patch", None) is not None:  # the learnt per-patch sensor model (R25)
            m.set_patch_noise(w.patch.patch_px, w.patch.coeffs, w.patch.sigma_min)
        return m

    # ------------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "_h", None):
            self._L.mrf_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _chk(self, st):
        _lib.check(st, self._h)

    # ------------------------------------------------------------------ hot path
    def add_frame(self, depth, K, T_wc) -> int:
        """mrf_add_frame: depth [H, W] float32 (numpy or torch, host or cuda)."""
        if isinstance(depth, np.ndarray):
            depth = np.ascontiguousarray(depth, dtype=np.float32)
        H, W = depth.shape
        Ka = (ctypes.c_double * 4)(*[float(x) for x in K])
        Ta = (ctypes.c_double * 12)(*[float(x) for x in np.asarray(T_wc, dtype=np.float64).reshape(-1)])
        fid = ctypes.c_int64()
        self._chk(self._L.mrf_add_frame(self._h, _ptr(depth), W, H, Ka, Ta, ctypes.byref(fid)))
        return fid.value

    def bp_iterate(self, n: int):
        self._chk(self._L.mrf_bp_iterate(self._h, int(n)))

    def marginals(self, out=None):
        """mrf_marginals -> float32 [V] (x fastest); `out` may be a cuda tensor."""
        if out is None:
            out = np.empty(self.V, np.float32)
        self._chk(self._L.mrf_marginals(self._h, _ptr(out), 1 if _is_device(out) else 0))
        return out

    # ------------------------------------------------------------------ runtime / introspection
    def set_stream(self, stream_ptr: int):
        self._chk(self._L.mrf_set_stream(self._h, ctypes.c_void_p(stream_ptr)))

    def reset(self):
        self._chk(self._L.mrf_reset(self._h))

    def reserve(self, n_rays, n_incidences):
        self._chk(self._L.mrf_reserve(self._h, int(n_rays), int(n_incidences)))

    def graph_sizes(self, active=True) -> dict:
        v = [ctypes.c_int64() for _ in range(5)]
        self._chk(self._L.mrf_graph_sizes(self._h, ctypes.byref(v[0]), ctypes.byref(v[1]),
                                          ctypes.byref(v[2]) if active else None, ctypes.byref(v[3]),
                                          ctypes.byref(v[4])))
        return dict(n_rays=v[0].value, E=v[1].value, n_active=v[2].value if active else None,
                    n_invalid=v[3].value, n_dropped=v[4].value)

    def layout_sizes(self) -> dict:
        """mrf_layout_sizes: padded incidence slots, K6 tile runs, belief slots."""
        v = [ctypes.c_int64() for _ in range(3)]
        self._chk(self._L.mrf_layout_sizes(self._h, *(ctypes.byref(x) for x in v)))
        return dict(n_slots=v[0].value, n_runs=v[1].value, n_belief_slots=v[2].value)

    def k6_path(self) -> str:
        """mrf_k6_path: "block" (K6b, the pixel-block hash reduction) or "tile" (tile runs)."""
        v = ctypes.c_int32()
        self._chk(self._L.mrf_k6_path(self._h, ctypes.byref(v)))
        return "block" if v.value == 1 else "tile"

    def evaluate(self, depth, K, T_wc, k_sigma=1.5, vis_threshold=0.5, mode=0):
        """mrf_evaluate: §III.D generating-surface accuracy of one posed depth image against the
        current beliefs -> (cls[H, W] int8, n_valid, n_accurate) for this rank's rows.
        mode 0: k_sigma band around s* (§V); mode 1: Z inside the argmax voxel (§III.D)."""
        is_dev = _is_device(depth)
        H, W = (depth.shape if hasattr(depth, "shape") else np.shape(depth))
        if not is_dev:
            depth = np.ascontiguousarray(depth, dtype=np.float32)
        K = np.ascontiguousarray(K, dtype=np.float64)
        T_wc = np.ascontiguousarray(T_wc, dtype=np.float64).reshape(-1)
        cls = np.zeros((H, W), np.int8)
        nv, na = ctypes.c_int64(), ctypes.c_int64()
        self._chk(self._L.mrf_evaluate(self._h, _ptr(depth), W, H, K.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                       T_wc.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), int(mode), float(k_sigma),
                                       float(vis_threshold), _ptr(cls), ctypes.byref(nv), ctypes.byref(na)))
        return cls, nv.value, na.value

    def export_rays(self, frame, pixel):
        """mrf_export_rays: incidence lists of the selected (frame, pixel) rays of this rank."""
        frame = np.ascontiguousarray(frame, dtype=np.int32)
        pixel = np.ascontiguousarray(pixel, dtype=np.int64)
        n = len(frame)
        row_ptr = np.zeros(n + 1, np.int64)
        self._chk(self._L.mrf_export_rays(self._h, n, _ptr(frame), _ptr(pixel), 0, _ptr(row_ptr), None, None, None))
        cap = int(row_ptr[-1])
        vid = np.zeros(max(cap, 1), np.int32)
        off_q = np.zeros(max(cap, 1), np.int16)
        lam = np.zeros(max(cap, 1), np.float32)
        self._chk(self._L.mrf_export_rays(self._h, n, _ptr(frame), _ptr(pixel), cap, _ptr(row_ptr), _ptr(vid),
                                          _ptr(off_q), _ptr(lam)))
        return dict(row_ptr=row_ptr, vid=vid[:cap], off_q=off_q[:cap], lam=lam[:cap])

    def export_graph(self):
        s = self.graph_sizes(active=False)
        ray_pixel = np.empty(s["n_rays"], np.int64)
        row_ptr = np.empty(s["n_rays"] + 1, np.int64)
        vid = np.empty(s["E"], np.int32)
        off_q = np.empty(s["E"], np.int16)
        self._chk(self._L.mrf_export_graph(self._h, _ptr(ray_pixel), _ptr(row_ptr), _ptr(vid), _ptr(off_q)))
        return dict(frame=(ray_pixel >> 32).astype(np.int32), pixel=ray_pixel & 0xffffffff, row_ptr=row_ptr,
                    vid=vid, off_q=off_q)

    def export_transpose(self):
        s = self.graph_sizes(active=False)
        col_ptr = np.empty(self.V + 1, np.int64)
        tr = np.empty(max(s["E"], 1), np.int32)
        self._chk(self._L.mrf_export_transpose(self._h, _ptr(col_ptr), _ptr(tr)))
        return col_ptr, tr[:s["E"]]

    def export_messages(self):
        E = self.graph_sizes(active=False)["E"]
        lam = np.empty(max(E, 1), np.float32)
        self._chk(self._L.mrf_export_messages(self._h, _ptr(lam)))
        return lam[:E]

    def import_messages(self, lam):
        lam = np.ascontiguousarray(lam, dtype=np.float32)
        self._chk(self._L.mrf_import_messages(self._h, _ptr(lam)))

    def set_message_mode(self, mode):
        """mrf_set_message_mode: MRF_MSG_PER_RAY (default) or MRF_MSG_KEYFRAME_AVG (the paper's
        per-keyframe average message; before the first frame, single rank)."""
        self._chk(self._L.mrf_set_message_mode(self._h, int(mode)))

    def export_keyframe_average(self, frame):
        """mrf_export_keyframe_average: the frame's average log-odds per voxel (float32[V],
        x fastest) in keyframe-average mode."""
        out = np.empty(self.V, np.float32)
        self._chk(self._L.mrf_export_keyframe_average(self._h, int(frame), _ptr(out)))
        return out

    def set_matrix_free(self, frames_per_chunk=4):
        """mrf_set_matrix_free: keep only the messages and the tile runs; re-walk the rays of each
        chunk of frames_per_chunk frames before every message pass (0 = stored graph)."""
        self._chk(self._L.mrf_set_matrix_free(self._h, int(frames_per_chunk)))

    def set_patch_noise(self, patch_px, coeffs, sigma_min=1e-4):
        """mrf_set_patch_noise: coeffs [n_py, n_px, 6] (b0, b1, b2, s0, s1, s2 per patch of
        patch_px x patch_px pixels); patch_px = 0 returns to the table."""
        if int(patch_px) == 0:
            self._chk(self._L.mrf_set_patch_noise(self._h, 0, 0, 0, None, 1.0))
            return
        c = np.ascontiguousarray(coeffs, dtype=np.float64)
        if c.ndim != 3 or c.shape[2] != 6:
            raise ValueError("coeffs must be [n_py, n_px, 6]")
        self._chk(self._L.mrf_set_patch_noise(self._h, int(patch_px), int(c.shape[1]), int(c.shape[0]),
                                              c.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), float(sigma_min)))

    def set_sparse_bricks(self, brick=8):
        """mrf_set_sparse_bricks: brick-sparse map with B^3 bricks allocated around the
        reprojected depth points and empty-skip ray walks; 0 = dense."""
        self._chk(self._L.mrf_set_sparse_bricks(self._h, int(brick)))
        self._brick = int(brick)

    def export_bricks(self):
        """mrf_export_bricks -> uint8[nbz, nby, nbx] allocation mask (1 = allocated)."""
        B = self._brick
        if B == 0:  # dense map: the library reports the state error
            self._chk(self._L.mrf_export_bricks(self._h, None, None))
        nx, ny, nz = self.dims
        out = np.zeros((-(-nz // B), -(-ny // B), -(-nx // B)), np.uint8)
        n = ctypes.c_int64()
        self._chk(self._L.mrf_export_bricks(self._h, _ptr(out), ctypes.byref(n)))
        assert n.value == int(np.count_nonzero(out))
        return out

    def export_beliefs(self):
        T = np.empty(self.V, np.int64)
        self._chk(self._L.mrf_export_beliefs(self._h, _ptr(T)))
        return T

    def bp_partial(self, partial_out, iterate=True):
        self._chk(self._L.mrf_bp_partial(self._h, 1 if iterate else 0, _ptr(partial_out)))

    def belief_slots(self) -> int:
        return int(self._L.mrf_belief_slots(self._h))

    def bp_finish(self, total):
        self._chk(self._L.mrf_bp_finish(self._h, _ptr(total)))

    def set_profiling(self, on=True):
        self._chk(self._L.mrf_set_profiling(self._h, 1 if on else 0))

    def profile_read(self) -> dict:
        n = (ctypes.c_int64 * _lib.MRF_K_COUNT)()
        ms = (ctypes.c_double * _lib.MRF_K_COUNT)()
        self._chk(self._L.mrf_profile_read(self._h, n, ms))
        return {k: (n[i], ms[i]) for i, k in enumerate(KERNEL_NAMES)}

    def launch_count(self) -> int:
        return int(self._L.mrf_launch_count(self._h))
