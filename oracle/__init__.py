"""fp64 CPU oracle for the MRFMap hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  It shares no code with paper_2006_03512_b200 (the
CUDA path) and the product never imports it.  The arithmetic lives in
mrf_oracle.c (plain C, fp64, no FMA contraction); this module only marshals
numpy arrays to it and assembles the per-frame CSR in canonical order
(frame add order, pixel index v*W+u, position along the ray).

Every function cites the SURVEY §8(c) step (B1..B7) / PAPER.md lines it follows;
the pins that tie it to the paper are in tests/test_oracle_*.py.  Parity status:
  B1 ray setup, B2 DDA, B3 offsets/LUT, B5 single-ray messages, B5+B6 on tree
  graphs, §III.D evaluation metric (vis_profile / eval_pixel), NEXT #3 keyframe averages
  (kf_*: SPEC's worked examples, and equal to B5 when each keyframe has one ray per voxel),
  NEXT #4 sparse bricks (alloc_bricks / dda_sparse: SPEC's allocation examples and coverage
  post-condition, the filtered brute-force-pinned dense walk, skipped = certainly-empty): pinned.
  NEXT #1 (matrix-free) needs no oracle of its own: it must equal the stored graph bit for bit.  B5+B6 on loopy graphs (several overlapping rays): parity
  unpinned beyond the invariants (loopy BP has no closed form).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mrf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

STATUS_KEPT, STATUS_INVALID, STATUS_DROPPED, STATUS_OTHER_RANK = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -ffp-contract=off -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math",
                               "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _P(t):
    return ctypes.POINTER(t)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            i32p, i64p, dp, fp = _P(ctypes.c_int32), _P(ctypes.c_int64), _P(ctypes.c_double), _P(ctypes.c_float)
            i16p, i8p = _P(ctypes.c_int16), _P(ctypes.c_int8)
            i32, i64, d = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
            L.orc_ray_setup.argtypes = [i32p, dp, dp, dp, dp, i32, i32, ctypes.c_float, i64p, i64p, dp, dp]
            L.orc_ray_setup.restype = ctypes.c_int
            L.orc_dda.argtypes = [i32p, i64p, i64p, d, d, i32p, i16p, dp, dp, i64]
            L.orc_dda.restype = i64
            L.orc_log_nu.argtypes = [fp, i32, i32, dp, d, i32]
            L.orc_log_nu.restype = d
            L.orc_ray_messages.argtypes = [i64, dp, dp, dp, dp, dp]
            L.orc_ray_messages.restype = None
            L.orc_ray_pass.argtypes = [i64, i64p, i32p, i16p, dp, fp, i32, i32, dp, d, dp, dp, dp]
            L.orc_ray_pass.restype = None
            L.orc_accumulate.argtypes = [i64, i32p, dp, i64, dp]
            L.orc_accumulate.restype = None
            L.orc_bp.argtypes = [i64, i64p, i32p, i16p, dp, fp, i32, i32, dp, d, i64, i32, dp, dp, dp]
            L.orc_bp.restype = None
            L.orc_marginals.argtypes = [i64, d, dp, dp]
            L.orc_marginals.restype = None
            L.orc_kf_beliefs.argtypes = [i64, i64, dp, dp]
            L.orc_kf_beliefs.restype = None
            L.orc_kf_average.argtypes = [i64, i64p, i32p, i32p, dp, i64, i64, dp]
            L.orc_kf_average.restype = None
            L.orc_kf_pass.argtypes = [i64, i64p, i32p, i16p, dp, i32p, fp, i32, i32, dp, d, i64, i64, dp, dp, dp]
            L.orc_kf_pass.restype = None
            L.orc_kf_bp.argtypes = [i64, i64p, i32p, i16p, dp, i32p, fp, i32, i32, dp, d, i64, i64, i32, dp, dp, dp, dp]
            L.orc_kf_bp.restype = None
            u8p = _P(ctypes.c_uint8)
            L.orc_frame_count.argtypes = [i32p, dp, dp, dp, dp, i32, i32, fp, i32, i32, i8p, i64p, dp, dp, u8p, i32,
                                          i32p, dp]
            L.orc_frame_count.restype = None
            L.orc_frame_fill.argtypes = [i32p, dp, dp, dp, dp, i32, i32, fp, i64p, i32p, i16p, u8p, i32, i32p, dp]
            L.orc_frame_fill.restype = None
            L.orc_alloc_bricks.argtypes = [i32p, dp, dp, dp, dp, i32, i32, fp, i32, i32p, u8p, dp]
            L.orc_alloc_bricks.restype = i64
            L.orc_dda_sparse.argtypes = [i32p, i64p, i64p, d, d, u8p, i32, i32p, i32p, i16p, dp, dp, i64]
            L.orc_dda_sparse.restype = i64
            L.orc_vis_profile.argtypes = [i64, dp, dp, d, dp, dp]
            L.orc_vis_profile.restype = i64
            L.orc_eval_pixel.argtypes = [i32p, dp, dp, dp, dp, i32, i32, ctypes.c_float, dp, d, d, i32, dp]
            L.orc_eval_pixel.restype = ctypes.c_int
            L.orc_eval_frame.argtypes = [i32p, dp, dp, dp, dp, i32, i32, fp, dp, d, d, i32, i32, i32, i8p, i64p, i64p, dp]
            L.orc_patch_log_nu.argtypes = [i64, i64p, i16p, dp, dp, d, dp]
            L.orc_patch_log_nu.restype = None
            L.orc_eval_frame.restype = None
            L.orc_set_num_threads.argtypes = [i32]
            L.orc_set_num_threads.restype = None
            L.orc_max_threads.argtypes = []
            L.orc_max_threads.restype = i32
            _lib = L
    return _lib


def set_num_threads(n: int):
    """OpenMP threads of the oracle's parallel loops (independent rays / voxels only)."""
    lib().orc_set_num_threads(int(n))


def max_threads() -> int:
    return int(lib().orc_max_threads())


def _ptr(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


class Params:
    """Grid + noise model, as plain arrays for the C entry points."""

    def __init__(self, dims, res, origin, prior, log_nu, z_lo, z_hi, off_lo, off_hi,
                 margin_min, margin_k, sigma_c, patch=None):
        self.dims = _c(dims, np.int32)
        self.geo = _c([res, origin[0], origin[1], origin[2]], np.float64)
        self.par = _c([z_lo, z_hi, off_lo, off_hi, margin_min, margin_k,
                       sigma_c[0], sigma_c[1], sigma_c[2]], np.float64)
        self.lut = _c(log_nu, np.float32)
        self.prior = float(prior)
        self.L0 = math.log(prior / (1.0 - prior))  # prior log-odds of Eq.2
        self.V = int(np.prod(self.dims.astype(np.int64)))
        # learnt per-patch noise model (NEXT #4 option, reading R25): synth.PatchNoise or None
        self.patch = patch

    @classmethod
    def from_workload(cls, w):
        return cls(w.dims, w.res, w.origin, w.prior, w.log_nu, w.z_lo, w.z_hi, w.off_lo, w.off_hi,
                   w.margin_min, w.margin_k, w.sigma_c, getattr(w, "patch", None))

    def pix_sigma(self, W, H):
        """Per-pixel sigma coefficients [H*W, 3] of the patch model (None without one)."""
        if self.patch is None:
            return None
        return _c(self.patch.pixel_coeffs(W, H)[:, 3:6], np.float64)

    def pix_par(self, W, u, v):
        """par of one pixel (the patch's sigma coefficients in place of c0, c1, c2)."""
        if self.patch is None:
            return self.par
        par = self.par.copy()
        par[6:9] = self.patch.coeffs[v // self.patch.patch_px, u // self.patch.patch_px, 3:6]
        return par


# --------------------------------------------------------------------------- B1..B3

def ray_setup(p: Params, K, T_wc, u, v, z, W=None):
    """B1 for one pixel -> (status, G0[3], G1[3], Z, L).  W: the frame width (the pixel's patch of a
    per-patch noise model, reading R25)."""
    par = p.pix_par(W, int(u), int(v)) if (p.patch is not None and W is not None) else p.par
    G0 = np.zeros(3, np.int64)
    G1 = np.zeros(3, np.int64)
    Z = ctypes.c_double(0.0)
    L = ctypes.c_double(0.0)
    K = _c(K, np.float64)
    T = _c(T_wc, np.float64)
    s = lib().orc_ray_setup(_ptr(p.dims, ctypes.c_int32), _ptr(p.geo, ctypes.c_double),
                            _ptr(par, ctypes.c_double), _ptr(K, ctypes.c_double), _ptr(T, ctypes.c_double),
                            int(u), int(v), float(z), _ptr(G0, ctypes.c_int64), _ptr(G1, ctypes.c_int64),
                            ctypes.byref(Z), ctypes.byref(L))
    return s, G0, G1, Z.value, L.value


def dda(dims, G0, G1, Z=0.0, L=1.0):
    """B2+B3 for one fixed-point segment -> (vid, off_q, t_in, t_out)."""
    dims = _c(dims, np.int32)
    G0 = _c(G0, np.int64)
    G1 = _c(G1, np.int64)
    L_ = lib()
    n = L_.orc_dda(_ptr(dims, ctypes.c_int32), _ptr(G0, ctypes.c_int64), _ptr(G1, ctypes.c_int64),
                   float(Z), float(L), None, None, None, None, 0)
    vid = np.zeros(n, np.int32)
    off = np.zeros(n, np.int16)
    tin = np.zeros(n, np.float64)
    tout = np.zeros(n, np.float64)
    L_.orc_dda(_ptr(dims, ctypes.c_int32), _ptr(G0, ctypes.c_int64), _ptr(G1, ctypes.c_int64),
               float(Z), float(L), _ptr(vid, ctypes.c_int32), _ptr(off, ctypes.c_int16),
               _ptr(tin, ctypes.c_double), _ptr(tout, ctypes.c_double), n)
    return vid, off, tin, tout


def log_nu(p: Params, Z, off_q):
    return lib().orc_log_nu(_ptr(p.lut, ctypes.c_float), p.lut.shape[0], p.lut.shape[1],
                            _ptr(p.par, ctypes.c_double), float(Z), int(off_q))


# --------------------------------------------------------------------------- graph

class Graph:
    """Canonical-order CSR of one rank's rays: row_ptr over kept rays, vid, off_q,
    plus per-ray range Z and the flat pixel id (frame, v*W+u)."""

    def __init__(self, row_ptr, vid, off_q, Z, frame, pixel, n_invalid, n_dropped, coef=None):
        self.row_ptr, self.vid, self.off_q, self.Z = row_ptr, vid, off_q, Z
        self.frame, self.pixel = frame, pixel
        self.n_invalid, self.n_dropped = n_invalid, n_dropped
        self.coef = coef  # per-ray patch coefficients [n_rays, 6] of the per-patch model (R25), or None

    @property
    def n_rays(self):
        return len(self.row_ptr) - 1

    @property
    def E(self):
        return int(self.row_ptr[-1])


class Bricks:
    """Brick allocation mask of a sparse map (NEXT #4, reading R23): mask[bz, by, bx] != 0 for an
    allocated brick of B^3 cells."""

    def __init__(self, p: Params, B: int = 8):
        self.B = int(B)
        self.nb = _c([-(-int(d) // self.B) for d in p.dims], np.int32)  # bricks per axis (x, y, z)
        self.mask = np.zeros((int(self.nb[2]), int(self.nb[1]), int(self.nb[0])), np.uint8)

    def cell_mask(self, p: Params):
        """Per-voxel allocation flag, x fastest (V,)."""
        nx, ny, nz = (int(d) for d in p.dims)
        z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        return self.mask[z // self.B, y // self.B, x // self.B].reshape(-1) != 0


def alloc_bricks(p: Params, frames, B: int = 8, bricks: Bricks = None) -> Bricks:
    """SPEC allocate_for_depth_image over the frames, in order -> Bricks (a new mask or the one given)."""
    bk = Bricks(p, B) if bricks is None else bricks
    bk.added = []
    for fr in frames:
        H, W = fr.depth.shape
        ps = p.pix_sigma(W, H)
        bk.added.append(int(lib().orc_alloc_bricks(
            _ptr(p.dims, ctypes.c_int32), _ptr(p.geo, ctypes.c_double), _ptr(p.par, ctypes.c_double),
            _ptr(_c(fr.K, np.float64), ctypes.c_double), _ptr(_c(fr.T_wc, np.float64), ctypes.c_double), W, H,
            _ptr(_c(fr.depth, np.float32), ctypes.c_float), bk.B, _ptr(bk.nb, ctypes.c_int32),
            _ptr(bk.mask, ctypes.c_uint8), _ptr(ps, ctypes.c_double) if ps is not None else None)))
    return bk


def dda_sparse(dims, G0, G1, bricks: Bricks, Z=0.0, L=1.0):
    """B2+B3 with empty skip: the cells of allocated bricks only -> (vid, off_q, t_in, t_out)."""
    dims = _c(dims, np.int32)
    G0 = _c(G0, np.int64)
    G1 = _c(G1, np.int64)
    L_ = lib()
    args = (_ptr(dims, ctypes.c_int32), _ptr(G0, ctypes.c_int64), _ptr(G1, ctypes.c_int64), float(Z), float(L),
            _ptr(bricks.mask, ctypes.c_uint8), bricks.B, _ptr(bricks.nb, ctypes.c_int32))
    n = L_.orc_dda_sparse(*args, None, None, None, None, 0)
    vid = np.zeros(n, np.int32)
    off = np.zeros(n, np.int16)
    tin = np.zeros(n, np.float64)
    tout = np.zeros(n, np.float64)
    L_.orc_dda_sparse(*args, _ptr(vid, ctypes.c_int32), _ptr(off, ctypes.c_int16), _ptr(tin, ctypes.c_double),
                      _ptr(tout, ctypes.c_double), n)
    return vid, off, tin, tout


def build_graph(p: Params, frames, rank: int = 0, world: int = 1, bricks: Bricks = None) -> Graph:
    """B1-B3 over every frame; keeps pixels of rows v % world == rank.  With
    `bricks`, only cells of allocated bricks become incidences (NEXT #4 empty skip, R23)."""
    L_ = lib()
    bm = (_ptr(bricks.mask, ctypes.c_uint8), bricks.B, _ptr(bricks.nb, ctypes.c_int32)) if bricks else (None, 0, None)
    parts = []
    total = 0
    n_inv = n_drop = 0
    for fi, fr in enumerate(frames):
        H, W = fr.depth.shape
        depth = _c(fr.depth, np.float32)
        K = _c(fr.K, np.float64)
        T = _c(fr.T_wc, np.float64)
        status = np.zeros(H * W, np.int8)
        count = np.zeros(H * W, np.int64)
        Z = np.zeros(H * W, np.float64)
        Lr = np.zeros(H * W, np.float64)
        ps = p.pix_sigma(W, H)
        psp = _ptr(ps, ctypes.c_double) if ps is not None else None
        L_.orc_frame_count(_ptr(p.dims, ctypes.c_int32), _ptr(p.geo, ctypes.c_double), _ptr(p.par, ctypes.c_double),
                           _ptr(K, ctypes.c_double), _ptr(T, ctypes.c_double), W, H, _ptr(depth, ctypes.c_float),
                           rank, world, _ptr(status, ctypes.c_int8), _ptr(count, ctypes.c_int64),
                           _ptr(Z, ctypes.c_double), _ptr(Lr, ctypes.c_double), *bm, psp)
        kept = np.nonzero(status == STATUS_KEPT)[0]
        n_inv += int(np.sum(status == STATUS_INVALID))
        n_drop += int(np.sum(status == STATUS_DROPPED))
        cf = p.patch.pixel_coeffs(W, H)[kept] if p.patch is not None else None
        parts.append((fi, depth, K, T, W, H, kept, count[kept], Z[kept], cf, ps))
        total += int(count[kept].sum())
    vid = np.zeros(total, np.int32)
    off_q = np.zeros(total, np.int16)
    row_ptr = [np.zeros(1, np.int64)]
    Zs, fids, pix, cfs = [], [], [], []
    base = 0
    for fi, depth, K, T, W, H, kept, cnt, Z, cf, ps in parts:
        offs = np.full(H * W, -1, np.int64)
        starts = base + np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.int64) if len(cnt) else np.zeros(0, np.int64)
        offs[kept] = starts
        L_.orc_frame_fill(_ptr(p.dims, ctypes.c_int32), _ptr(p.geo, ctypes.c_double), _ptr(p.par, ctypes.c_double),
                          _ptr(K, ctypes.c_double), _ptr(T, ctypes.c_double), W, H, _ptr(depth, ctypes.c_float),
                          _ptr(offs, ctypes.c_int64), _ptr(vid, ctypes.c_int32), _ptr(off_q, ctypes.c_int16), *bm,
                          _ptr(ps, ctypes.c_double) if ps is not None else None)
        cfs.append(cf)
        row_ptr.append(base + np.cumsum(cnt).astype(np.int64))
        base += int(cnt.sum())
        Zs.append(Z)
        fids.append(np.full(len(kept), fi, np.int32))
        pix.append(kept.astype(np.int64))
    return Graph(np.concatenate(row_ptr), vid, off_q, np.concatenate(Zs) if Zs else np.zeros(0),
                 np.concatenate(fids) if fids else np.zeros(0, np.int32),
                 np.concatenate(pix) if pix else np.zeros(0, np.int64), n_inv, n_drop,
                 (np.concatenate(cfs) if cfs else np.zeros((0, 6))) if p.patch is not None else None)


def trace_pixels(p: Params, frame, pixels, frame_index: int = 0, bricks: Bricks = None) -> Graph:
    """B1-B3 for selected pixel ids (v*W+u) of one frame, one by one (sampled parity at full
    size).  Only kept pixels (status 0) become rays, in the order given.  With `bricks`, the
    empty-skip walk (NEXT #4)."""
    H, W = frame.depth.shape
    row_ptr = [0]
    vids, offs, Zs, pix = [], [], [], []
    n_inv = n_drop = 0
    for px in pixels:
        v, u = divmod(int(px), W)
        s, G0, G1, Z, L = ray_setup(p, frame.K, frame.T_wc, u, v, float(frame.depth[v, u]), W)
        if s == STATUS_INVALID:
            n_inv += 1
            continue
        if s == STATUS_DROPPED:
            n_drop += 1
            continue
        vid, off, _, _ = dda(p.dims, G0, G1, Z, L) if bricks is None else dda_sparse(p.dims, G0, G1, bricks, Z, L)
        vids.append(vid)
        offs.append(off)
        row_ptr.append(row_ptr[-1] + len(vid))
        Zs.append(Z)
        pix.append(int(px))
    cat = lambda a, t: np.concatenate(a).astype(t) if a else np.zeros(0, t)  # noqa: E731
    coef = None
    if p.patch is not None:
        coef = p.patch.pixel_coeffs(W, H)[np.array(pix, np.int64)] if pix else np.zeros((0, 6))
    return Graph(np.array(row_ptr, np.int64), cat(vids, np.int32), cat(offs, np.int16), np.array(Zs),
                 np.full(len(pix), frame_index, np.int32), np.array(pix, np.int64), n_inv, n_drop, coef)


# --------------------------------------------------------------------------- B4..B6

def patch_log_nu(p: Params, g: Graph):
    """log nu of every incidence under the per-patch model (R25) -> float64[E], or None when the
    map uses the global LUT."""
    if p.patch is None or g.coef is None:
        return None
    lnu = np.zeros(g.E)
    lib().orc_patch_log_nu(g.n_rays, _ptr(g.row_ptr, ctypes.c_int64), _ptr(g.off_q, ctypes.c_int16),
                           _ptr(_c(g.Z, np.float64), ctypes.c_double), _ptr(_c(g.coef, np.float64), ctypes.c_double),
                           float(p.patch.sigma_min), _ptr(lnu, ctypes.c_double))
    return lnu


def _lnu_arg(p, g):
    lnu = patch_log_nu(p, g)
    return (_ptr(lnu, ctypes.c_double) if lnu is not None else None), lnu


def ray_messages(c, lnu):
    """B5 core for one ray: (lpos, lneg) = log of Eq.13 / Eq.14 messages."""
    c = _c(c, np.float64)
    lnu = _c(lnu, np.float64)
    n = len(c)
    lpos = np.zeros(n)
    lneg = np.zeros(n)
    work = np.zeros(5 * max(n, 1))
    lib().orc_ray_messages(n, _ptr(c, ctypes.c_double), _ptr(lnu, ctypes.c_double), _ptr(lpos, ctypes.c_double),
                           _ptr(lneg, ctypes.c_double), _ptr(work, ctypes.c_double))
    return lpos, lneg


def ray_pass(p: Params, g: Graph, T, lam):
    """One flooding pass (B5) in place on lam (float64[E]) from snapshot T (float64[V])."""
    T = _c(T, np.float64)
    assert lam.dtype == np.float64 and lam.flags.c_contiguous
    le, _keep = _lnu_arg(p, g)
    lib().orc_ray_pass(g.n_rays, _ptr(g.row_ptr, ctypes.c_int64), _ptr(g.vid, ctypes.c_int32),
                       _ptr(g.off_q, ctypes.c_int16), _ptr(_c(g.Z, np.float64), ctypes.c_double),
                       _ptr(p.lut, ctypes.c_float), p.lut.shape[0], p.lut.shape[1], _ptr(p.par, ctypes.c_double),
                       p.L0, _ptr(T, ctypes.c_double), _ptr(lam, ctypes.c_double), le)
    return lam


def accumulate(p: Params, g: Graph, lam):
    T = np.zeros(p.V)
    lib().orc_accumulate(g.E, _ptr(g.vid, ctypes.c_int32), _ptr(_c(lam, np.float64), ctypes.c_double),
                         p.V, _ptr(T, ctypes.c_double))
    return T


def bp(p: Params, g: Graph, n_iter: int, lam=None):
    """B4 (lam = 0) + n flooding iterations (B5, B7) -> (lam, T)."""
    lam = np.zeros(g.E) if lam is None else _c(lam, np.float64).copy()
    T = np.zeros(p.V)
    le, _keep = _lnu_arg(p, g)
    lib().orc_bp(g.n_rays, _ptr(g.row_ptr, ctypes.c_int64), _ptr(g.vid, ctypes.c_int32),
                 _ptr(g.off_q, ctypes.c_int16), _ptr(_c(g.Z, np.float64), ctypes.c_double),
                 _ptr(p.lut, ctypes.c_float), p.lut.shape[0], p.lut.shape[1], _ptr(p.par, ctypes.c_double),
                 p.L0, p.V, int(n_iter), _ptr(lam, ctypes.c_double), _ptr(T, ctypes.c_double), le)
    return lam, T


def marginals(p: Params, T):
    """B6: p_v = sigma(L0 + T_v) (Eq.8)."""
    T = _c(T, np.float64)
    out = np.zeros(len(T))
    lib().orc_marginals(len(T), p.L0, _ptr(T, ctypes.c_double), _ptr(out, ctypes.c_double))
    return out


# --------------------------------------------------------------------------- NEXT #3

def kf_average(g: Graph, lam, F: int, V: int):
    """Keyframe averages (SPEC accumulate_outgoing): lbar[f, v] = log(mean sigma(lam) /
    mean sigma(-lam)) over keyframe f's incidences of v, 0 where f has none."""
    lbar = np.zeros(F * V)
    lib().orc_kf_average(g.n_rays, _ptr(g.row_ptr, ctypes.c_int64), _ptr(g.vid, ctypes.c_int32),
                         _ptr(_c(g.frame, np.int32), ctypes.c_int32), _ptr(_c(lam, np.float64), ctypes.c_double),
                         F, V, _ptr(lbar, ctypes.c_double))
    return lbar.reshape(F, V)


def kf_beliefs(lbar):
    """T_v = sum_f lbar[f, v] (one message per keyframe)."""
    lbar = _c(lbar, np.float64)
    F, V = lbar.shape
    T = np.zeros(V)
    lib().orc_kf_beliefs(F, V, _ptr(lbar, ctypes.c_double), _ptr(T, ctypes.c_double))
    return T


def kf_pass(p: Params, g: Graph, lbar):
    """One flooding pass of the keyframe-average variant from the snapshot lbar[F, V] ->
    per-incidence messages (cavity excludes the ray's whole keyframe)."""
    lbar = _c(lbar, np.float64)
    F, V = lbar.shape
    lam = np.zeros(g.E)
    le, _keep = _lnu_arg(p, g)
    lib().orc_kf_pass(g.n_rays, _ptr(g.row_ptr, ctypes.c_int64), _ptr(g.vid, ctypes.c_int32),
                      _ptr(g.off_q, ctypes.c_int16), _ptr(_c(g.Z, np.float64), ctypes.c_double),
                      _ptr(_c(g.frame, np.int32), ctypes.c_int32), _ptr(p.lut, ctypes.c_float), p.lut.shape[0],
                      p.lut.shape[1], _ptr(p.par, ctypes.c_double), p.L0, F, V, _ptr(lbar, ctypes.c_double),
                      _ptr(lam, ctypes.c_double), le)
    return lam


def kf_bp(p: Params, g: Graph, n_iter: int, F: int, lbar=None):
    """n iterations of the keyframe-average variant -> (lam, lbar[F, V], T)."""
    lbar = np.zeros((F, p.V)) if lbar is None else _c(lbar, np.float64).copy()
    lam = np.zeros(g.E)
    T = np.zeros(p.V)
    le, _keep = _lnu_arg(p, g)
    lib().orc_kf_bp(g.n_rays, _ptr(g.row_ptr, ctypes.c_int64), _ptr(g.vid, ctypes.c_int32),
                    _ptr(g.off_q, ctypes.c_int16), _ptr(_c(g.Z, np.float64), ctypes.c_double),
                    _ptr(_c(g.frame, np.int32), ctypes.c_int32), _ptr(p.lut, ctypes.c_float), p.lut.shape[0],
                    p.lut.shape[1], _ptr(p.par, ctypes.c_double), p.L0, F, p.V, int(n_iter),
                    _ptr(lam, ctypes.c_double), _ptr(lbar, ctypes.c_double), _ptr(T, ctypes.c_double), le)
    return lam, lbar, T


def run(workload, n_iter=None, rank=0, world=1):
    """Convenience: graph + BP + marginals for a synth.Workload."""
    p = Params.from_workload(workload)
    g = build_graph(p, workload.frames, rank, world)
    lam, T = bp(p, g, workload.n_iter if n_iter is None else n_iter)
    return p, g, lam, T, marginals(p, T)


# --------------------------------------------------------------------------- §III.D metric

def vis_profile(x, ell, res):
    """Visibility / generating-surface density along one ray (Eq.15-18):
    per step occupancy log-odds x_i and traversed length ell_i -> (ln vis[0..n], ln omega[0..n-1],
    argmax_i ln omega_i or -1)."""
    x = _c(x, np.float64)
    ell = _c(ell, np.float64)
    n = len(x)
    lvis = np.zeros(n + 1)
    lom = np.zeros(max(n, 1))
    best = lib().orc_vis_profile(n, _ptr(x, ctypes.c_double), _ptr(ell, ctypes.c_double), float(res),
                                 _ptr(lvis, ctypes.c_double), _ptr(lom, ctypes.c_double))
    return lvis, lom[:n], int(best)


def eval_pixel(p: Params, frame, u, v, xmap, k_sigma=1.5, vis_thr=0.5, mode=0):
    """One pixel against the map xmap[V] (occupancy log-odds): (class, Z, s*, s_inf, vis_inf).
    mode 0: 1.5-sigma band around s* (§V); mode 1: Z inside the argmax voxel (§III.D)."""
    out = np.zeros(4)
    K = _c(frame.K, np.float64)
    T = _c(frame.T_wc, np.float64)
    xm = _c(xmap, np.float64)
    par = p.pix_par(frame.depth.shape[1], int(u), int(v))
    r = lib().orc_eval_pixel(_ptr(p.dims, ctypes.c_int32), _ptr(p.geo, ctypes.c_double), _ptr(par, ctypes.c_double),
                             _ptr(K, ctypes.c_double), _ptr(T, ctypes.c_double), int(u), int(v),
                             float(frame.depth[v, u]), _ptr(xm, ctypes.c_double), float(k_sigma), float(vis_thr),
                             int(mode), _ptr(out, ctypes.c_double))
    return (int(r),) + tuple(float(a) for a in out)


def eval_frame(p: Params, frame, xmap, k_sigma=1.5, vis_thr=0.5, rank=0, world=1, mode=0):
    """§V per-image accuracy: per-pixel class (-1 invalid, 0 / 1, -2 other rank), n_valid,
    n_accurate."""
    H, W = frame.depth.shape
    cls = np.zeros(H * W, np.int8)
    nv = ctypes.c_int64()
    na = ctypes.c_int64()
    depth = _c(frame.depth, np.float32)
    K = _c(frame.K, np.float64)
    T = _c(frame.T_wc, np.float64)
    xm = _c(xmap, np.float64)
    ps = p.pix_sigma(W, H)
    lib().orc_eval_frame(_ptr(p.dims, ctypes.c_int32), _ptr(p.geo, ctypes.c_double), _ptr(p.par, ctypes.c_double),
                         _ptr(K, ctypes.c_double), _ptr(T, ctypes.c_double), W, H, _ptr(depth, ctypes.c_float),
                         _ptr(xm, ctypes.c_double), float(k_sigma), float(vis_thr), int(mode), rank, world,
                         _ptr(cls, ctypes.c_int8), ctypes.byref(nv), ctypes.byref(na),
                         _ptr(ps, ctypes.c_double) if ps is not None else None)
    return cls.reshape(H, W), nv.value, na.value
