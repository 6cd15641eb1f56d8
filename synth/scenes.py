"""Seeded synthetic scenes, cameras and depth frames (SURVEY.md §8(d) generator spec).

The paper measures on ICL-NUIM livingroom1, a Gazebo scene
and a D435/Kinect capture; none is available, so these seeded scenes
stand in for them with the paper's shapes: 640x480 Kinect-style frames
(fx=fy=525), 0.02-0.05 m voxels, room-scale volumes and tens of keyframes
(P:290).  BASELINE.json `configs` fixes the five workloads.

Conventions (shared by both sides of every parity test):
  * pinhole camera, OpenCV axes (x right, y down, z forward), pixel centres at
    integer (u, v); x_c = (u-cx)/fx, y_c = (v-cy)/fy;
  * T_wc is 3x4 row-major world-from-camera [R | C];
  * depth images hold fp32 z-depth in metres, 0 = invalid.
Sub-streams of numpy default_rng: scene=seed, trajectory=seed+1,
noise=seed+2, invalid mask=seed+3.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .lut import build_log_nu_lut, OUTLIER_LO, OUTLIER_HI

INSET = 0.15  # walls/floor inset from the grid faces


@dataclass
class Frame:
    depth: np.ndarray          # float32 [H, W] z-depth (m), 0 = invalid
    K: np.ndarray              # float64 [4] fx, fy, cx, cy
    T_wc: np.ndarray           # float64 [12] row-major 3x4 world-from-camera

    @property
    def height(self) -> int:
        return int(self.depth.shape[0])

    @property
    def width(self) -> int:
        return int(self.depth.shape[1])


@dataclass
class Workload:
    name: str
    dims: tuple                # (nx, ny, nz) voxels
    res: float                 # voxel side (m)
    origin: tuple              # grid origin (m)
    prior: float               # gamma (Eq.2)
    log_nu: np.ndarray         # float32 [n_z, n_off]
    z_lo: float
    z_hi: float
    off_lo: float
    off_hi: float
    margin_min: float
    margin_k: float
    sigma_c: tuple
    n_iter: int
    frames: list = field(default_factory=list)
    seed: int = 0
    patch: "PatchNoise" = None   # learnt per-patch noise model (NEXT #4 option, reading R25); None: the LUT

    @property
    def n_voxels(self) -> int:
        return int(self.dims[0]) * int(self.dims[1]) * int(self.dims[2])

    def noise_kwargs(self) -> dict:
        return dict(log_nu=self.log_nu, z_lo=self.z_lo, z_hi=self.z_hi,
                    off_lo=self.off_lo, off_hi=self.off_hi,
                    margin_min=self.margin_min, margin_k=self.margin_k,
                    sigma_c=self.sigma_c)


# --------------------------------------------------------------------------- per-patch noise

@dataclass
class PatchNoise:
    """The paper's learnt sensor model: per 20x20-pixel patch a 2nd-degree polynomial
    bias b(d) = b0 + b1 d + b2 d^2 and standard deviation s(d) = s0 + s1 d + s2 d^2 of the measured
    range given the true range d ("fit a 2nd degree polynomial"; the measurement is
    distributed around the bias-predicted mean with the learnt noise).  Synthetic here:
    no calibration data exists; the coefficients are seeded smooth fields around the global model."""
    patch_px: int
    coeffs: np.ndarray          # float64 [n_py, n_px, 6]: b0, b1, b2, s0, s1, s2
    sigma_min: float = 1e-4

    def pixel_coeffs(self, W, H):
        """[H*W, 6] per pixel (patch (u // patch_px, v // patch_px))."""
        v, u = np.divmod(np.arange(W * H), W)
        return self.coeffs[v // self.patch_px, u // self.patch_px].reshape(W * H, 6)


def patch_noise_model(W, H, seed=0, patch_px=20, sigma_c=(0.0, 0.0, 0.0012), bias_amp=4e-4, sigma_spread=0.3):
    """Seeded per-patch coefficients: s2 = c2 (1 + sigma_spread f), b2 = bias_amp g, with f, g
    smooth fields in [-1, 1] over the patch grid (a vignetting-like pattern plus a random phase)."""
    n_px, n_py = -(-W // patch_px), -(-H // patch_px)
    rs = np.random.default_rng(seed + 5)
    ph = rs.uniform(0, 2 * math.pi, 4)
    x = (np.arange(n_px) + 0.5) / n_px - 0.5
    y = (np.arange(n_py) + 0.5) / n_py - 0.5
    X, Y = np.meshgrid(x, y)
    f = np.clip(2.0 * (X * X + Y * Y) - 0.25 + 0.25 * np.sin(2 * math.pi * X + ph[0]) * np.cos(2 * math.pi * Y + ph[1]),
                -1.0, 1.0)
    g = np.sin(math.pi * X + ph[2]) * np.cos(math.pi * Y + ph[3])
    c = np.zeros((n_py, n_px, 6))
    c[..., 3], c[..., 4] = sigma_c[0], sigma_c[1]
    c[..., 5] = sigma_c[2] * (1.0 + sigma_spread * f)
    c[..., 2] = bias_amp * g
    return PatchNoise(patch_px, c)


# --------------------------------------------------------------------------- geometry

class _Scene:
    """Axis-aligned rectangles, axis-aligned boxes and z-rotated boxes."""

    def __init__(self):
        self.rects = []   # (axis, coord, lo2[2], hi2[2]) : plane x_axis = coord, bounds on the other axes
        self.boxes = []   # (lo[3], hi[3])
        self.obbs = []    # (centre[3], half[3], yaw)

    def render_depth(self, W, H, K, R, C) -> np.ndarray:
        """Exact fp64 nearest hit per pixel (C renderer); returns z-depth t (inf = no hit).

        Rays are C + t * (R @ (x_c, y_c, 1)), so t is the camera z-depth.
        """
        rects = [(ax, co, lo2[0], lo2[1], hi2[0], hi2[1]) for ax, co, lo2, hi2 in self.rects]
        boxes = [tuple(lo) + tuple(hi) for lo, hi in self.boxes]
        obbs = [tuple(c) + tuple(h) + (yaw,) for c, h, yaw in self.obbs]
        return _native.render(W, H, K, R, C, rects, boxes, obbs)


def _room(scene: _Scene, size, with_back_wall_only=False):
    sx, sy, sz = size
    lo, hx, hy, hz = INSET, sx - INSET, sy - INSET, sz - INSET
    # walls (no ceiling: "walls and floor")
    scene.rects.append((0, lo, (lo, lo), (hy, hz)))
    scene.rects.append((0, hx, (lo, lo), (hy, hz)))
    scene.rects.append((1, lo, (lo, lo), (hx, hz)))
    scene.rects.append((1, hx, (lo, lo), (hx, hz)))
    scene.rects.append((2, lo, (lo, lo), (hx, hy)))


def _camera_rotation(yaw: float, pitch: float = 0.0) -> np.ndarray:
    """World-from-camera rotation, optical axis at (yaw, pitch), zero roll."""
    f = np.array([math.cos(yaw) * math.cos(pitch), math.sin(yaw) * math.cos(pitch), math.sin(pitch)])
    right = np.cross(f, np.array([0.0, 0.0, 1.0]))
    right /= np.linalg.norm(right)
    down = np.cross(f, right)
    return np.stack([right, down, f], axis=1)


def _rot_axis(axis, ang):
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + math.sin(ang) * K + (1 - math.cos(ang)) * (K @ K)


def _pixel_dirs(W, H, K):
    fx, fy, cx, cy = K
    u, v = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
    xc = (u.ravel() - cx) / fx
    yc = (v.ravel() - cy) / fy
    Dc = np.stack([xc, yc, np.ones_like(xc)], axis=1)
    rho = np.sqrt((xc * xc + yc * yc) + 1.0)
    return Dc, rho


def _render_frame(scene, W, H, K, R, C, sigma_c, outlier_pi, rng_noise, invalid_p, rng_invalid, patch=None):
    _, rho = _pixel_dirs(W, H, K)
    t = scene.render_depth(W, H, K, R, C)
    valid = np.isfinite(t)
    Z = np.where(valid, t * rho, 0.0)
    if patch is None:
        c0, c1, c2 = sigma_c
        sig = c0 + c1 * Z + c2 * Z * Z
        Z = Z + rng_noise.standard_normal(Z.shape) * sig  # noise along the range (§8(d))
    else:  # the per-patch model: bias-predicted mean, per-patch sigma
        pc = patch.pixel_coeffs(W, H)
        bias = pc[:, 0] + pc[:, 1] * Z + pc[:, 2] * Z * Z
        sig = np.maximum(pc[:, 3] + pc[:, 4] * Z + pc[:, 5] * Z * Z, patch.sigma_min)
        Z = Z + bias + rng_noise.standard_normal(Z.shape) * sig
    if outlier_pi > 0:
        out = rng_noise.random(Z.shape) < outlier_pi
        Z = np.where(out, rng_noise.uniform(OUTLIER_LO, OUTLIER_HI, Z.shape), Z)
    z = np.where(valid, Z / rho, 0.0)
    if invalid_p > 0:
        z = np.where(rng_invalid.random(z.shape) < invalid_p, 0.0, z)
    z = np.where(z > 0, z, 0.0)
    T = np.concatenate([R, C[:, None]], axis=1).reshape(-1)
    return Frame(depth=z.reshape(H, W).astype(np.float32), K=np.asarray(K, dtype=np.float64),
                 T_wc=T.astype(np.float64))


def _near_box(p, scene, clearance):
    for lo, hi in scene.boxes:
        if np.all(p > np.asarray(lo) - clearance) and np.all(p < np.asarray(hi) + clearance):
            return True
    for centre, half, yaw in scene.obbs:
        c, s = math.cos(yaw), math.sin(yaw)
        Rz = np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])
        q = Rz.T @ (p - np.asarray(centre))
        if np.all(np.abs(q) < np.asarray(half) + clearance):
            return True
    return False


def _random_walk(n, start, size, scene, rng, yaw0):
    """Smooth seeded random walk: exactly 0.05 m and 2 deg per step (configs[2..4])."""
    poses = []
    p = np.asarray(start, dtype=np.float64)
    R = _camera_rotation(yaw0)
    heading = rng.uniform(0, 2 * math.pi)
    omega = 0.0
    beta = 0.0
    yaw_sign = 1.0
    lo_x, hi_x = INSET + 0.6, size[0] - INSET - 0.6
    lo_y, hi_y = INSET + 0.6, size[1] - INSET - 0.6
    for k in range(n):
        poses.append((R.copy(), p.copy()))
        omega = 0.8 * omega + rng.normal(0.0, 0.2)
        heading += omega
        for _ in range(8):
            step = 0.05 * np.array([math.cos(heading), math.sin(heading), 0.0])
            q = p + step
            if q[0] < lo_x or q[0] > hi_x:
                heading = math.pi - heading
                continue
            if q[1] < lo_y or q[1] > hi_y:
                heading = -heading
                continue
            if _near_box(q, scene, 0.3):
                heading += math.pi
                continue
            break
        p = p + 0.05 * np.array([math.cos(heading), math.sin(heading), 0.0])
        # rotation: exactly 2 degrees about a camera-frame axis mixing yaw (cam y)
        # with a small pitch component (cam x); |pitch| kept <= 15 degrees.
        beta = float(np.clip(0.8 * beta + rng.normal(0.0, 0.3), -0.6, 0.6))
        if rng.random() < 0.1:
            yaw_sign = -yaw_sign
        axis = np.array([math.sin(beta), yaw_sign * math.cos(beta), 0.0])
        Rn = R @ _rot_axis(axis, math.radians(2.0))
        if abs(math.degrees(math.asin(np.clip(Rn[2, 2], -1, 1)))) > 15.0:
            axis[0] = -axis[0]
            Rn = R @ _rot_axis(axis, math.radians(2.0))
        # re-orthonormalise (keeps ||R^T R - I|| far below the ABI's 1e-6 check)
        u_, _, vt = np.linalg.svd(Rn)
        R = u_ @ vt
    return poses


def _add_boxes(scene, rng, n, size, side_lo=0.2, side_hi=1.0):
    lo, hx, hy = INSET, size[0] - INSET, size[1] - INSET
    for _ in range(n):
        s = rng.uniform(side_lo, side_hi, 3)
        cx = rng.uniform(lo + s[0] / 2, hx - s[0] / 2)
        cy = rng.uniform(lo + s[1] / 2, hy - s[1] / 2)
        blo = (cx - s[0] / 2, cy - s[1] / 2, INSET)
        bhi = (cx + s[0] / 2, cy + s[1] / 2, INSET + s[2])
        scene.boxes.append((blo, bhi))


def _add_slabs(scene, rng, n, size):
    """Thin 1.5 x 0.02 x 1.0 m panels with seeded yaw (glancing rays, configs[3])."""
    half = (0.75, 0.01, 0.5)
    reach = math.hypot(half[0], half[1])
    lo, hx, hy = INSET, size[0] - INSET, size[1] - INSET
    for _ in range(n):
        yaw = rng.uniform(0, math.pi)
        cx = rng.uniform(lo + reach, hx - reach)
        cy = rng.uniform(lo + reach, hy - reach)
        scene.obbs.append(((cx, cy, INSET + half[2]), half, yaw))


# --------------------------------------------------------------------------- configs

def _tiny_scene(rs):
    scene = _Scene()
    # back wall x = 1.45 over the full y-z face
    scene.rects.append((0, 1.45, (0.0, 0.0), (1.6, 1.6)))
    for _ in range(3):
        s = rs.uniform(0.2, 0.6, 3)
        x0 = rs.uniform(0.9, 1.45 - s[0])
        cy, cz = rs.uniform(0.45, 1.15, 2)
        scene.boxes.append(((x0, cy - s[1] / 2, cz - s[2] / 2), (x0 + s[0], cy + s[1] / 2, cz + s[2] / 2)))
    return scene


def tiny(seed: int = 0) -> Workload:
    """BASELINE.json configs[0]: 64x48 frame, 32^3 grid @0.05 m, camera on a voxel corner."""
    rs = np.random.default_rng(seed)
    scene = _tiny_scene(rs)
    K = (60.0, 60.0, 32.0, 24.0)
    R = np.array([[0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]])
    C = np.array([0.8, 0.8, 0.8])
    sigma_c = (0.0, 0.0, 0.0012)
    fr = _render_frame(scene, 64, 48, K, R, C, sigma_c, 0.0,
                       np.random.default_rng(seed + 2), 0.1, np.random.default_rng(seed + 3))
    lut = build_log_nu_lut(64, 128, 0.0, 2.0, -0.2, 0.2, sigma_c, 0.0)
    return Workload("tiny", (32, 32, 32), 0.05, (0.0, 0.0, 0.0), 0.5, lut, 0.0, 2.0, -0.2, 0.2,
                    0.1, 3.0, sigma_c, 10, [fr], seed)


def tiny_frames(seed: int = 0, n_frames: int = 4) -> Workload:
    """Test workload: the tiny scene seen from n_frames nearby poses (camera moved back along
    -x by up to 0.3 m and yawed by up to +-8 degrees), so that several keyframes observe the
    same voxels -- the small multi-keyframe case of the keyframe-average parity tests."""
    rs = np.random.default_rng(seed)
    scene = _tiny_scene(rs)
    K = (60.0, 60.0, 32.0, 24.0)
    R0 = np.array([[0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]])
    sigma_c = (0.0, 0.0, 0.0012)
    rn, ri = np.random.default_rng(seed + 2), np.random.default_rng(seed + 3)
    frames = []
    for i in range(n_frames):
        a = math.radians(8.0) * math.sin(1.7 * i)
        Rz = np.array([[math.cos(a), -math.sin(a), 0.0], [math.sin(a), math.cos(a), 0.0], [0.0, 0.0, 1.0]])
        C = np.array([0.8 - 0.3 * i / max(1, n_frames - 1), 0.8 + 0.05 * math.cos(i), 0.8 + 0.04 * math.sin(2 * i)])
        frames.append(_render_frame(scene, 64, 48, K, Rz @ R0, C, sigma_c, 0.0, rn, 0.1, ri))
    lut = build_log_nu_lut(64, 128, 0.0, 2.0, -0.2, 0.2, sigma_c, 0.0)
    return Workload(f"tiny_frames[{n_frames}]", (32, 32, 32), 0.05, (0.0, 0.0, 0.0), 0.1, lut, 0.0, 2.0, -0.2,
                    0.2, 0.1, 3.0, sigma_c, 10, frames, seed)


def _room_workload(name, size, res, n_frames, n_boxes, n_slabs, outlier_pi, lut_z_hi, lut_off,
                   n_iter, seed, start, fixed_camera=False):
    rs = np.random.default_rng(seed)
    scene = _Scene()
    _room(scene, size)
    _add_boxes(scene, rs, n_boxes, size)
    _add_slabs(scene, rs, n_slabs, size)
    rt = np.random.default_rng(seed + 1)
    yaw0 = rt.uniform(0, 2 * math.pi)
    if fixed_camera:
        poses = [(_camera_rotation(yaw0), np.asarray(start, dtype=np.float64))]
    else:
        poses = _random_walk(n_frames, start, size, scene, rt, yaw0)
    rn = np.random.default_rng(seed + 2)
    sigma_c = (0.0, 0.0, 0.0012)
    K = (525.0, 525.0, 319.5, 239.5)
    frames = [_render_frame(scene, 640, 480, K, R, C, sigma_c, outlier_pi, rn, 0.0, None)
              for (R, C) in poses]
    lut = build_log_nu_lut(256, 256, 0.0, lut_z_hi, -lut_off, lut_off, sigma_c, outlier_pi)
    dims = tuple(int(round(s / res)) for s in size)
    return Workload(name, dims, res, (0.0, 0.0, 0.0), 0.1, lut, 0.0, lut_z_hi, -lut_off, lut_off,
                    0.1, 3.0, sigma_c, n_iter, frames, seed)


def single_frame(seed: int = 0) -> Workload:
    """configs[1]: one 640x480 frame, 6x6x3 m room @0.05 m, 1% outliers, 8 iterations."""
    return _room_workload("frame1", (6.0, 6.0, 3.0), 0.05, 1, 20, 0, 0.01, 9.0, 0.5, 8, seed,
                          (3.0, 3.0, 1.5), fixed_camera=True)


def frames30(seed: int = 0, n_frames: int = 30) -> Workload:
    """configs[2]: 30 random-walk frames in the 6x6x3 m room @0.05 m, 10 iterations."""
    return _room_workload("frames30" if n_frames == 30 else f"frames30[:{n_frames}]",
                          (6.0, 6.0, 3.0), 0.05, n_frames, 20, 0, 0.01, 9.0, 0.5, 10, seed,
                          (3.0, 3.0, 1.5))


def frames100(seed: int = 0, n_frames: int = 100) -> Workload:
    """configs[3]: 100 frames, 8x8x3 m @0.02 m (400x400x150), boxes + thin slabs, 10 iterations."""
    return _room_workload("frames100" if n_frames == 100 else f"frames100[:{n_frames}]",
                          (8.0, 8.0, 3.0), 0.02, n_frames, 60, 20, 0.0, 12.0, 1.0, 10, seed,
                          (4.0, 4.0, 1.5))


def sweep300(seed: int = 0, n_frames: int = 300) -> Workload:
    """configs[4]: 300 frames, 10x10x3 m @0.02 m (500x500x150), 15 iterations."""
    return _room_workload("sweep300" if n_frames == 300 else f"sweep300[:{n_frames}]",
                          (10.0, 10.0, 3.0), 0.02, n_frames, 60, 20, 0.0, 15.0, 1.0, 15, seed,
                          (5.0, 5.0, 1.5))


CONFIG_NAMES = {"tiny": tiny, "frame1": single_frame, "frames30": frames30,
                "frames100": frames100, "sweep300": sweep300}


def make_workload(name: str, seed: int = 0, **kw) -> Workload:
    return CONFIG_NAMES[name](seed=seed, **kw)


def tiny_patch(seed: int = 0) -> Workload:
    """The tiny config with the learnt per-patch noise model (20x20-pixel patches: 4 x 3 over 64x48)."""
    w = tiny(seed)
    rs = np.random.default_rng(seed)
    scene = _tiny_scene(rs)
    pm = patch_noise_model(64, 48, seed, 20, w.sigma_c)
    fr = w.frames[0]
    R = fr.T_wc.reshape(3, 4)[:, :3]
    C = fr.T_wc.reshape(3, 4)[:, 3]
    w.frames = [_render_frame(scene, 64, 48, tuple(fr.K), R, C, w.sigma_c, 0.0, np.random.default_rng(seed + 2), 0.1,
                              np.random.default_rng(seed + 3), patch=pm)]
    w.patch = pm
    w.name = "tiny_patch"
    return w


def frame1_patch(seed: int = 0) -> Workload:
    """configs[1]'s room and camera with the per-patch noise model (32 x 24 patches)."""
    rs = np.random.default_rng(seed)
    scene = _Scene()
    size = (6.0, 6.0, 3.0)
    _room(scene, size)
    _add_boxes(scene, rs, 20, size)
    rt = np.random.default_rng(seed + 1)
    yaw0 = rt.uniform(0, 2 * math.pi)
    R, C = _camera_rotation(yaw0), np.array([3.0, 3.0, 1.5])
    sigma_c = (0.0, 0.0, 0.0012)
    pm = patch_noise_model(640, 480, seed, 20, sigma_c)
    fr = _render_frame(scene, 640, 480, (525.0, 525.0, 319.5, 239.5), R, C, sigma_c, 0.0,
                       np.random.default_rng(seed + 2), 0.0, None, patch=pm)
    lut = build_log_nu_lut(256, 256, 0.0, 9.0, -0.5, 0.5, sigma_c, 0.0)
    return Workload("frame1_patch", (120, 120, 60), 0.05, (0.0, 0.0, 0.0), 0.1, lut, 0.0, 9.0, -0.5, 0.5,
                    0.1, 3.0, sigma_c, 8, [fr], seed, pm)


CONFIG_NAMES.update({"tiny_patch": tiny_patch, "frame1_patch": frame1_patch})
