"""Forward sensor model tabulated as log nu(Z, delta) (input bytes, not method arithmetic).

PAPER.md Eq.4: nu_r(d_i) = N(Z_r; d_i, sigma(d_i)), with a depth
dependent sigma.  Main-text reading (reading R1 /
SURVEY §8(c) A1): the measurement Z is evaluated under a Gaussian centred at the
voxel depth d (identity bias here) with sigma(d) = c0 + c1 d + c2 d^2, floored
at 1e-4 m.  Optional outlier mixture (1-pi) N + pi U(Z; 0.3, 5) for the
"Gaussian-plus-outlier" configs (BASELINE.json configs[1], configs[2]).

Axes: row i <-> measured range Z_i = z_lo + (i+0.5)(z_hi-z_lo)/n_z,
column j <-> offset delta_j = off_lo + (j+0.5)(off_hi-off_lo)/n_off, the voxel
depth being d = Z + delta.  Each row is floored at (row max - floor_nats)
 so that the table stays finite.
"""

from __future__ import annotations

import math

import numpy as np

SIGMA_MIN = 1e-4
OUTLIER_LO = 0.3
OUTLIER_HI = 5.0


def build_log_nu_lut(n_z: int, n_off: int, z_lo: float, z_hi: float,
                     off_lo: float, off_hi: float, sigma_c=(0.0, 0.0, 0.0012),
                     outlier_pi: float = 0.0, floor_nats: float = 100.0) -> np.ndarray:
    """Return float32 [n_z, n_off] table of log nu at the bin centres."""
    zc = z_lo + (np.arange(n_z, dtype=np.float64) + 0.5) * (z_hi - z_lo) / n_z
    dc = off_lo + (np.arange(n_off, dtype=np.float64) + 0.5) * (off_hi - off_lo) / n_off
    Z = zc[:, None]
    delta = dc[None, :]
    d = Z + delta
    c0, c1, c2 = sigma_c
    sigma = np.maximum(c0 + c1 * d + c2 * d * d, SIGMA_MIN)
    log_g = -0.5 * (delta / sigma) ** 2 - np.log(sigma * math.sqrt(2.0 * math.pi))
    if outlier_pi > 0.0:
        in_range = (Z >= OUTLIER_LO) & (Z <= OUTLIER_HI)
        log_u = np.where(in_range, math.log(outlier_pi / (OUTLIER_HI - OUTLIER_LO)), -np.inf)
        log_nu = np.logaddexp(math.log1p(-outlier_pi) + log_g, np.broadcast_to(log_u, log_g.shape))
    else:
        log_nu = log_g
    row_max = log_nu.max(axis=1, keepdims=True)
    log_nu = np.maximum(log_nu, row_max - floor_nats)
    out = log_nu.astype(np.float32)
    assert np.all(np.isfinite(out))
    return out
