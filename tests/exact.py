"""Exact, independent reference computations used as pins for the oracle.

Nothing here calls oracle/ or the CUDA path.  Each routine is the *definition*
of the quantity, evaluated by brute force in exact or fp64 arithmetic:

* dda_bruteforce: every grid cell whose intersection with the fixed-point segment
  has positive length, by slab intersection with exact rationals (Python ints),
  sorted by entry parameter (SURVEY §8(c) B2 pin; reading R13).
* enum_ray_messages: Eq.12 evaluated over all 2^N occupancy
  configurations with the case table of Eq.5; the all-empty
  configuration has potential 0 (Eq.3).
* enum_joint_marginals: exact marginals of the MRF joint of Eq.1 with
  phi of Eq.2 and psi of Eq.3, by enumeration over all voxel configurations.
"""

from __future__ import annotations

import itertools
import math
from fractions import Fraction

import numpy as np

ONE = 65536


def _floor_div(a, b):
    return a // b  # Python floors


def dda_bruteforce(dims, G0, G1):
    """Return [(vid, t_in: Fraction, t_out: Fraction)] sorted by t_in."""
    dG = [G1[k] - G0[k] for k in range(3)]
    lo_c, hi_c = [], []
    for k in range(3):
        a, b = sorted((G0[k], G1[k]))
        lo_c.append(max(0, _floor_div(a, ONE) - 1))
        hi_c.append(min(dims[k] - 1, _floor_div(b, ONE) + 1))
    out = []
    for cz in range(lo_c[2], hi_c[2] + 1):
        for cy in range(lo_c[1], hi_c[1] + 1):
            for cx in range(lo_c[0], hi_c[0] + 1):
                c = (cx, cy, cz)
                t_lo, t_hi = Fraction(0), Fraction(1)
                ok = True
                for k in range(3):
                    if dG[k] == 0:
                        if _floor_div(G0[k], ONE) != c[k]:  # half-open cell [c, c+1)
                            ok = False
                            break
                        continue
                    ta = Fraction(c[k] * ONE - G0[k], dG[k])
                    tb = Fraction((c[k] + 1) * ONE - G0[k], dG[k])
                    if ta > tb:
                        ta, tb = tb, ta
                    t_lo = max(t_lo, ta)
                    t_hi = min(t_hi, tb)
                if ok and t_hi > t_lo:
                    out.append((cx + dims[0] * (cy + dims[1] * cz), t_lo, t_hi))
    out.sort(key=lambda x: x[1])
    return out


def sigmoid(x):
    return 1.0 / (1.0 + math.exp(-x))


def enum_ray_messages(c, nu):
    """Eq.12 by enumeration: returns (pos[i], neg[i]) = mu_{psi->o_i}(1), mu_{psi->o_i}(0)
    with incoming mu_j(1) = sigmoid(c_j), mu_j(0) = 1 - mu_j(1) and uniform mu(d)."""
    N = len(c)
    m1 = [sigmoid(x) for x in c]
    m0 = [sigmoid(-x) for x in c]
    pos = [0.0] * N
    neg = [0.0] * N
    for conf in itertools.product((0, 1), repeat=N):
        if 1 not in conf:
            continue  # psi = 0 for the all-empty configuration
        first = conf.index(1)
        psi = nu[first]
        for i in range(N):
            w = psi
            for j in range(N):
                if j != i:
                    w *= m1[j] if conf[j] else m0[j]
            if conf[i]:
                pos[i] += w
            else:
                neg[i] += w
    return np.array(pos), np.array(neg)


def enum_joint_marginals(n_vox, rays, gamma):
    """rays: list of (voxel list in order, nu list).  Exact p(o_v = 1) of Eq.1."""
    Zs = 0.0
    p1 = np.zeros(n_vox)
    for conf in itertools.product((0, 1), repeat=n_vox):
        w = 1.0
        for v in range(n_vox):
            w *= gamma if conf[v] else (1.0 - gamma)
        for vox, nu in rays:
            hit = None
            for i, v in enumerate(vox):
                if conf[v]:
                    hit = i
                    break
            if hit is None:
                w = 0.0
                break
            w *= nu[hit]
        if w == 0.0:
            continue
        Zs += w
        for v in range(n_vox):
            if conf[v]:
                p1[v] += w
    return p1 / Zs


def single_ray_marginals(nu, gamma):
    """Closed form for one ray (a tree): w_j = nu_j gamma (1-gamma)^(j-1),
    p_i = (gamma sum_{j<i} w_j + w_i) / sum_j w_j  (derived from Eq.3/Eq.5 + Eq.8)."""
    w = [nu[j] * gamma * (1.0 - gamma) ** j for j in range(len(nu))]
    Zs = sum(w)
    return np.array([(gamma * sum(w[:i]) + w[i]) / Zs for i in range(len(nu))])
