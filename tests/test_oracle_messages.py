"""Pins for oracle B5 (single-ray factor->occupancy messages, Eq.13/14) and B3 LUT lookup.

The linear-time closed forms (division-free o=0 form P:524) must equal
the O(2^N) marginalisation of Eq.12 with the Eq.5 case table
 -- the derivation the paper gives in its supplement.
"""

import json
import math
import os

import numpy as np
import pytest

import oracle
from tests.exact import enum_ray_messages

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_messages_match_enumeration_random():
    rng = np.random.default_rng(0)
    worst = 0.0
    for _ in range(3000):
        N = int(rng.integers(1, 11))
        c = rng.uniform(-8, 8, N)
        lnu = rng.uniform(-6, 0, N)
        lpos, lneg = oracle.ray_messages(c, lnu)
        pos, neg = enum_ray_messages(c, np.exp(lnu))
        assert np.allclose(np.exp(lpos), pos, rtol=1e-12, atol=0)
        nz = neg > 0
        assert np.allclose(np.exp(lneg[nz]), neg[nz], rtol=1e-12, atol=0)
        assert np.all(np.isneginf(lneg[~nz]))  # only N = 1 has an empty o=0 sum
        worst = max(worst, float(np.max(np.abs(np.exp(lpos) / pos - 1))))
    assert worst < 1e-12


@pytest.mark.parametrize("N", [12, 14])
def test_messages_match_enumeration_long(N):
    rng = np.random.default_rng(N)
    for _ in range(5):
        c = rng.uniform(-20, 20, N)
        lnu = rng.uniform(-30, 5, N)
        lpos, lneg = oracle.ray_messages(c, lnu)
        pos, neg = enum_ray_messages(c, np.exp(lnu))
        assert np.allclose(lpos - lneg, np.log(pos) - np.log(neg), rtol=1e-10, atol=1e-10)


def test_spec_hand_example():
    g = json.load(open(os.path.join(GOLDEN, "spec_hand_examples.json")))
    c = [math.log(m / (1 - m)) for m in g["mu1"]]
    lpos, lneg = oracle.ray_messages(c, np.log(g["nu"]))
    assert np.allclose(np.exp(lpos), g["unnormalised_pos"], rtol=1e-12)
    assert np.allclose(np.exp(lneg), g["unnormalised_neg"], rtol=1e-12)
    pairs = np.stack([np.exp(lneg), np.exp(lpos)], 1)
    pairs /= pairs.sum(1, keepdims=True)
    assert np.allclose(pairs, g["normalised_pairs"], rtol=0, atol=1e-12)


def test_first_voxel_positive_message_is_nu():
    """i = 1 -> mu(o_1 = 1) = nu_1 (first sum empty, empty product)."""
    c = np.array([0.3, -2.0, 1.0])
    lnu = np.array([-1.5, 0.2, -0.7])
    lpos, _ = oracle.ray_messages(c, lnu)
    assert abs(lpos[0] - lnu[0]) < 1e-15


def test_visibility_saturation():
    """S:311 / P:163: behind a voxel with mu(o=0) -> 0 the messages become uniform."""
    c = np.array([-1.0, 900.0, 0.5, -3.0, 2.0])
    lnu = np.array([-2.0, -1.0, 1.0, 0.0, -4.0])
    lpos, lneg = oracle.ray_messages(c, lnu)
    assert np.all(np.abs((lpos - lneg)[2:]) < 1e-12)


def test_nu_scale_invariance():
    """adding a constant to log nu of a ray leaves the log-odds messages unchanged."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        N = int(rng.integers(2, 30))
        c = rng.uniform(-10, 10, N)
        lnu = rng.uniform(-50, 5, N)
        a = oracle.ray_messages(c, lnu)
        b = oracle.ray_messages(c, lnu + rng.uniform(-40, 40))
        assert np.allclose(a[0] - a[1], b[0] - b[1], rtol=1e-9, atol=1e-9)


def test_extreme_inputs_stay_finite():
    """Reading R9: log domain throughout; nu spanning e^{+-100}, cavities of +-1e4."""
    rng = np.random.default_rng(9)
    for _ in range(100):
        N = int(rng.integers(2, 200))
        c = rng.uniform(-1e4, 1e4, N)
        lnu = rng.uniform(-250, 10, N)
        lpos, lneg = oracle.ray_messages(c, lnu)
        assert np.all(np.isfinite(lpos)) and np.all(np.isfinite(lneg))


def _lut_params(lut, z_lo=0.0, z_hi=2.0, off_lo=-1.0, off_hi=1.0):
    return oracle.Params((4, 4, 4), 0.05, (0, 0, 0), 0.5, lut, z_lo, z_hi, off_lo, off_hi, 0.1, 3.0, (0, 0, 0.0012))


def test_log_nu_bilinear_pins():
    """B3: value at a bin centre is the table entry; clamped outside; bilinear in between."""
    rng = np.random.default_rng(2)
    lut = rng.normal(size=(8, 64)).astype(np.float32)
    p = _lut_params(lut)
    for i in range(8):
        for j in range(64):
            Z = 0.0 + (i + 0.5) * 2.0 / 8
            off_q = int((j - 31.5) * 1024)  # bin centre: -1 + (j+0.5)/32 m, exactly
            assert oracle.log_nu(p, Z, off_q) == float(lut[i, j])
    # clamp below / above both axes
    assert oracle.log_nu(p, -5.0, -32767) == float(lut[0, 0])
    assert oracle.log_nu(p, 50.0, 32767) == float(lut[7, 63])
    # halfway between two centres along each axis
    Zm = (1 + 0.5 + 0.5) * 2.0 / 8
    assert abs(oracle.log_nu(p, Zm, int((5 - 31.5) * 1024)) - 0.5 * (lut[1, 5] + lut[2, 5])) < 1e-12
    assert abs(oracle.log_nu(p, (3 + 0.5) * 0.25, int((5 - 31.0) * 1024)) - 0.5 * (lut[3, 5] + lut[3, 6])) < 1e-12
