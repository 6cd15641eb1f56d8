"""CPU-side checks of the boundary: libmrf.so loads, exports every symbol include/mrf.h
declares, and rejects bad arguments before touching the device (no compute calls)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2006_03512_b200 as pkg
from paper_2006_03512_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "mrf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mrf_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = pkg.load()
    syms = _header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(_lib.EXPORTS) == syms


def test_header_documents_paper_passages():
    src = open(os.path.join(ROOT, "include", "mrf.h")).read()
    for cite in ("P:200", "P:205", "Eq.13", "Eq.14", "Eq.8", "Eq.6"):
        assert cite in src


def _noise(n_z=4, n_off=4):
    return dict(log_nu=np.zeros((n_z, n_off), np.float32), z_lo=0.0, z_hi=2.0, off_lo=-0.2, off_hi=0.2)


@pytest.mark.parametrize("kw,msg", [
    (dict(dims=(0, 4, 4)), "dims"),
    (dict(dims=(9000, 4, 4)), "dims"),
    (dict(dims=(2048, 2048, 1024)), "2^31"),
    (dict(res=0.0), "resolution"),
    (dict(res=float("nan")), "resolution"),
    (dict(prior=1.0), "prior"),
    (dict(prior=0.0), "prior"),
    (dict(noise=dict(log_nu=np.zeros((1, 4), np.float32))), "2x2"),
    (dict(noise=dict(z_hi=0.0)), "z_hi"),
    (dict(noise=dict(off_lo=-2.0)), "offset"),
    (dict(noise=dict(log_nu=np.full((4, 4), np.inf, np.float32))), "non-finite"),
    (dict(noise=dict(margin_min=1.0)), "margin bound"),
    (dict(noise=dict(sigma_c=(0.0, 0.0, 50.0))), "margin bound"),
])
def test_create_rejects_bad_arguments(kw, msg):
    args = dict(dims=(4, 4, 4), res=0.05, origin=(0, 0, 0), prior=0.5)
    noise = _noise()
    noise.update(kw.pop("noise", {}))
    args.update(kw)
    with pytest.raises(pkg.MrfError) as ei:
        pkg.MRFMap(args["dims"], args["res"], args["origin"], args["prior"], **noise)
    assert ei.value.status == _lib.MRF_ERR_INVALID_ARG
    assert msg in str(ei.value)


def test_null_ctx_is_rejected():
    L = pkg.load()
    assert L.mrf_bp_iterate(None, 1) == _lib.MRF_ERR_INVALID_ARG
    assert L.mrf_destroy(None) == _lib.MRF_OK
    assert L.mrf_launch_count(None) == 0


def test_product_path_does_not_import_oracle():
    """The product package must never reach the oracle (no CPU fallback)."""
    pkg_dir = os.path.join(ROOT, "paper_2006_03512_b200")
    for dp, _, files in os.walk(pkg_dir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dp, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "mrf_oracle" not in src and "orc_" not in src, f
