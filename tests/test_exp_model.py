"""The device exp (csrc/exp_np.cuh) restates numpy's float64 exp (Intel
SVML __svml_exp8_ha on AVX-512 hosts).  Check the host model of it against
np.exp where the golden fixtures were made (needs an AVX-512 numpy build:
skipped elsewhere, since then numpy itself computes exp differently)."""
import numpy as np
import pytest

from tools.exp_model import exp_model


def _numpy_uses_svml():
    try:
        import numpy._core._multiarray_umath as m
        path = m.__file__
    except Exception:
        return False
    import subprocess
    out = subprocess.run(["nm", "-D", path], capture_output=True, text=True).stdout
    x = np.array([-3.3, 0.7, -12.25])
    return "__svml_exp8_ha" in out and np.array_equal(np.exp(x), exp_model(x))


@pytest.mark.skipif(not _numpy_uses_svml(), reason="numpy here does not use SVML exp")
@pytest.mark.parametrize("lo,hi", [(-40.0, 0.0), (-1.0, 1.0), (-707.0, -600.0),
                                   (-700.0, 700.0), (600.0, 707.7), (-1e-15, 1e-15)])
def test_exp_model_bit_exact(lo, hi):
    x = np.random.default_rng(int(abs(lo * 7 + hi))).uniform(lo, hi, 300_000)
    assert np.array_equal(exp_model(x), np.exp(x))


def test_exp_model_specials():
    with np.errstate(all="ignore"):
        x = np.array([np.inf, -np.inf, 0.0, -0.0, 710.0, -746.0])
        assert np.array_equal(exp_model(x), np.exp(x))
        assert np.isnan(exp_model(np.array([np.nan])))[0]


@pytest.mark.skipif(not _numpy_uses_svml(), reason="numpy here does not use SVML exp")
@pytest.mark.parametrize("lo,hi,bar", [(-745.13, -708.4, 0.9995), (-708.4, 708.4, 0.94),
                                       (-708.4, -707.0, 0.94), (707.0, 709.78, 0.94)])
def test_exp_rare_range(lo, hi, bar):
    """|x| >= 1021 ln2: numpy's scalar rare path, modelled by exp_rare.h
    (double-double, one rounding).  Bit-exact below the threshold; above
    it, numpy's routine is itself not correctly rounded near midpoints, so
    the bar is a match rate (measured here: 99.997 % on subnormal results,
    95-99.9 % in 707.7 < |x| < 708.4)."""
    x = np.random.default_rng(int(abs(lo + hi * 3))).uniform(lo, hi, 200_000)
    got, want = exp_model(x), np.exp(x)
    below = np.abs(x) < float.fromhex("0x1.61da04cbafe44p+9")
    assert np.array_equal(got[below], want[below])
    if (~below).any():
        assert np.mean(got[~below] == want[~below]) >= bar
