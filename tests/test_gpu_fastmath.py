"""The device exp / reciprocal of the d(v) rows (hyg_fastmath.cuh) against
numpy (correctly rounded to ~0.5 ulp): within 2 ulp on the d(v) argument
range and beyond, flush-to-zero below -708, NaN propagation."""
import ctypes as C

import numpy as np
import pytest

from paper_1703_10119_b200 import api

pytestmark = pytest.mark.gpu


def _run(x):
    lib = api.load_library()
    x = np.ascontiguousarray(x, dtype=np.float64)
    e, r = np.empty_like(x), np.empty_like(x)
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    assert lib.hyg_selftest_fastmath(0, x.size, p(x), p(e), p(r)) == 0
    return e, r


def _ulps(a, b):
    return np.abs(a - b) / np.spacing(np.abs(b))


def test_fexp_frcp_accuracy():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.uniform(-10.0, 0.0, 200_000),       # d(v): -p2 (v - p3)^2
                        rng.uniform(-700.0, 700.0, 100_000), np.linspace(-1.0, 1.0, 10_001)])
    e, r = _run(x)
    assert _ulps(e, np.exp(x)).max() <= 2.0
    nz = x[np.abs(x) > 1e-300]
    _, rr = _run(nz)
    assert _ulps(rr, 1.0 / nz).max() <= 2.0
    e2, _ = _run(np.array([-800.0, -708.5, np.nan, 710.0, 0.0]))
    assert e2[0] == 0.0 and e2[1] == 0.0 and np.isnan(e2[2]) and np.isinf(e2[3]) and e2[4] == 1.0


def test_dv_half_node_exp_and_two_fma_reciprocal():
    """fexp_addend (256-entry table, degree 4, no clamp; -700 <= x <= 0): within
    2 ulp + |x| 3.3e-17 relative of exp (the reduction uses ln2/256 as one rounded
    constant, whose relative error is 3.3e-17: 3 ulp at the edge of the d(v) range
    |x| <= 6.4, and an absolute error of the Gaussian below 1.3e-17 everywhere);
    frcp2 below 1.1e-12 relative (measured 9.7e-13 = the square of rcp.approx's 2^-20) and never above the true reciprocal in magnitude."""
    lib = api.load_library()
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.uniform(0.0, 10.0, 200_000), rng.uniform(0.0, 180.0, 100_000),
                        rng.uniform(180.0, 700.0, 50_000), np.linspace(0.0, 1.0, 10_001)])
    e, r = np.empty_like(x), np.empty_like(x)
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    d = np.ascontiguousarray(rng.uniform(1.0, 200.0, x.size) * rng.choice([-1.0, 1.0], x.size))
    assert lib.hyg_selftest_dvmath(0, x.size, p(x), p(e), p(r)) == 0
    ref = np.exp(-x)
    u = _ulps(e, ref)
    assert (u <= 2.0 + x * 3.4e-17 / 1.1e-16).all(), u.max()
    assert u[x <= 6.4].max() <= 3.0 and np.abs(e - ref).max() <= 1.3e-17 + 2.3e-16, (u[x <= 6.4].max(), np.abs(e - ref).max())
    assert lib.hyg_selftest_dvmath(0, d.size, p(d), p(e), p(r)) == 0
    rel = (r - 1.0 / d) * d
    assert np.abs(rel).max() <= 1.1e-12 and rel.max() <= 2.0 ** -52, (np.abs(rel).max(), rel.max())


def test_flog_accuracy():
    """flog_pos (material correlations): within 2 ulp of the result, or 2 ulp
    of ln 2 where ln x cancels near 1 (absolute 2.5e-16), on the box's ranges
    (phi in [0.01, 0.99], capillary potentials, 1 + x^a) and far beyond."""
    lib = api.load_library()
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.uniform(0.01, 0.99, 200_000), 10.0 ** rng.uniform(-300, 300, 100_000),
                        1.0 + 10.0 ** rng.uniform(-16, 2, 50_000), np.array([1.0, 2.0, 0.5, 1e-300, 1e300])])
    out = np.empty_like(x)
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    assert lib.hyg_selftest_fastlog(0, x.size, p(x), p(out)) == 0
    ref = np.log(x)
    err = np.abs(out - ref)
    assert np.all(err <= np.maximum(2.0 * np.spacing(np.abs(ref)), 2.0 * np.spacing(np.log(2.0))))
    assert out[-5] == 0.0


def _cr(vals, fn):
    """Correctly rounded reference values (mpmath, 60 digits)."""
    import mpmath as mp
    mp.mp.dps = 60
    return np.array([float(fn(mp.mpf(float(v)))) for v in vals])


def test_crmath_correctly_rounded():
    """The accurate exp/log/log10/pow of the material parity path
    (hyg_crmath.cuh) return the correctly rounded double on samples spanning
    the material correlations' arguments (and beyond)."""
    import mpmath as mp
    rng = np.random.default_rng(7)
    x = np.concatenate([rng.uniform(1e-6, 3.0, 3000), np.exp(rng.uniform(-30, 30, 3000)),
                        1.0 + rng.uniform(-1e-3, 1e-3, 1000), [1.0, 2.0, 0.5, 10.0, 1e-300 * 1e10]])
    y = np.concatenate([rng.choice([1.65, -0.39, 6.0, -0.83, 0.65, 5.0, -1.39, -1.83], x.size - 10),
                        rng.uniform(-3, 3, 10)])
    ex = rng.uniform(-700, 700, x.size)
    lib = api.load_library()
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    out = np.empty(4 * x.size)
    assert lib.hyg_selftest_crmath(0, x.size, p(ex), p(y), p(out)) == 0
    e = out[:x.size]
    assert np.array_equal(e, _cr(ex, mp.exp)), np.flatnonzero(e != _cr(ex, mp.exp))[:5]
    assert lib.hyg_selftest_crmath(0, x.size, p(np.ascontiguousarray(x)), p(y), p(out)) == 0
    lg, l10, pw = out[x.size:2 * x.size], out[2 * x.size:3 * x.size], out[3 * x.size:]
    assert np.array_equal(lg, _cr(x, mp.log))
    assert np.array_equal(l10, _cr(x, mp.log10))
    ref = np.array([float(mp.power(mp.mpf(float(a)), mp.mpf(float(b)))) for a, b in zip(x, y)])
    finite = np.isfinite(ref) & (ref > 1e-300)
    assert np.array_equal(pw[finite], ref[finite])
