"""Device math of the force kernel (tsf_math.cuh) through tsf_math_probe.

* exp / log with constant-bank polynomials against libdevice: <= 2 / 3 ulp,
  overflow to inf and underflow to 0 like exp();
* the bond order's series path (beta zeta small: the Tersoff 1989 SiC table)
  and log-space path (Si(B): u ~ 27 in the crystal) against the reference's pow form
  (proj/include/tmd/potential.hpp:107-120): 1e-14 relative in double, 2e-6
  in float; the series path is the one taken for physical zeta.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def probe(tb, params, fn, x):
    from paper_1607_02904_b200 import _lib as L
    x = np.ascontiguousarray(x, np.float64)
    out = np.zeros(2 * len(x))
    rc = L.lib().tsf_math_probe(params._h, fn, len(x), x.ctypes.data_as(C.c_void_p),
                                out.ctypes.data_as(C.c_void_p))
    assert rc == 0
    return out[0::2], out[1::2]


def ulps(a, b):
    return np.abs(a - b) / np.spacing(np.abs(b))


def test_exp_against_libdevice(tb, si):
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.uniform(-1, 1, 20000), rng.uniform(-80, 80, 20000),
                        rng.uniform(-700, 700, 20000)])
    a, _ = probe(tb, si, 0, x)
    r, _ = probe(tb, si, 2, x)
    assert ulps(a, r).max() <= 2.0
    big, _ = probe(tb, si, 0, [709.7, 709.8, 800.0, 2000.0, -745.2, -800.0, -2000.0, 0.0])
    assert np.isfinite(big[0]) and np.isinf(big[1:4]).all()
    assert (big[4:7] == 0).all() and big[7] == 1.0


def test_log_against_libdevice(tb, si):
    rng = np.random.default_rng(4)
    x = np.exp(rng.uniform(-690, 690, 40000))
    x = np.concatenate([x, 1 + rng.uniform(-1e-3, 1e-3, 2000), [1.0, 2.0, 0.5, np.sqrt(2.0)]])
    a, _ = probe(tb, si, 1, x)
    r, _ = probe(tb, si, 3, x)
    err = np.abs(a - r) / np.maximum(np.spacing(np.abs(r)), np.spacing(1.0) * 1e-3)
    assert err.max() <= 3.0 or np.abs(a - r).max() <= 4e-16


@pytest.mark.parametrize("table", ["si", "sic"])
def test_bond_order_paths(tb, si, sic_text, table):
    params = si if table == "si" else tb.parse_params(sic_text)
    zeta = np.concatenate([np.geomspace(1e-8, 1e6, 4000), [0.0, -1.0, 3.4, 20.0]])
    b, db = probe(tb, params, 4, zeta)
    rb, rdb = probe(tb, params, 6, zeta)
    assert np.abs(b - rb).max() <= 1e-14
    scale = np.maximum(np.abs(rdb), 1e-300)
    assert (np.abs(db - rdb) / scale).max() <= 1e-12
    fb, fdb = probe(tb, params, 5, zeta)
    assert np.abs(fb - rb).max() <= 2e-6
    ok = np.abs(rdb) > 1e-30
    assert (np.abs(fdb[ok] - rdb[ok]) / np.abs(rdb[ok])).max() <= 1e-4
    # the series path serves small-beta tables (Tersoff 1989 SiC: beta ~ 1e-6,
    # u = (beta zeta)^eta < 2^-12 for every physical zeta); Si(B) (beta 0.33675,
    # eta 22.956: u ~ 27 in the crystal) takes the log-space form
    taken, lnu = probe(tb, params, 7, np.array([0.5, 1.0, 3.4, 10.0, 20.0]))
    if table == "sic":
        assert (taken == 1.0).all(), lnu
    else:   # only for tiny zeta (u < 2^-12)
        assert list(taken) == [1.0, 1.0, 0.0, 0.0, 0.0] and lnu[2] > 0, lnu


def test_ramp_sincospi_against_libdevice(tb, si):
    """The cutoff ramp's branch-free sin(pi x), cos(pi x) (|x| <= 1/2, the
    whole ramp R - D < r < R + D; potential.hpp:58-69) against libdevice's
    sincospi: within 2.5e-16 absolute, exact at the ramp's centre."""
    rng = np.random.default_rng(5)
    x = np.concatenate([rng.uniform(-0.5, 0.5, 40000), [-0.5, -0.25, 0.0, 0.25, 0.5]])
    s, c = probe(tb, si, 8, x)
    rs, rc = probe(tb, si, 9, x)
    assert np.abs(s - rs).max() <= 2.5e-16 and np.abs(c - rc).max() <= 2.5e-16
    s0, c0 = probe(tb, si, 8, [0.0])
    assert s0[0] == 0.0 and c0[0] == 1.0
