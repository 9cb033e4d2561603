"""The reference's error contract on the GPU path (error.hpp:9-21):

* NumericError where the double reference throws it (potential_ref.cpp:109-112,
  kernels.hpp:160-167): a close contact whose (beta zeta)^eta overflows
   and a NaN coordinate — in every precision and both
  scatter modes, through the Python surface and the C-ABI return code
  TSF_ERR_NUMERIC (3);
* the context stays usable after the error.
"""
import ctypes as C

import numpy as np
import pytest

import systems

pytestmark = pytest.mark.gpu


def _ctx(tb, case):
    params = tb.parse_params(case.params_text)
    ctx = tb.Context(params, 0)
    ctx.set_system(case.xyz, case.species, case.box, case.periodic)
    ctx.build_neighbor_list(params.r_cut_max, case.skin)
    return ctx


@pytest.mark.parametrize("cells,jitter,seed", [(2, 0.7, 1), (2, 0.8, 3)])
def test_close_contact_numeric_error(tb, oracle, cells, jitter, seed):
    from oracle.oracle import OracleNumericError, parse_param_text
    case = systems.perturbed(tb, cells, jitter, seed, skin=0.5)
    op = parse_param_text(case.params_text)
    off, nb = oracle.build_neighbor_list(case.xyz, case.box, case.periodic, op.r_cut_max,
                                         case.skin)
    with pytest.raises(OracleNumericError):
        oracle.compute_ref(op, case.xyz, case.species, case.box, case.periodic, off, nb)
    ctx = _ctx(tb, case)
    for prec in ("double", "mixed", "single"):
        for det in (False, True):
            with pytest.raises(tb.NumericError):
                ctx.compute(prec, deterministic=det)
    # the C-ABI code, and a clean system afterwards
    from paper_1607_02904_b200 import _lib as L
    e = C.c_double()
    assert L.lib().tsf_compute_f64(ctx._h, 0, C.byref(e), None, None) == L.TSF_ERR_NUMERIC
    good = systems.perturbed(tb, cells, 0.1, seed, skin=0.5)
    ctx.set_system(good.xyz, good.species, good.box, good.periodic)
    ctx.build_neighbor_list(tb.builtin_silicon().r_cut_max, 0.5)
    e1, f1, _ = ctx.compute("double")
    assert np.isfinite(e1) and np.isfinite(f1).all()
    ctx.close()


def test_nan_coordinate_numeric_error(tb, oracle):
    from oracle.oracle import OracleNumericError, parse_param_text
    case = systems.perturbed(tb, 3, 0.1, 5, skin=0.5)
    op = parse_param_text(case.params_text)
    off, nb = oracle.build_neighbor_list(case.xyz, case.box, case.periodic, op.r_cut_max,
                                         case.skin)
    bad = case.xyz.copy()
    bad[7, 1] = np.nan
    with pytest.raises(OracleNumericError):
        oracle.compute_ref(op, bad, case.species, case.box, case.periodic, off, nb)
    ctx = _ctx(tb, case)
    for prec in ("double", "mixed", "single"):
        for det in (False, True):
            ctx.set_positions(bad)
            with pytest.raises(tb.NumericError):
                ctx.compute(prec, deterministic=det)
    ctx.set_positions(case.xyz)
    e, f, _ = ctx.compute("double")
    ref = oracle.compute_ref(op, case.xyz, case.species, case.box, case.periodic, off, nb)
    assert abs(e - ref["energy"]) <= 1e-12 * abs(ref["energy"])
    ctx.close()
