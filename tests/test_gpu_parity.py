"""GPU parity: libtersoff_b200.so against the CPU oracle on identical inputs.

Bars (BASELINE.json north star):
  neighbor lists and per-atom counts  bit-exact
  double   energy rel <= 1e-12, forces abs <= 1e-10 eV/A
  mixed / single  energy rel <= 1e-6, forces <= 1e-4 * max(1, max|F_ref|)
Large-N energy is gated against the long-double oracle sum.
"""
import numpy as np
import pytest

import systems

pytestmark = pytest.mark.gpu

E_TOL_D, F_TOL_D = 1e-12, 1e-10
E_TOL_M, F_TOL_M = 1e-6, 1e-4


def _ctx(tb, case):
    params = tb.parse_params(case.params_text)
    ctx = tb.Context(params, 0)
    ctx.set_system(case.xyz, case.species, case.box, case.periodic)
    ctx.build_neighbor_list(params.r_cut_max, case.skin)
    return params, ctx


def _oracle(oracle, case, params):
    from oracle.oracle import parse_param_text
    op = parse_param_text(case.params_text)
    off, nb = oracle.build_neighbor_list(case.xyz, case.box, case.periodic, op.r_cut_max,
                                         case.skin)
    ref = oracle.compute_ref(op, case.xyz, case.species, case.box, case.periodic, off, nb)
    return op, off, nb, ref


def _cases(tb, sic_text):
    return [
        systems.diamond(tb, 4),
        systems.perturbed(tb, 4, 0.12, 32, skin=0.5),
        systems.perturbed(tb, 2, 0.12, 722, skin=0.5),
        systems.perturbed(tb, 2, 0.35, 41, skin=0.6),
        systems.zincblende(tb, sic_text, 4, jitter=0.1, seed=1, skin=0.5),
        systems.zincblende(tb, sic_text, 3, jitter=0.0, skin=1.0),
        systems.liquid_like(tb, 4, 0.35, 5),
        systems.open_cluster(tb),
        systems.slab_mixed(tb),
        systems.dimer(tb),
    ]


@pytest.fixture(scope="module")
def cases(tb, sic_text):
    return _cases(tb, sic_text)


def test_neighbor_lists_bit_exact(tb, oracle, cases):
    for case in cases:
        params, ctx = _ctx(tb, case)
        off, nb = ctx.export_neighbors("skin")
        ooff, onb = oracle.build_neighbor_list(case.xyz, case.box, case.periodic,
                                               params.r_cut_max, case.skin)
        assert np.array_equal(off, ooff), case.name
        assert np.array_equal(nb, onb), case.name
        soff, snb = ctx.export_neighbors("short")
        xoff, xnb = oracle.filter(case.xyz, case.box, case.periodic, ooff, onb, params.r_cut_max)
        assert np.array_equal(soff, xoff), case.name
        assert np.array_equal(snb, xnb), case.name
        ctx.close()


def test_neighbor_list_matches_brute_force(tb, oracle):
    case = systems.perturbed(tb, 2, 0.35, 41, skin=0.6)
    params, ctx = _ctx(tb, case)
    off, nb = ctx.export_neighbors("skin")
    boff, bnb = oracle.brute_neighbor_list(case.xyz, case.box, case.periodic,
                                           params.r_cut_max + 0.6)
    assert np.array_equal(off, boff) and np.array_equal(nb, bnb)


@pytest.mark.parametrize("deterministic", [True, False])
def test_double_parity(tb, oracle, cases, deterministic):
    for case in cases:
        params, ctx = _ctx(tb, case)
        _, _, _, ref = _oracle(oracle, case, params)
        e, f, w = ctx.compute("double", deterministic=deterministic)
        scale = abs(ref["energy"]) if ref["energy"] != 0 else 1.0
        assert abs(e - ref["energy"]) <= E_TOL_D * scale, (case.name, e, ref["energy"])
        assert np.abs(f - ref["forces"]).max(initial=0) <= F_TOL_D, case.name
        wscale = max(1.0, np.abs(ref["virial"]).max())
        assert np.abs(w - ref["virial"]).max() <= 1e-10 * wscale, (case.name, w, ref["virial"])
        ctx.close()


@pytest.mark.parametrize("precision", ["mixed", "single"])
@pytest.mark.parametrize("deterministic", [True, False])
def test_reduced_precision(tb, oracle, cases, precision, deterministic):
    for case in cases:
        params, ctx = _ctx(tb, case)
        _, _, _, ref = _oracle(oracle, case, params)
        e, f, w = ctx.compute(precision, deterministic=deterministic)
        scale = abs(ref["energy"]) if ref["energy"] != 0 else 1.0
        assert abs(e - ref["energy"]) <= E_TOL_M * scale, (case.name, e, ref["energy"])
        fscale = max(1.0, np.abs(ref["forces"]).max(initial=0))
        assert np.abs(f - ref["forces"]).max(initial=0) <= F_TOL_M * fscale, case.name
        ctx.close()


def test_appendix_d_goldens(tb):
    """SURVEY.md Appendix D energies (bitwise reference outputs), double mode."""
    params = tb.builtin_silicon()
    for case, e_gold in [(systems.diamond(tb, 4), -2370.7709768772361),
                         (systems.perturbed(tb, 4, 0.12, 32, 0.5), -2318.8092698921296),
                         (systems.perturbed(tb, 2, 0.12, 722, 0.5), -289.24149471763792)]:
        _, ctx = _ctx(tb, case)
        e, f, _ = ctx.compute("double", deterministic=True)
        assert abs(e - e_gold) <= 1e-12 * abs(e_gold)
        ctx.close()
    case = systems.perturbed(tb, 4, 0.12, 32, 0.5)
    _, ctx = _ctx(tb, case)
    _, f, _ = ctx.compute("double")
    np.testing.assert_allclose(f[0], [-1.5906421510252808, -1.1016438175896053,
                                      1.0033862477768203], rtol=0, atol=1e-10)


def test_deterministic_mode_is_bitwise_reproducible(tb, sic_text):
    for case in [systems.liquid_like(tb, 4, 0.35, 5), systems.zincblende(tb, sic_text, 4, jitter=0.1)]:
        _, ctx = _ctx(tb, case)
        for prec in ("double", "mixed", "single"):
            e1, f1, w1 = ctx.compute(prec, deterministic=True)
            e2, f2, w2 = ctx.compute(prec, deterministic=True)
            assert e1 == e2 and np.array_equal(f1, f2) and np.array_equal(w1, w2)
        ctx.close()


def test_virial_free_kernels_match(tb, sic_text):
    """TSF_NO_VIRIAL / a NULL virial next to energy or forces selects kernels
    that never form the virial (the MD loop and the drop-in shim use them):
    in deterministic mode energy and forces are bitwise those of the full
    kernels — the G = 4 main launch, the packed main launch (SiC) and the
    packed tier (a liquid-like system at G = 4) — and the device virial is
    zero; all three precisions."""
    from paper_1607_02904_b200 import _lib as L
    import ctypes as C
    cases = [systems.perturbed(tb, 4, 0.12, 52, skin=0.5), systems.liquid_like(tb, 4, 0.35, 5),
             systems.zincblende(tb, sic_text, 4, jitter=0.1)]
    for case in cases:
        _, ctx = _ctx(tb, case)
        for prec in ("double", "mixed", "single"):
            e1, f1, w1 = ctx.compute(prec, deterministic=True)
            e2, f2, w2 = ctx.compute(prec, deterministic=True, virial=False)
            assert w2 is None and e1 == e2 and np.array_equal(f1, f2), (case.name, prec)
            e3, f3, _ = ctx.compute(prec, deterministic=True, energy=True, forces=True,
                                    virial=False, form_virial=False)
            assert e1 == e3 and np.array_equal(f1, f3)
            ctx.compute(prec, deterministic=True, energy=False, forces=False, virial=False,
                        form_virial=False)
            import torch
            d = torch.empty(7, dtype=torch.float64, device="cuda:0")
            ctx._ok(L.lib().tsf_results_device(ctx._h, C.c_void_p(d.data_ptr()), None))
            torch.cuda.synchronize()
            ev = d.cpu().numpy()
            assert ev[0] == e1 and np.all(ev[1:] == 0.0), (case.name, prec, ev)
            assert np.abs(w1).max() > 0
        ctx.close()


def test_filter_off_matches_filter_on(tb, oracle):
    """Acceptance criterion 5 (acceptance.cpp:195-230): 1e-12 relative."""
    case = systems.perturbed(tb, 4, 0.12, 52, skin=0.5)
    _, ctx = _ctx(tb, case)
    e1, f1, _ = ctx.compute("double", deterministic=True, filter=True)
    e2, f2, _ = ctx.compute("double", deterministic=True, filter=False)
    scale = max(1.0, np.abs(f1).max())
    assert abs(e1 - e2) <= 1e-12 * abs(e1)
    assert np.abs(f1 - f2).max() <= 1e-12 * scale


def test_overflow_path_between_rebuilds(tb, oracle):
    """List built on an ordered lattice (4 short neighbours -> group width 4),
    then atoms move inside the skin so some gain 5-8 short neighbours without
    a rebuild: those atoms take the G = 32 overflow launch."""
    base = systems.diamond(tb, 4, skin=1.0)
    params, ctx = _ctx(tb, base)
    rng = np.random.default_rng(9)
    moved = np.mod(base.xyz + rng.uniform(-0.4, 0.4, base.xyz.shape), base.box)
    ctx.set_positions(moved)
    from oracle.oracle import parse_param_text
    op = parse_param_text(base.params_text)
    off, nb = ctx.export_neighbors("skin")          # the list built on `base`
    soff, _ = ctx.export_neighbors("short")
    assert np.diff(soff).max() > 4
    ref = oracle.compute_ref(op, moved, base.species, base.box, base.periodic, off, nb)
    for det in (True, False):
        e, f, _ = ctx.compute("double", deterministic=det)
        assert abs(e - ref["energy"]) <= E_TOL_D * abs(ref["energy"])
        assert np.abs(f - ref["forces"]).max() <= F_TOL_D


def test_external_neighbor_list(tb, oracle):
    """tsf_set_neighbor_list: evaluate on a list built elsewhere (the
    reference's NeighborList), here the oracle's."""
    case = systems.perturbed(tb, 3, 0.2, 7, skin=0.5)
    params = tb.builtin_silicon()
    op, off, nb, ref = _oracle(oracle, case, params)
    ctx = tb.Context(params, 0)
    ctx.set_system(case.xyz, case.species, case.box, case.periodic)
    ctx.set_neighbor_list(off, nb, params.r_cut_max, case.skin)
    e, f, _ = ctx.compute("double", deterministic=True)
    assert abs(e - ref["energy"]) <= E_TOL_D * abs(ref["energy"])
    assert np.abs(f - ref["forces"]).max() <= F_TOL_D


def test_needs_rebuild_threshold(tb):
    """test_neighbor.cpp:65-76: exactly skin/2 does not trigger, 0.51 skin does."""
    xyz = np.array([[1.0, 1.0, 1.0], [3.0, 1.0, 1.0]])
    box = np.array([60.0, 60.0, 60.0])
    ctx = tb.Context(None, 0)
    ctx.set_system(xyz, [0, 0], box, [0, 0, 0])
    ctx.build_neighbor_list(2.5, 0.5)
    assert not ctx.needs_rebuild()
    x2 = xyz.copy()
    x2[0, 0] = 0.75
    ctx.set_positions(x2)
    assert not ctx.needs_rebuild()
    x2[0, 0] = 1.0 - 0.51 * 0.5
    ctx.set_positions(x2)
    assert ctx.needs_rebuild()


def test_neighbor_boundary_inclusive(tb):
    """test_neighbor.cpp:17-32: d = 3.5 with cutoff 3.0 + skin 0.5 is listed."""
    for dist, listed in [(2.0, True), (3.5, True), (3.6, False)]:
        ctx = tb.Context(None, 0)
        ctx.set_system([[5, 5, 5], [5 + dist, 5, 5]], [0, 0], [60.0, 60.0, 60.0], [0, 0, 0])
        ctx.build_neighbor_list(3.0, 0.5)
        off, nb = ctx.export_neighbors("skin")
        assert list(np.diff(off)) == ([1, 1] if listed else [0, 0])


def test_bad_inputs_refused(tb):
    params = tb.builtin_silicon()
    case = systems.perturbed(tb, 2, 0.1, 3)
    ctx = tb.Context(params, 0)
    ctx.set_system(case.xyz, case.species, case.box, case.periodic)
    with pytest.raises(tb.ConfigError):
        ctx.build_neighbor_list(3.2, -0.1)
    ctx.set_system(case.xyz, case.species, case.box * np.array([1, 0.6, 1]), case.periodic)
    with pytest.raises(tb.ConfigError):
        ctx.build_neighbor_list(3.2, 0.5)
    with pytest.raises(tb.ConfigError):
        ctx.set_system(case.xyz, np.full(len(case.xyz), 3, np.int32), case.box, case.periodic)
    fresh = tb.Context(params, 0)
    fresh.set_system(case.xyz, case.species, case.box, case.periodic)
    with pytest.raises(tb.ConfigError):
        fresh.compute("double")


def test_trivial_systems(tb, oracle):
    params = tb.builtin_silicon()
    ctx = tb.Context(params, 0)
    ctx.set_system(np.zeros((1, 3)) + 5.0, [0], [60.0, 60.0, 60.0], [0, 0, 0])
    ctx.build_neighbor_list(params.r_cut_max, 0.5)
    e, f, w = ctx.compute("double")
    assert e == 0.0 and np.all(f == 0)
    case = systems.dimer(tb, 2.25)
    _, ctx = _ctx(tb, case)
    e, f, _ = ctx.compute("double", deterministic=True)
    ref = _oracle(oracle, case, params)[3]
    assert abs(e - ref["energy"]) <= 1e-14 * abs(ref["energy"])
    assert f[0, 1] == 0 and f[0, 2] == 0 and abs(f[0, 0] + f[1, 0]) <= 1e-15


def test_evaluate_forces_api(tb, oracle):
    """The tersoffmd-shaped surface: options validated like potential_opt.cpp."""
    params = tb.builtin_silicon()
    s = tb.perturbed_lattice(params, 2, 0.12, 722)
    lst = tb.build_neighbor_list(s, params.r_cut_max, 0.5)
    assert lst.natoms == 64 and lst.pair_count == 312
    assert not tb.needs_rebuild(lst, s)
    e, f = tb.evaluate_forces(s, lst, params)
    assert abs(e - (-289.24149471763792)) <= 1e-12 * 289.3
    assert np.abs(f.sum(axis=0)).max() < 1e-10
    e8, f8 = tb.evaluate_forces(s, lst, params, scheme="v2", width=8, deterministic=False)
    assert abs(e8 - e) <= 1e-12 * abs(e) and np.abs(f8 - f).max() <= 1e-10
    es, _ = tb.evaluate_forces(s, lst, params, precision="single")
    assert abs(es - e) <= 1e-6 * abs(e)
    with pytest.raises(tb.ConfigError):
        tb.evaluate_forces(s, lst, params, scheme="v9")
    with pytest.raises(tb.ConfigError):
        tb.evaluate_forces(s, lst, params, width=3)
    with pytest.raises(tb.ConfigError):
        tb.evaluate_forces(s, lst, params, scheme="ref", precision="single")


def test_melted_liquid(tb, oracle):
    """A real liquid (GPU melt, SURVEY.md 8d cfg 5 protocol, shortened):
    irregular short counts, atoms in the cutoff ramp, G = 8/16 groups."""
    s = tb.melt(tb.make_diamond_lattice(3, 3, 3), tb.builtin_silicon(), hot_ps=0.25,
                hold_ps=0.25)
    case = systems.Case("melt216", s.positions, s.species, s.box.lengths, s.box.periodic, 1.0,
                        systems.si_text(tb))
    params, ctx = _ctx(tb, case)
    op, off, nb, ref = _oracle(oracle, case, params)
    goff, gnb = ctx.export_neighbors("skin")
    assert np.array_equal(goff, off) and np.array_equal(gnb, nb)
    soff, _ = ctx.export_neighbors("short")
    assert np.diff(soff).max() > 4 and np.diff(soff).min() < 4
    for det in (True, False):
        e, f, _ = ctx.compute("double", deterministic=det)
        assert abs(e - ref["energy"]) <= E_TOL_D * abs(ref["energy"])
        assert np.abs(f - ref["forces"]).max() <= F_TOL_D
        for prec in ("mixed", "single"):
            e, f, _ = ctx.compute(prec, deterministic=det)
            assert abs(e - ref["energy"]) <= E_TOL_M * abs(ref["energy"])
            assert np.abs(f - ref["forces"]).max() <= F_TOL_M * np.abs(ref["forces"]).max()


def test_large_n_against_compensated_oracle(tb, oracle):
    """32k atoms (cfg-2 size): energy vs the long-double oracle sum."""
    s = tb.make_diamond_lattice(20, 20, 10)
    rng = np.random.default_rng(2)
    xyz = np.mod(s.positions + rng.uniform(-0.1, 0.1, s.positions.shape), s.box.lengths)
    case = systems.Case("si32k", xyz, s.species, s.box.lengths, s.box.periodic, 1.0,
                        systems.si_text(tb))
    params, ctx = _ctx(tb, case)
    _, _, _, ref = _oracle(oracle, case, params)
    for det in (True, False):
        e, f, _ = ctx.compute("double", deterministic=det)
        assert abs(e - ref["energy_ld"]) <= 1e-12 * abs(ref["energy_ld"])
        assert np.abs(f - ref["forces"]).max() <= F_TOL_D
    for prec in ("mixed", "single"):
        e, f, _ = ctx.compute(prec)
        assert abs(e - ref["energy_ld"]) <= E_TOL_M * abs(ref["energy_ld"])
        assert np.abs(f - ref["forces"]).max() <= F_TOL_M * max(1, np.abs(ref["forces"]).max())


@pytest.mark.parametrize("width", ["4", "8", "16", "32"])
def test_group_width_tiers(tb, oracle, monkeypatch, width):
    """Pinned main group width on a dense packing (8..21 short neighbours):
    atoms over the width go through the G=16 and G=32 tier launches; every
    width gives the oracle's energy, forces and virial."""
    monkeypatch.setenv("TSF_GROUP_WIDTH", width)
    case = systems.dense_random(tb)
    params, ctx = _ctx(tb, case)
    _, _, _, ref = _oracle(oracle, case, params)
    fscale = max(1.0, np.abs(ref["forces"]).max())
    for det in (True, False):
        e, f, w = ctx.compute("double", deterministic=det)
        assert abs(e - ref["energy"]) <= E_TOL_D * abs(ref["energy"])
        assert np.abs(f - ref["forces"]).max() <= F_TOL_D * fscale
        assert np.abs(w - ref["virial"]).max() <= 1e-10 * max(1.0, np.abs(ref["virial"]).max())
        e, f, _ = ctx.compute("single", deterministic=det)
        assert abs(e - ref["energy"]) <= E_TOL_M * abs(ref["energy"])
        assert np.abs(f - ref["forces"]).max() <= F_TOL_M * fscale
    ctx.close()


def test_short_export_keeps_reference_filter(tb, oracle, sic_text):
    """The force path filters SiC pairs by their species-pair cutoff; the
    exported short list stays the reference's r_cut_max list
    (neighbor.cpp:143-180) before and after a force evaluation."""
    case = systems.zincblende(tb, sic_text, 4, jitter=0.1, seed=1, skin=0.5)
    params, ctx = _ctx(tb, case)
    ooff, onb = oracle.build_neighbor_list(case.xyz, case.box, case.periodic, params.r_cut_max,
                                           case.skin)
    xoff, xnb = oracle.filter(case.xyz, case.box, case.periodic, ooff, onb, params.r_cut_max)
    for _ in range(2):
        ctx.compute("double")
        soff, snb = ctx.export_neighbors("short")
        assert np.array_equal(soff, xoff) and np.array_equal(snb, xnb)
    ctx.close()


def test_lammps_style_table_gives_identical_results(tb, sic_text):
    """n = beta = 0 on the cross rows changes nothing: those fields are never
    read, so the LAMMPS-format table gives bitwise the same energy, forces and
    virial as the golden file (which carries n = 1 there)."""
    case = systems.zincblende(tb, sic_text, 4, jitter=0.1, seed=1, skin=0.5)
    out = []
    for text in (case.params_text, systems.lammps_style(case.params_text)):
        params = tb.parse_params(text)
        ctx = tb.Context(params, 0)
        ctx.set_system(case.xyz, case.species, case.box, case.periodic)
        ctx.build_neighbor_list(params.r_cut_max, case.skin)
        out.append([ctx.compute(p, deterministic=True) for p in ("double", "mixed", "single")])
        ctx.close()
    for (e1, f1, w1), (e2, f2, w2) in zip(*out):
        assert e1 == e2 and np.array_equal(f1, f2) and np.array_equal(w1, w2)


def test_graph_replay_follows_new_positions(tb, oracle):
    """Steady-state evaluations replay a captured CUDA graph (evaluate() in
    tsf_capi.cu): after set_positions (same list, no rebuild) the replay must
    use the new positions — equal to a fresh context's eager evaluation (to
    summation order) and to the oracle on the moved configuration."""
    case = systems.perturbed(tb, 4, 0.12, 32, skin=0.5)
    params, ctx = _ctx(tb, case)
    for _ in range(3):                        # eager, capture, replay
        ctx.compute("double", deterministic=True)
    rng = np.random.default_rng(5)
    moved = np.mod(case.xyz + rng.uniform(-0.05, 0.05, case.xyz.shape), case.box)
    ctx.set_positions(moved)                  # within skin/2: no rebuild
    e1, f1, w1 = ctx.compute("double", deterministic=True)   # a replay
    e1b, f1b, _ = ctx.compute("double", deterministic=True)
    assert e1 == e1b and np.array_equal(f1, f1b)
    fresh = tb.Context(params, 0)             # its first evaluation is eager
    fresh.set_system(moved, case.species, case.box, case.periodic)
    fresh.set_neighbor_list(*ctx.export_neighbors("skin"), params.r_cut_max, case.skin)
    e2, f2, w2 = fresh.compute("double", deterministic=True)
    assert abs(e1 - e2) <= 1e-13 * abs(e2) and np.abs(f1 - f2).max() <= 1e-12
    from oracle.oracle import parse_param_text
    op = parse_param_text(case.params_text)
    off, nb = ctx.export_neighbors("skin")
    ref = oracle.compute_ref(op, moved, case.species, case.box, case.periodic, off, nb)
    assert abs(e1 - ref["energy"]) <= E_TOL_D * abs(ref["energy"])
    assert np.abs(f1 - ref["forces"]).max() <= F_TOL_D
    for c in (ctx, fresh):
        c.close()


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["crystal", "liquid", "sic"])
def test_near_list_filter_is_exact(tb, kind, sic_text):
    """While 2 |d|max < h (h = s/4, s/2) the filter reads a near list — the
    skin entries within r_cut_max + h at the build — instead of the skin list
    (Ctx::near_list in tsf_context.hpp).  Move every atom by exactly |d| = D
    (random directions, so pairs approach by up to 2 D) on both sides of each
    switch (D = s/8, s/4) and check the short list and forces against a
    context fed the same skin list externally, which never uses a near list."""
    if kind == "crystal":
        case = systems.perturbed(tb, 4, 0.12, 32, skin=1.0)
    elif kind == "liquid":
        case = systems.liquid_like(tb, cells=4, skin=1.0)
    else:
        case = systems.zincblende(tb, sic_text, cells=4, jitter=0.1, seed=3, skin=1.0)
    params, ctx = _ctx(tb, case)
    skin_off, skin_nb = ctx.export_neighbors("skin")
    fresh = tb.Context(params, 0)
    rng = np.random.default_rng(11)
    reach = case.skin         # list cutoff r_cut_max + skin: s = skin
    for frac in (0.0, 0.05, 0.124, 0.126, 0.2, 0.249, 0.251, 0.3, 0.49):
        d = rng.normal(size=case.xyz.shape)
        d *= (frac * reach) / np.linalg.norm(d, axis=1, keepdims=True)
        moved = np.mod(case.xyz + d, case.box)
        ctx.set_positions(moved)
        assert not ctx.needs_rebuild()
        fresh.set_system(moved, case.species, case.box, case.periodic)
        fresh.set_neighbor_list(skin_off, skin_nb, params.r_cut_max, case.skin)
        for which in ("short",):
            a_off, a_nb = ctx.export_neighbors(which)
            b_off, b_nb = fresh.export_neighbors(which)
            assert np.array_equal(a_off, b_off) and np.array_equal(a_nb, b_nb), frac
        for prec in ("double", "mixed"):
            e1, f1, _ = ctx.compute(prec, deterministic=True)
            e2, f2, _ = fresh.compute(prec, deterministic=True)
            # same lists; the two contexts differ only in slot order (summation
            # order of the energy, and of float partials in mixed)
            tol = 1e-13 if prec == "double" else 1e-6
            assert abs(e1 - e2) <= tol * abs(e2), (frac, prec)
            ftol = 1e-12 if prec == "double" else 2e-6 * max(1.0, np.abs(f2).max())
            assert np.abs(f1 - f2).max() <= ftol, (frac, prec)
    if kind == "sic":
        # a species change keeps the list (set_system, same n and box): the
        # sure bits are species-independent, so the lists still agree
        ctx.set_positions(case.xyz)
        ctx.build_neighbor_list(params.r_cut_max, case.skin)   # |d|max = 0: near lists
        skin_off, skin_nb = ctx.export_neighbors("skin")
        sp = case.species.copy()
        flip = rng.random(len(sp)) < 0.3
        sp[flip] = 1 - sp[flip]
        ctx.set_system(case.xyz, sp, case.box, case.periodic)
        assert not ctx.needs_rebuild()
        fresh.set_system(case.xyz, sp, case.box, case.periodic)
        fresh.set_neighbor_list(skin_off, skin_nb, params.r_cut_max, case.skin)
        a_off, a_nb = ctx.export_neighbors("short")
        b_off, b_nb = fresh.export_neighbors("short")
        assert np.array_equal(a_off, b_off) and np.array_equal(a_nb, b_nb)
        e1, f1, _ = ctx.compute("double", deterministic=True)
        e2, f2, _ = fresh.compute("double", deterministic=True)
        assert abs(e1 - e2) <= 1e-13 * abs(e2) and np.abs(f1 - f2).max() <= 1e-12
    for c in (ctx, fresh):
        c.close()


@pytest.mark.parametrize("mode", ["0", "1", "2"])
def test_packed_lane_groups(tb, oracle, sic_text, monkeypatch, mode):
    """Packed lane groups (tsf_force_packed.cuh) against the oracle on the
    irregular systems: TSF_PACKED=0 the G-tier chain, 1 (default) one packed
    launch behind the G = 4 main launch (or packed from the start for
    irregular systems), 2 packed main launch everywhere — all precisions,
    both scatter modes; deterministic mode bitwise reproducible."""
    monkeypatch.setenv("TSF_PACKED", mode)
    for case in [systems.dense_random(tb), systems.liquid_like(tb, 4, 0.35, 5),
                 systems.zincblende(tb, sic_text, 4, jitter=0.1, seed=1, skin=0.5),
                 systems.perturbed(tb, 4, 0.12, 32, skin=0.5)]:
        params, ctx = _ctx(tb, case)
        _, _, _, ref = _oracle(oracle, case, params)
        fscale = max(1.0, np.abs(ref["forces"]).max())
        for det in (True, False):
            e, f, w = ctx.compute("double", deterministic=det)
            assert abs(e - ref["energy"]) <= E_TOL_D * abs(ref["energy"]), (case.name, det)
            assert np.abs(f - ref["forces"]).max() <= F_TOL_D * fscale, (case.name, det)
            assert np.abs(w - ref["virial"]).max() <= 1e-10 * max(1.0, np.abs(ref["virial"]).max())
            for prec in ("mixed", "single"):
                e, f, _ = ctx.compute(prec, deterministic=det)
                assert abs(e - ref["energy"]) <= E_TOL_M * abs(ref["energy"]), (case.name, prec)
                assert np.abs(f - ref["forces"]).max() <= F_TOL_M * fscale, (case.name, prec)
        e1, f1, w1 = ctx.compute("double", deterministic=True)
        e2, f2, w2 = ctx.compute("double", deterministic=True)
        assert e1 == e2 and np.array_equal(f1, f2) and np.array_equal(w1, w2)
        ctx.close()


def test_asymmetric_cutoff_table(tb, oracle, sic_text):
    """A LAMMPS-format table may give rows (i, *, k) and (k, *, i) different
    cutoffs: here every Si-*-C row reaches 2.75 A and every
    C-*-Si row 2.51 A, on a zincblende lattice stretched so the Si-C first
    shell sits at 2.6 A.  The short-list bounds are symmetrised, so the
    deterministic scatter (each atom gathers the slots of the centres in its
    own list) and the atomics agree with the oracle."""
    rows = []
    for line in sic_text.splitlines():
        t = line.split()
        if len(t) == 17 and not line.lstrip().startswith("#"):
            if t[0] == "Si" and t[2] == "C":
                t[13], t[14] = "2.65", "0.10"          # R, D: cutoff 2.75
            elif t[0] == "C" and t[2] == "Si":
                t[13], t[14] = "2.41", "0.10"          # cutoff 2.51
            line = " ".join(t)
        rows.append(line)
    text = "\n".join(rows) + "\n"
    case = systems.zincblende(tb, text, 3, a0=6.0, jitter=0.12, seed=4, skin=0.5)
    params, ctx = _ctx(tb, case)
    _, _, _, ref = _oracle(oracle, case, params)
    assert ref["energy"] != 0
    for det in (True, False):
        e, f, w = ctx.compute("double", deterministic=det)
        assert abs(e - ref["energy"]) <= E_TOL_D * abs(ref["energy"]), det
        assert np.abs(f - ref["forces"]).max() <= F_TOL_D, det
    ctx.close()


def test_evaluate_forces_resident_species(tb, oracle):
    """tsf_evaluate_forces with species = NULL on a repeat call keeps the
    resident species (the e2e path sends positions only); NULL before any
    species were given is a ConfigError."""
    import ctypes as C
    from paper_1607_02904_b200 import _lib as L
    case = systems.perturbed(tb, 3, 0.15, 8, skin=0.5)
    params = tb.parse_params(case.params_text)
    _, _, _, ref = _oracle(oracle, case, params)
    lib = L.lib()
    ctx = tb.Context(params, 0)
    n = len(case.xyz)
    xyz = np.ascontiguousarray(case.xyz)
    box = np.ascontiguousarray(case.box, np.float64)
    per = np.ascontiguousarray(case.periodic, np.uint8)
    sp = np.ascontiguousarray(case.species, np.int32)
    e = C.c_double()
    f = np.zeros((n, 3))
    vp = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    assert lib.tsf_evaluate_forces(ctx._h, 0, n, vp(xyz), None, vp(box), vp(per), 0.5, 0,
                                   C.byref(e), vp(f), None) == L.TSF_ERR_CONFIG
    for species in (vp(sp), None, None):
        assert lib.tsf_evaluate_forces(ctx._h, 0, n, vp(xyz), species, vp(box), vp(per), 0.5,
                                       L.TSF_DETERMINISTIC, C.byref(e), vp(f), None) == 0
        assert abs(e.value - ref["energy"]) <= E_TOL_D * abs(ref["energy"])
        assert np.abs(f - ref["forces"]).max() <= F_TOL_D
    ctx.close()
