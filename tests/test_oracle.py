"""The CPU oracle pinned before it is trusted (CPU only).

* against the SURVEY.md Appendix D hexfloat goldens (reference outputs);
* against tests/golden/goldens.json, written from the unmodified reference
  by tools/make_goldens.py (bitwise: energies, forces, lists);
* against the live reference library when oracle/_ref is present;
* known-answer tests of the scalar pieces (proj/tests/test_potential.cpp);
* analytic forces vs central differences; virial vs strain derivatives.
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

import systems
from oracle.oracle import parse_param_text

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def golden_cases(tb):
    sic = open(os.path.join(GOLDEN, "SiC.tersoff")).read()
    cs = {c.name: c for c in [
        systems.diamond(tb, 4),
        systems.perturbed(tb, 4, 0.12, 32, skin=0.5),
        systems.perturbed(tb, 2, 0.12, 722, skin=0.5),
        systems.perturbed(tb, 2, 0.35, 41, skin=0.6),
        systems.perturbed(tb, 3, 0.2, 7, skin=0.5),
        systems.zincblende(tb, sic, 4, jitter=0.0, skin=1.0),
        systems.zincblende(tb, sic, 4, jitter=0.1, seed=1, skin=0.5),
        systems.liquid_like(tb, 4, 0.35, 5),
        systems.open_cluster(tb),
        systems.slab_mixed(tb),
        systems.dimer(tb),
    ]}
    return cs


def run_oracle(oracle, c):
    op = parse_param_text(c.params_text)
    off, nb = oracle.build_neighbor_list(c.xyz, c.box, c.periodic, op.r_cut_max, c.skin)
    soff, snb = oracle.filter(c.xyz, c.box, c.periodic, off, nb, op.r_cut_max)
    ref = oracle.compute_ref(op, c.xyz, c.species, c.box, c.periodic, off, nb)
    return op, off, nb, soff, snb, ref


def test_appendix_d_hexfloats(tb, oracle):
    for case, hexe in [(systems.diamond(tb, 4), "-0x1.2858abd7b3367p+11"),
                       (systems.perturbed(tb, 4, 0.12, 32, 0.5), "-0x1.21d9e589f90abp+11"),
                       (systems.perturbed(tb, 2, 0.12, 722, 0.5), "-0x1.213dd2990a696p+8")]:
        *_, ref = run_oracle(oracle, case)
        assert ref["energy"].hex() == hexe, case.name
    *_, ref = run_oracle(oracle, systems.perturbed(tb, 4, 0.12, 32, 0.5))
    assert ref["forces"][0].tolist() == [-1.5906421510252808, -1.1016438175896053,
                                         1.0033862477768203]


def test_committed_goldens_bitwise(tb, oracle):
    """The oracle reproduces the reference's bits on every committed fixture."""
    gold = {c["name"]: c for c in json.load(open(os.path.join(GOLDEN, "goldens.json")))["cases"]}
    cases = golden_cases(tb)
    assert set(cases) <= set(gold)
    for name, c in cases.items():
        g = gold[name]
        assert sha(np.asarray(c.xyz, np.float64)) == g["xyz_sha256"], name
        op, off, nb, soff, snb, ref = run_oracle(oracle, c)
        assert ref["energy"].hex() == g["energy_hex"], name
        assert sha(ref["forces"]) == g["forces_sha256"], name
        assert sha(np.concatenate([off, nb])) == g["skin_sha256"], name
        assert sha(np.concatenate([soff, snb])) == g["short_sha256"], name


def test_against_live_reference(tb, oracle, reference):
    R = reference
    for name, c in golden_cases(tb).items():
        ph = R.params(c.params_text)
        sh = R.system(c.xyz, c.species, [28.0855, 12.011][: int(c.species.max()) + 1], c.box,
                      c.periodic)
        lh = R.neighbor_list(sh, R.lib.tmdref_params_r_cut_max(ph), c.skin)
        e, f = R.compute_ref(sh, lh, ph, len(c.xyz))
        op, off, nb, soff, snb, ref = run_oracle(oracle, c)
        roff, rnb = R.list_csr(lh, len(c.xyz))
        assert np.array_equal(off, roff) and np.array_equal(nb, rnb), name
        assert ref["energy"] == e and np.array_equal(ref["forces"], f), name


def test_brute_force_equals_cell_list(tb, oracle):
    for c in [systems.perturbed(tb, 2, 0.35, 41, skin=0.6), systems.open_cluster(tb),
              systems.slab_mixed(tb)]:
        op = parse_param_text(c.params_text)
        off, nb = oracle.build_neighbor_list(c.xyz, c.box, c.periodic, op.r_cut_max, c.skin)
        boff, bnb = oracle.brute_neighbor_list(c.xyz, c.box, c.periodic, op.r_cut_max + c.skin)
        assert np.array_equal(off, boff) and np.array_equal(nb, bnb), c.name


def test_neighbor_list_rejections(oracle):
    from oracle.oracle import OracleConfigError
    xyz = np.zeros((2, 3)) + 1.0
    with pytest.raises(OracleConfigError):
        oracle.build_neighbor_list(xyz, [60, 60, 60], [1, 1, 1], 3.2, -0.1)
    with pytest.raises(OracleConfigError):   # periodic edge below 2 (rc + skin)
        oracle.build_neighbor_list(xyz, [60, 7.3, 60], [1, 1, 1], 3.2, 0.5)


# ---- known answers, proj/tests/test_potential.cpp ------------------------
TEST_ENTRY = "Xx Xx Xx 1 1.2 0.9 1.5 0.8 -0.3 0.9 0.4 1.7 12.0 2.0 0.5 2.1 25.0\n"


def test_cutoff_ramp_pins(oracle):
    assert oracle.cutoff_fc(1.2, 2.0, 0.5) == (1.0, 0.0)
    v, d = oracle.cutoff_fc(2.0, 2.0, 0.5)
    assert v == 0.5 and abs(d - (-math.pi / 2)) <= 1e-15 * math.pi / 2
    assert oracle.cutoff_fc(2.5, 2.0, 0.5)[0] == 0.0     # upper boundary is outside
    assert oracle.cutoff_fc(1.5, 2.0, 0.5)[0] == 1.0     # lower boundary is inside
    for r in (1.7, 1.9, 2.0, 2.2, 2.4):
        h = 1e-7
        fd = (oracle.cutoff_fc(r + h, 2.0, 0.5)[0] - oracle.cutoff_fc(r - h, 2.0, 0.5)[0]) / (2 * h)
        assert abs(oracle.cutoff_fc(r, 2.0, 0.5)[1] - fd) <= 1e-6 * max(1, abs(fd))


def test_bond_order_pins(oracle):
    row = parse_param_text(TEST_ENTRY).rows[0].copy()
    assert oracle.bond_order(0.0, row) == (1.0, 0.0)
    row[5], row[6] = 1.0, 1.0                             # beta = eta = 1
    assert oracle.bond_order(3.0, row)[0] == 0.5


def test_forces_are_energy_gradient(tb, oracle):
    """Acceptance criterion 3 (acceptance.cpp:130-148): h = 1e-5, 1e-6 relative."""
    c = systems.perturbed(tb, 2, 0.12, 33, skin=0.5)
    op = parse_param_text(c.params_text)
    off, nb = oracle.build_neighbor_list(c.xyz, c.box, c.periodic, op.r_cut_max, c.skin)
    ref = oracle.compute_ref(op, c.xyz, c.species, c.box, c.periodic, off, nb)
    h = 1e-5
    fd = np.zeros_like(ref["forces"])
    for a in range(len(c.xyz)):
        for k in range(3):
            xp, xm = c.xyz.copy(), c.xyz.copy()
            xp[a, k] += h
            xm[a, k] -= h
            ep = oracle.compute_ref(op, xp, c.species, c.box, c.periodic, off, nb)["energy"]
            em = oracle.compute_ref(op, xm, c.species, c.box, c.periodic, off, nb)["energy"]
            fd[a, k] = -(ep - em) / (2 * h)
    scale = max(1.0, np.abs(ref["forces"]).max())
    assert np.abs(fd - ref["forces"]).max() / scale < 1e-6


def _strained_energy(oracle, op, c, off, nb, eps):
    F = np.eye(3) + eps
    return oracle.compute_ref(op, c.xyz @ F.T, c.species, np.diag(F) * c.box, c.periodic, off,
                              nb)["energy_ld"]


def test_virial_is_strain_derivative(tb, oracle):
    """NEW output (no reference counterpart): W_ab = sum d_a f_b.
    Periodic box: diagonal vs -dE/d eps_aa under affine scaling.  Open cluster:
    all six components vs -dE/d eps_ab (no box to shear)."""
    h = 1e-6
    for c, comps in [(systems.perturbed(tb, 2, 0.12, 9, skin=0.5), [(0, 0), (1, 1), (2, 2)]),
                     (systems.open_cluster(tb), [(0, 0), (1, 1), (2, 2), (0, 1), (0, 2),
                                                 (1, 2)])]:
        op = parse_param_text(c.params_text)
        off, nb = oracle.build_neighbor_list(c.xyz, c.box, c.periodic, op.r_cut_max, c.skin)
        w = oracle.compute_ref(op, c.xyz, c.species, c.box, c.periodic, off, nb)["virial"]
        idx = {(0, 0): 0, (1, 1): 1, (2, 2): 2, (0, 1): 3, (0, 2): 4, (1, 2): 5}
        for a, b in comps:
            e = np.zeros((3, 3))
            e[a, b] = h
            fd = -(_strained_energy(oracle, op, c, off, nb, e) -
                   _strained_energy(oracle, op, c, off, nb, -e)) / (2 * h)
            # W_ab = sum d_a f_b = -dE/d eps_ba
            assert abs(w[idx[(a, b)]] - fd) <= 1e-6 * max(1.0, abs(fd)), (c.name, a, b, w, fd)


def test_compensated_energy_tracks_naive(tb, oracle):
    *_, ref = run_oracle(oracle, systems.perturbed(tb, 4, 0.12, 32, 0.5))
    assert abs(ref["energy"] - ref["energy_ld"]) <= 1e-13 * abs(ref["energy"])


def test_cfg2_nve_golden(reference):
    """SURVEY.md 8d cfg 2: the reference Engine (ref scheme, 1 thread) on
    20x20x10 cells at 1600 K, seed 12345, dt 1 fs, skin 1, 100 steps gives
    Etot0 / Etot100 / rebuilds — the golden test_gpu_scale.py holds the GPU
    engine to (bitwise here: this glibc and these compile flags)."""
    from oracle.oracle import SI_TEXT
    from test_gpu_scale import CFG2_ETOT0, CFG2_ETOT100, CFG2_REBUILDS
    R = reference
    h = R.diamond_lattice(20, 20, 10)
    R.init_velocities(h, 1600.0, 12345)
    ph = R.params(SI_TEXT)
    rep = R.run_nve(h, ph, 100, dt=0.001, skin=1.0, scheme="ref", precision="ref",
                    thermo_every=10)
    assert rep["etot_first"] == CFG2_ETOT0
    assert rep["etot_last"] == CFG2_ETOT100
    assert rep["rebuilds"] == CFG2_REBUILDS
    R.free_system(rep["final"])
    R.free_system(h)
    R.free_params(ph)
