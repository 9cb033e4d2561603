"""Seeded test systems shared by the CPU and GPU suites.

Positions come from the product generators (bit-identical to the reference's
make_diamond_lattice / perturbed_lattice, pinned in test_generators.py) or from
numpy with a fixed seed; the same arrays feed the GPU path and the oracle.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Case:
    name: str
    xyz: np.ndarray
    species: np.ndarray
    box: np.ndarray
    periodic: np.ndarray
    skin: float
    params_text: str


def _wrap(xyz, box):
    return np.mod(xyz, box)


def si_text(tb):
    return tb.builtin_silicon().serialize()


def diamond(tb, cells=4, a0=5.431, skin=1.0, name=None):
    s = tb.make_diamond_lattice(cells, cells, cells, a0)
    return Case(name or f"diamond{cells}", s.positions, s.species, s.box.lengths,
                s.box.periodic, skin, si_text(tb))


def perturbed(tb, cells, jitter, seed, skin=0.5, text=None):
    params = tb.builtin_silicon() if text is None else tb.parse_params(text)
    s = tb.perturbed_lattice(params, cells, jitter, seed)
    return Case(f"perturbed{cells}_{jitter}_{seed}", s.positions, s.species, s.box.lengths,
                s.box.periodic, skin, params.serialize())


def zincblende(tb, sic_text, cells=4, a0=4.32, jitter=0.0, seed=1, skin=1.0):
    """3C-SiC: basis 0-3 Si, 4-7 C (SURVEY.md 8d cfg 3)."""
    s = tb.make_diamond_lattice(cells, cells, cells, a0)
    sp = np.where(np.arange(s.natoms) % 8 < 4, 0, 1).astype(np.int32)
    xyz = s.positions.copy()
    if jitter:
        rng = np.random.default_rng(seed)
        xyz = _wrap(xyz + rng.uniform(-jitter, jitter, xyz.shape), s.box.lengths)
    return Case(f"sic{cells}_{jitter}", xyz, sp, s.box.lengths, s.box.periodic, skin, sic_text)


def liquid_like(tb, cells=4, jitter=0.35, seed=5, skin=1.0):
    """Strongly disordered Si: irregular short counts (3..8+) exercise the
    group-width choice and the overflow path."""
    s = tb.make_diamond_lattice(cells, cells, cells, 5.431)
    rng = np.random.default_rng(seed)
    xyz = _wrap(s.positions + rng.uniform(-jitter, jitter, s.positions.shape), s.box.lengths)
    return Case(f"disordered{cells}_{jitter}", xyz, s.species, s.box.lengths, s.box.periodic,
                skin, si_text(tb))


def open_cluster(tb, n=64, seed=3, skin=0.5):
    """Atoms in an open (non-periodic) box: occupied-extent binning path."""
    s = tb.make_diamond_lattice(2, 2, 2, 5.431)
    rng = np.random.default_rng(seed)
    xyz = s.positions[:n] + 10.0 + rng.uniform(-0.1, 0.1, (n, 3))
    return Case("open_cluster", xyz, s.species[:n], np.array([60.0, 60.0, 60.0]),
                np.zeros(3, np.uint8), skin, si_text(tb))


def dimer(tb, r=2.25):
    xyz = np.array([[5.0, 5.0, 5.0], [5.0 + r, 5.0, 5.0]])
    return Case("dimer", xyz, np.zeros(2, np.int32), np.array([60.0, 60.0, 60.0]),
                np.zeros(3, np.uint8), 0.5, si_text(tb))


def slab_mixed(tb):
    """Periodic in x and y, open in z."""
    s = tb.make_diamond_lattice(3, 3, 2, 5.431)
    rng = np.random.default_rng(11)
    xyz = s.positions + rng.uniform(-0.1, 0.1, s.positions.shape)
    xyz[:, :2] = np.mod(xyz[:, :2], s.box.lengths[:2])
    return Case("slab_xy", xyz, s.species, s.box.lengths, np.array([1, 1, 0], np.uint8), 0.8,
                si_text(tb))


def dense_random(tb, n=1200, density=0.14, dmin=1.5, seed=21, skin=0.5):
    """Random sequential packing (no pair closer than dmin) at ~2x the
    crystal density: 3..25 short neighbours per atom, so every lane-group
    tier (4 -> 16 -> 32) carries atoms."""
    rng = np.random.default_rng(seed)
    box = np.full(3, (n / density) ** (1.0 / 3.0))
    pts = np.empty((n, 3))
    m = 0
    while m < n:
        p = rng.uniform(0.0, box)
        if m:
            d = pts[:m] - p
            d -= box * np.round(d / box)
            if (d * d).sum(axis=1).min() < dmin * dmin:
                continue
        pts[m] = p
        m += 1
    return Case(f"dense_random{n}", pts, np.zeros(n, np.int32), box, np.ones(3, np.uint8), skin,
                si_text(tb))


def lammps_style(text):
    """The same table as LAMMPS writes it: n = beta = 0 on the cross rows
    (i, j, k), j != k, whose bond-order fields are never read (only (i, j, j)
    rows feed b_ij and the pair terms)."""
    out = []
    for line in text.splitlines():
        t = line.split()
        if len(t) == 17 and not line.lstrip().startswith("#") and t[1] != t[2]:
            t[9] = "0.0"    # eta (n)
            t[10] = "0.0"   # beta
            line = " ".join(t)
        out.append(line)
    return "\n".join(out) + "\n"


# ---- BASELINE.json configurations at their full sizes -------
LIQUID_SNAPSHOT = "liquid512k.tsfsnap"      # under tests/golden (tools/make_liquid_snapshot.py)


def baseline_cfg4(tb, cells=(80, 80, 40)):
    """cfg 4 as bench.py times it: Si diamond 80x80x40 = 2,048,000 atoms with a
    seeded uniform +-0.15 A jitter (seed 12345), wrapped into the box; skin 1."""
    s = tb.make_diamond_lattice(*cells, 5.431)
    rng = np.random.default_rng(12345)
    xyz = _wrap(s.positions + rng.uniform(-0.15, 0.15, s.positions.shape), s.box.lengths)
    return Case("cfg4_si2m", xyz, s.species, s.box.lengths, s.box.periodic, 1.0, si_text(tb))


def baseline_cfg3(tb, sic_text):
    """cfg 3 as bench.py times it: 3C-SiC 32^3 cells = 262,144 atoms at
    a0 = 4.32, +-0.10 A jitter (seed 12345)."""
    c = zincblende(tb, sic_text, 32, a0=4.32, jitter=0.10, seed=12345, skin=1.0)
    c.name = "cfg3_sic262k"
    return c


def baseline_cfg5(golden_dir):
    """cfg 5: the committed liquid-Si snapshot (512,000 atoms, 3000 K), read by
    the independent numpy reader so the oracle side never loads the product."""
    import os
    from oracle import snapshot as osnap
    from oracle.oracle import SI_TEXT
    d = osnap.read(os.path.join(golden_dir, LIQUID_SNAPSHOT))
    return Case("cfg5_liquid512k", d["positions"], d["species"], d["box"], d["periodic"], 1.0,
                SI_TEXT)
