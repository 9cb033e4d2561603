#!/usr/bin/env python
"""Regenerate tests/golden/goldens.json from the UNMODIFIED reference.

Runs only in the dev container (needs oracle/_ref/libtmdref.so, built from
/root/reference/proj/src by oracle/Makefile).  The fixtures it writes travel
with the repo, so the GPU box — where /root/reference does not exist — can
still pin the oracle and the GPU path to the reference's own outputs.

Per system: the inputs' recipe, the reference's energy (hexfloat), SHA-256 of
its forces (float64 bytes) and of its skin / short neighbor lists (int32
CSR bytes), a few force rows, and the reference's single/mixed-precision
energies (evaluate_forces v2/w8).

  python tools/make_goldens.py
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1607_02904_b200 as tb  # noqa: E402  (host-side generators only)
import systems  # noqa: E402
from oracle.oracle import Reference  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sic_jittered_mt(tb, sic_text):
    """SURVEY.md Appendix F check: zincblende 512 atoms, a0 = 4.32, jittered
    +-0.1 A by mt19937_64 seed 1 (verify.cpp:27-36 draws), skin 0.5."""
    s = tb.make_diamond_lattice(4, 4, 4, 4.32)
    sp = np.where(np.arange(s.natoms) % 8 < 4, 0, 1).astype(np.int32)
    # same draws as perturbed_lattice: mt19937_64, 53-bit uniforms, x then y then z
    params = tb.parse_params(sic_text)
    pl = tb.perturbed_lattice(params, 4, 0.1, 1)   # gives the jittered lattice at a0 = 1.697*3.0
    # rescale the jitter onto the a0 = 4.32 lattice: recompute offsets
    base = tb.make_diamond_lattice(4, 4, 4, 1.697 * params.r_cut_max).positions
    off = pl.positions - base
    off -= pl.box.lengths * np.round(off / pl.box.lengths)
    xyz = np.mod(s.positions + off, s.box.lengths)
    return systems.Case("sic4_mt1", xyz, sp, s.box.lengths, s.box.periodic, 0.5, sic_text)


def main():
    R = Reference()
    sic_text = open(os.path.join(ROOT, "tests", "golden", "SiC.tersoff")).read()
    cases = [
        systems.diamond(tb, 4),
        systems.perturbed(tb, 4, 0.12, 32, skin=0.5),
        systems.perturbed(tb, 2, 0.12, 722, skin=0.5),
        systems.perturbed(tb, 2, 0.35, 41, skin=0.6),
        systems.perturbed(tb, 3, 0.2, 7, skin=0.5),
        systems.zincblende(tb, sic_text, 4, jitter=0.0, skin=1.0),
        systems.zincblende(tb, sic_text, 4, jitter=0.1, seed=1, skin=0.5),
        sic_jittered_mt(tb, sic_text),
        systems.liquid_like(tb, 4, 0.35, 5),
        systems.open_cluster(tb),
        systems.slab_mixed(tb),
        systems.dimer(tb),
    ]
    out = []
    for c in cases:
        ph = R.params(c.params_text)
        masses = [28.0855, 12.011][: int(c.species.max()) + 1]
        sh = R.system(c.xyz, c.species, masses, c.box, c.periodic)
        n = len(c.xyz)
        lh = R.neighbor_list(sh, R.lib.tmdref_params_r_cut_max(ph), c.skin)
        off, nb = R.list_csr(lh, n)
        soff, snb = R.filter_csr(lh, sh, R.lib.tmdref_params_r_cut_max(ph), n)
        e, f = R.compute_ref(sh, lh, ph, n)
        def reduced(prec):
            # the reference's float pow bond order overflows for beta*zeta > ~48
            # (SURVEY.md 7c-4): record the NumericError instead of a number
            try:
                return R.evaluate(sh, lh, ph, n, "v2", prec, 8)[0]
            except Exception as exc:  # noqa: BLE001
                return f"error: {exc}"
        es, em = reduced("opt-s"), reduced("opt-m")
        out.append({
            "name": c.name, "n": n, "skin": c.skin,
            "xyz_sha256": sha(np.asarray(c.xyz, np.float64)),
            "energy": e, "energy_hex": float(e).hex(),
            "forces_sha256": sha(f), "forces_head": f[:4].tolist(),
            "max_abs_force": float(np.abs(f).max()),
            "skin_entries": int(len(nb)), "skin_sha256": sha(np.concatenate([off, nb])),
            "short_entries": int(len(snb)), "short_sha256": sha(np.concatenate([soff, snb])),
            "ref_opt_s_energy": es, "ref_opt_m_energy": em,
        })
        for h in (lh,):
            R.free_list(h)
        R.free_system(sh)
        R.free_params(ph)
        print(f"{c.name:24s} n={n:5d} E={e:.13f} skin={len(nb)} short={len(snb)}")
    path = os.path.join(ROOT, "tests", "golden", "goldens.json")
    with open(path, "w") as fh:
        json.dump({"generator": "tools/make_goldens.py", "reference": "/root/reference/proj "
                   "(oracle/_ref/libtmdref.so, g++ -O3 -DNDEBUG -ffp-contract=off)",
                   "cases": out}, fh, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
