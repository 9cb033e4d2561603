#!/usr/bin/env python
"""Generate the BASELINE cfg 5 fixture: liquid Si, 40^3 diamond cells
(512,000 atoms), melted on the GPU with the SURVEY.md 8d recipe and saved as a
TSFSNAP1 snapshot (float32 coordinates: the stored, checksummed state is the
one every consumer evaluates).

Recipe (SURVEY.md 8d cfg 5; verified there on 1,728 atoms with the reference
Engine): make_diamond_lattice(40,40,40, 5.431), init_velocities(6000 K, seed
12345), hold 2 ps at 6000 K, then 4 ps at 3000 K, dt 0.5 fs, velocity
rescaling to the target every 50 steps; double precision, atomics scatter.

  python tools/make_liquid_snapshot.py [--cells 40] [--out tests/golden/liquid512k.tsfsnap]

Writes the snapshot and <out>.json (recipe, SHA-256, neighbor statistics).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=40)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "liquid512k.tsfsnap"))
    ap.add_argument("--hot-ps", type=float, default=2.0)
    ap.add_argument("--hold-ps", type=float, default=4.0)
    args = ap.parse_args()
    import paper_1607_02904_b200 as tb
    params = tb.builtin_silicon()
    s = tb.make_diamond_lattice(args.cells, args.cells, args.cells, 5.431)
    t0 = time.time()
    liq = tb.melt(s, params, hot_temperature=6000.0, hot_ps=args.hot_ps, temperature=3000.0,
                  hold_ps=args.hold_ps, dt=0.0005, rescale_every=50, seed=12345)
    t_melt = time.time() - t0
    sha = tb.save_snapshot(args.out, liq, float32_coords=True)
    back = tb.load_snapshot(args.out)
    ctx = tb.Context(params, 0)
    ctx.load(back)
    ctx.build_neighbor_list(params.r_cut_max, 1.0)
    so, _ = ctx.export_neighbors("short")
    ko, _ = ctx.export_neighbors("skin")
    e, _, _ = ctx.compute("double", deterministic=True, forces=False)
    sc, kc = np.diff(so), np.diff(ko)
    meta = {
        "file": os.path.relpath(args.out, ROOT), "sha256": sha, "natoms": back.natoms,
        "box": back.box.lengths.tolist(),
        "recipe": {"lattice": f"make_diamond_lattice({args.cells},{args.cells},{args.cells},5.431)",
                   "init_velocities": "6000 K, seed 12345", "hot": f"{args.hot_ps} ps at 6000 K",
                   "hold": f"{args.hold_ps} ps at 3000 K", "dt_ps": 0.0005,
                   "rescale_every": 50, "precision": "double", "scatter": "atomics",
                   "coords": "float32 (stored state)", "tool": "tools/make_liquid_snapshot.py"},
        "melt_wall_s": round(t_melt, 1),
        "stats": {"skin_mean": float(kc.mean()), "skin_max": int(kc.max()),
                  "short_mean": float(sc.mean()), "short_max": int(sc.max()),
                  "short_hist": {int(k): int(v) for k, v in
                                 zip(*np.unique(sc, return_counts=True))},
                  "pe_per_atom_eV": e / back.natoms},
    }
    json.dump(meta, open(args.out + ".json", "w"), indent=1)
    print(json.dumps(meta))


if __name__ == "__main__":
    main()
