#!/usr/bin/env python
"""BASELINE cfg 2 and the north star's NVE drift report, on one B200.

Si diamond 20x20x10 (32,000 atoms), Maxwell-Boltzmann 1600 K (seed 12345),
dt = 1 fs, skin 1.0 A, rebuild check every step (engine.cpp:142-166 loop, run
GPU-resident by tsf_md_run).  For each precision: total-energy drift over the
run, rebuild count, and MD throughput (atom-steps/s including rebuilds and
thermo).  With --reference, the reference Engine::run (oracle/_ref, 1 thread,
Ref scheme) is timed on 100 steps of the same start state on this host.

  python tools/nve_drift.py [--steps 1000] [--reference] > profiles/nve_drift.json
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
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--cells", type=int, nargs=3, default=[20, 20, 10])
    ap.add_argument("--temperature", type=float, default=1600.0)
    ap.add_argument("--reference", action="store_true")
    args = ap.parse_args()
    import paper_1607_02904_b200 as tb

    params = tb.builtin_silicon()
    out = {"system": f"Si diamond {'x'.join(map(str, args.cells))}, "
                     f"{args.temperature:.0f} K seed 12345, dt 1 fs, skin 1.0 A",
           "steps": args.steps, "runs": {}}
    for prec in ("double", "mixed", "single"):
        s = tb.make_diamond_lattice(*args.cells)
        tb.init_velocities(s, args.temperature, 12345)
        rep = tb.run_nve(s, params, args.steps, dt=0.001, skin=1.0, precision=prec,
                         thermo_every=10)
        e = np.array([x["etot_eV"] for x in rep["samples"]])
        out["runs"][prec] = {
            "etot_first": float(e[0]), "etot_last": float(e[-1]),
            "max_rel_drift": float(np.abs(e - e[0]).max() / abs(e[0])),
            "final_rel_drift": float(abs(e[-1] - e[0]) / abs(e[0])),
            "final_temperature_K": rep["samples"][-1]["temp_K"],
            "rebuilds": rep["neighbor_rebuilds"],
            "wall_seconds": rep["wall_seconds"],
            "atom_steps_per_s": s.natoms * args.steps / rep["wall_seconds"],
            "ns_per_day": rep["ns_per_day"],
        }
        print(prec, out["runs"][prec], file=sys.stderr)
    if args.reference:
        from oracle.oracle import SI_TEXT, Reference, reference_available
        if reference_available():
            R = Reference()
            h = R.diamond_lattice(*args.cells)
            R.init_velocities(h, args.temperature, 12345)
            steps = 100
            rep = R.run_nve(h, R.params(SI_TEXT), steps, dt=0.001, skin=1.0, scheme="ref",
                            precision="ref", thermo_every=10)
            n = int(np.prod(args.cells)) * 8
            out["reference_engine"] = {
                "path": "Engine::run, compute_ref (1 thread), oracle/_ref", "steps": steps,
                "wall_seconds": rep["wall_seconds"], "rebuilds": rep["rebuilds"],
                "atom_steps_per_s": n * steps / rep["wall_seconds"],
                "etot_first": rep["etot_first"], "etot_last": rep["etot_last"],
                "cores": 1}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
