"""Margin of the reduced-precision paths against the parity gates: for every
GPU parity case, |dE|/|E| (gate 1e-6) and max|dF| / max(1, max|F|) (gate
1e-4) of mixed and single against the FP64 oracle.  Run on a GPU box."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1607_02904_b200 as tb  # noqa: E402
import systems  # noqa: E402
from oracle.oracle import Oracle, parse_param_text  # noqa: E402


def main():
    sic = open(os.path.join(ROOT, "tests", "golden", "SiC.tersoff")).read()
    cases = [systems.diamond(tb, 4), systems.perturbed(tb, 4, 0.12, 32, skin=0.5),
             systems.perturbed(tb, 2, 0.35, 41, skin=0.6),
             systems.zincblende(tb, sic, 4, jitter=0.1, seed=1, skin=0.5),
             systems.liquid_like(tb, 4, 0.35, 5), systems.dense_random(tb),
             systems.open_cluster(tb), systems.slab_mixed(tb)]
    orc = Oracle()
    out = {}
    for case in cases:
        params = tb.parse_params(case.params_text)
        ctx = tb.Context(params, 0)
        ctx.set_system(case.xyz, case.species, case.box, case.periodic)
        ctx.build_neighbor_list(params.r_cut_max, case.skin)
        op = parse_param_text(case.params_text)
        off, nb = orc.build_neighbor_list(case.xyz, case.box, case.periodic, op.r_cut_max,
                                          case.skin)
        ref = orc.compute_ref(op, case.xyz, case.species, case.box, case.periodic, off, nb)
        fscale = max(1.0, np.abs(ref["forces"]).max(initial=0))
        row = {}
        for prec in ("mixed", "single"):
            e, f, _ = ctx.compute(prec)
            row[prec] = {"dE_rel": abs(e - ref["energy"]) / max(abs(ref["energy"]), 1e-300),
                         "dF_scaled": float(np.abs(f - ref["forces"]).max(initial=0) / fscale)}
        out[case.name] = row
        ctx.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
