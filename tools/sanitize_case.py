"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
512-atom Si lattice (G = 4 main launch), a disordered 512-atom system and a
dense random packing (G = 8/16/32 tier launches), both scatter modes, all
three precisions, CUDA-graph replay, a 30-step GPU-resident NVE run with
rebuilds, and the list exports.
  compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_1607_02904_b200 as tb  # noqa: E402
import systems  # noqa: E402

sic = open(os.path.join(ROOT, "tests", "golden", "SiC.tersoff")).read()
cases = [systems.perturbed(tb, 4, 0.12, 32, skin=0.5), systems.liquid_like(tb, 4, 0.35, 5),
         systems.dense_random(tb, 600), systems.zincblende(tb, sic, 3, jitter=0.1)]
for case in cases:
    params = tb.parse_params(case.params_text)
    ctx = tb.Context(params, 0)
    ctx.set_system(case.xyz, case.species, case.box, case.periodic)
    ctx.build_neighbor_list(params.r_cut_max, case.skin)
    ctx.export_neighbors("skin")
    ctx.export_neighbors("short")
    for prec in ("double", "mixed", "single"):
        for det in (False, True):
            for _ in range(3):            # eager, warm, graph capture + replay
                e, f, w = ctx.compute(prec, deterministic=det)
            assert np.isfinite(e), case.name
    ctx.close()
s = tb.make_diamond_lattice(4, 4, 4)
tb.init_velocities(s, 1600.0, 12345)
rep = tb.run_nve(s, tb.builtin_silicon(), 30, thermo_every=10)
print("sanitize case done:", len(cases), "systems; NVE rebuilds", rep["neighbor_rebuilds"])
