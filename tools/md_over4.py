"""Short-count histogram of the 2M-atom Si crystal during the 1600 K NVE run
(the atoms the G = 4 main launch queues for the packed tier launch), and the
evaluation's stage split at that state.  Run on a GPU box."""
import json
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1607_02904_b200 as tb  # noqa: E402

p = tb.builtin_silicon()
s = tb.make_diamond_lattice(80, 80, 40)
tb.init_velocities(s, 1600.0, 12345)
ctx = tb.Context(p, 0)
ctx.load(s)
ctx.build_neighbor_list(p.r_cut_max, 1.0)
ctx.md_set_state(s.velocities, s.species_masses)
out = []
for seg in range(6):
    ctx.md_run(20, 0.001, "double", thermo_every=100)
    off, _ = ctx.export_neighbors("short")
    cnt = np.diff(off)
    h = np.bincount(cnt, minlength=8)
    ctx.profile(True)
    for _ in range(20):
        ctx.compute("double", energy=False, forces=False, virial=False)
    pr = ctx.profile_read(reset=True)
    ctx.profile(False)
    out.append({"step": 20 * (seg + 1), "hist": h.tolist(), "over4": int((cnt > 4).sum()),
                "stages_ms": {k: v / max(pr["calls"], 1) for k, v in pr.items() if k.endswith("_ms")}})
print(json.dumps(out))
