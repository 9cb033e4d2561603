"""MD step time (2M and 32k Si, 1600 K, f64) under different segment / graph
settings, each in a fresh process: python tools/md_segments_ab.py"""
import json
import os
import subprocess
import sys

CODE = r'''
import sys, time, json
sys.path.insert(0, ".")
import torch, paper_1607_02904_b200 as tb
cells = tuple(int(x) for x in sys.argv[1].split("x"))
p = tb.builtin_silicon(); s = tb.make_diamond_lattice(*cells); tb.init_velocities(s, 1600.0, 12345)
ctx = tb.Context(p, 0); ctx.load(s); ctx.build_neighbor_list(p.r_cut_max, 1.0)
ctx.md_set_state(s.velocities, s.species_masses)
ctx.md_run(40, 0.001, "double", thermo_every=100)
torch.cuda.synchronize(); t = time.perf_counter()
_, reb = ctx.md_run(400, 0.001, "double", thermo_every=100)
torch.cuda.synchronize()
print(json.dumps({"us_per_step": (time.perf_counter() - t) / 400 * 1e6, "rebuilds": reb}))
'''
# extra variants: python tools/md_segments_ab.py [LIB ...] (TSF_LIBRARY builds to compare)
VARIANTS = [{}, {"TSF_MD_SEGMENT": "1"}, {"TSF_MD_SEGMENT": "16"}, {"TSF_GRAPHS": "0"}]
VARIANTS += [{"TSF_LIBRARY": lib} for lib in sys.argv[1:]]
for cells in ("80x80x40", "20x20x10"):
    for env in VARIANTS:
        out = subprocess.run([sys.executable, "-c", CODE, cells], capture_output=True, text=True,
                             env=dict(os.environ, **env))
        print(cells, env, out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:],
              flush=True)
