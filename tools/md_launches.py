"""Short GPU-resident NVE run of cfg 4 (2,048,000 Si, 1600 K) inside an NVTX
range "md_steps", for an ncu launch list of the MD step:
  ncu --metrics gpu__time_duration.sum --nvtx --nvtx-include md_steps/ \\
      --csv python tools/md_launches.py [precision] [steps]"""
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

import paper_1607_02904_b200 as tb  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "double"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
p = tb.builtin_silicon()
s = tb.make_diamond_lattice(80, 80, 40)
tb.init_velocities(s, 1600.0, 12345)
ctx = tb.Context(p, 0)
ctx.load(s)
ctx.build_neighbor_list(p.r_cut_max, 1.0)
ctx.md_set_state(s.velocities, s.species_masses)
ctx.md_run(20, 0.001, prec, thermo_every=100)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("md_steps")
_, reb = ctx.md_run(steps, 0.001, prec, thermo_every=100)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("rebuilds", reb)
