"""cfg 2 (Si 32,000 atoms, 1600 K) NVE inside NVTX range "md_steps" for an
ncu launch list of the small-system MD step (the paper's benchmark size)."""
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

import paper_1607_02904_b200 as tb  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "double"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
p = tb.builtin_silicon()
s = tb.make_diamond_lattice(20, 20, 10)
tb.init_velocities(s, 1600.0, 12345)
ctx = tb.Context(p, 0)
ctx.load(s)
ctx.build_neighbor_list(p.r_cut_max, 1.0)
ctx.md_set_state(s.velocities, s.species_masses)
ctx.md_run(30, 0.001, prec, thermo_every=100)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("md_steps")
_, reb = ctx.md_run(steps, 0.001, prec, thermo_every=100)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("rebuilds", reb)
