"""2M-atom Si, 60 NVE steps at 1600 K (the 5-neighbour population near its
peak), then three evaluations inside NVTX range "tier_eval" — for ncu
captures of the packed tier launch on an MD state (tools/ncu_md_tier.sh)."""
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

import paper_1607_02904_b200 as tb  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "double"
p = tb.builtin_silicon()
s = tb.make_diamond_lattice(80, 80, 40)
tb.init_velocities(s, 1600.0, 12345)
ctx = tb.Context(p, 0)
ctx.load(s)
ctx.build_neighbor_list(p.r_cut_max, 1.0)
ctx.md_set_state(s.velocities, s.species_masses)
ctx.md_run(60, 0.001, prec, thermo_every=100)
for _ in range(2):
    ctx.compute(prec, energy=False, forces=False, virial=False, form_virial=False)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("tier_eval")
for _ in range(3):
    ctx.compute(prec, energy=False, forces=False, virial=False, form_virial=False)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
