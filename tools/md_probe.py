"""GPU-resident NVE step time at 2M atoms (tsf_md_run, f64, 1600 K): 20 steps
warm-up, then ms/step over 50 steps, rebuilds included.  Run on a GPU box."""
import sys, time
sys.path.insert(0, '.')
import torch, bench, paper_1607_02904_b200 as tb
text, xyz, species, box, per, masses = bench.make_system("si2m")
p = tb.parse_params(text)
s = tb.make_diamond_lattice(80, 80, 40)
tb.init_velocities(s, 1600.0, 12345)
ctx = tb.Context(p, 0); ctx.load(s); ctx.build_neighbor_list(p.r_cut_max, 1.0)
ctx.md_set_state(s.velocities, s.species_masses)
ctx.md_run(20, 0.001, "double", thermo_every=100)
torch.cuda.synchronize(); t = time.perf_counter()
rep = ctx.md_run(50, 0.001, "double", thermo_every=100)
torch.cuda.synchronize(); print("ms/step", (time.perf_counter() - t) / 50 * 1e3, "rebuilds", rep[1])
