import sys, time
sys.path.insert(0,'.')
import torch, paper_1607_02904_b200 as tb
for cells in [(20,20,10),(80,80,40)]:
    p=tb.builtin_silicon(); s=tb.make_diamond_lattice(*cells); tb.init_velocities(s,1600.0,12345)
    ctx=tb.Context(p,0); ctx.load(s); ctx.build_neighbor_list(p.r_cut_max,1.0); ctx.md_set_state(s.velocities,s.species_masses)
    ctx.md_run(30,0.001,"double",thermo_every=100)
    for prec in ("double","mixed"):
        torch.cuda.synchronize(); t=time.perf_counter()
        th,reb=ctx.md_run(300,0.001,prec,thermo_every=100)
        torch.cuda.synchronize(); dt=(time.perf_counter()-t)/300
        print(cells, prec, f"{dt*1e6:.1f} us/step", reb, f"{s.natoms/dt:.3e} atom-steps/s")
    ctx.close()
