import sys, time, os
sys.path.insert(0,'.')
import torch, paper_1607_02904_b200 as tb
p=tb.builtin_silicon(); s=tb.make_diamond_lattice(20,20,10); tb.init_velocities(s,1600.0,12345)
ctx=tb.Context(p,0); ctx.load(s); ctx.build_neighbor_list(p.r_cut_max,1.0); ctx.md_set_state(s.velocities,s.species_masses)
for prec in ["double"]*3+["mixed"]*4+["double"]*2:
    l0=ctx.launches; torch.cuda.synchronize(); t=time.perf_counter()
    th,reb=ctx.md_run(100,0.001,prec,thermo_every=100)
    torch.cuda.synchronize(); dt=(time.perf_counter()-t)/100
    print(prec, f"{dt*1e6:.1f} us/step reb {reb} launches/step {(ctx.launches-l0)/100:.1f}", flush=True)
