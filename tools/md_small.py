import sys, time
sys.path.insert(0,'.')
import torch, paper_1607_02904_b200 as tb
p=tb.builtin_silicon(); s=tb.make_diamond_lattice(20,20,10); tb.init_velocities(s,1600.0,12345)
for prec in ("mixed","double","mixed"):
    ctx=tb.Context(p,0); ctx.load(s); ctx.build_neighbor_list(p.r_cut_max,1.0); ctx.md_set_state(s.velocities,s.species_masses)
    ctx.md_run(30,0.001,prec,thermo_every=100)
    torch.cuda.synchronize(); t=time.perf_counter()
    th,reb=ctx.md_run(300,0.001,prec,thermo_every=100)
    torch.cuda.synchronize(); dt=(time.perf_counter()-t)/300
    l0=ctx.launches
    ctx.profile(True); ctx.md_run(100,0.001,prec,thermo_every=100); pr=ctx.profile_read(); ctx.profile(False)
    print(prec, f"{dt*1e6:.1f} us/step", reb, {k: round(v/max(pr['calls'],1)*1e3,2) for k,v in pr.items() if k.endswith('_ms')}, pr['calls'])
    t=time.perf_counter()
    for _ in range(5): ctx.build_neighbor_list(p.r_cut_max,1.0)
    torch.cuda.synchronize(); print(' build us', (time.perf_counter()-t)/5*1e6)
    for _ in range(3): ctx.compute(prec, energy=False, forces=False, virial=False)
    torch.cuda.synchronize(); t=time.perf_counter()
    for _ in range(200): ctx.compute(prec, energy=False, forces=False, virial=False)
    torch.cuda.synchronize(); print(' eval us', (time.perf_counter()-t)/200*1e6)
    ctx.close()
