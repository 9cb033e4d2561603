"""Where the GPU-resident NVE step goes at cfg 4 (2,048,000 Si, 1600 K, f64):
md_run ms/step over 200 steps, the per-stage split of its evaluations
(profile mode), list-build time, and the kick.  Run on a GPU box."""
import json
import sys
import time

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
ctx.md_run(20, 0.001, prec, thermo_every=100)
out = {"precision": prec}
torch.cuda.synchronize()
t = time.perf_counter()
_, reb = ctx.md_run(200, 0.001, prec, thermo_every=100)
torch.cuda.synchronize()
out["md_ms_per_step"] = (time.perf_counter() - t) / 200 * 1e3
out["rebuilds_per_200"] = reb
ctx.profile(True)
ctx.md_run(100, 0.001, prec, thermo_every=100)
pr = ctx.profile_read(reset=True)
ctx.profile(False)
out["eval_stages_ms"] = {k: v / max(pr["calls"], 1) for k, v in pr.items() if k.endswith("_ms")}
out["eval_calls"] = pr["calls"]
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    ctx.build_neighbor_list(p.r_cut_max, 1.0)
torch.cuda.synchronize()
out["list_build_ms"] = (time.perf_counter() - t) / 5 * 1e3
# first evaluation after a build (reads the short-count distribution back)
torch.cuda.synchronize()
t = time.perf_counter()
ctx.compute(prec, energy=False, forces=False, virial=False)
torch.cuda.synchronize()
out["first_eval_after_build_ms"] = (time.perf_counter() - t) * 1e3
for _ in range(3):
    ctx.compute(prec, energy=False, forces=False, virial=False)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(50):
    ctx.compute(prec, energy=False, forces=False, virial=False)
torch.cuda.synchronize()
out["eval_fresh_list_ms"] = (time.perf_counter() - t) / 50 * 1e3
t = time.perf_counter()
for _ in range(50):
    ctx.md_kick(0.001, drift=True, kicks=2, check=True)
torch.cuda.synchronize()
out["kick_with_flag_readback_ms"] = (time.perf_counter() - t) / 50 * 1e3
print(json.dumps(out))
