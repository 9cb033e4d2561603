"""Per-rank projection of the C++ decomposition (csrc/tsf_dd.cu) on ONE GPU.

Every rank of an N-way x-slab split of a bench workload is set up exactly as
`bench.py --gpus N` sets it up (tsf_dd over the LOCAL transport: one host
thread per rank, ghosts selected and exchanged on the device), then each
rank's evaluation is timed ALONE on the GPU with CUDA events (graph replay,
steady state): the compute side of a rank's step — what the N GPUs would run
concurrently.  The bound on strong-scaling efficiency from compute alone is
T1 / (N x slowest rank).  The NVLink exchange itself is not measured (one GPU).

  python tools/rank_share_dd.py [config] [precision] [N ...]
"""
import json
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1607_02904_b200 as tb  # noqa: E402
from paper_1607_02904_b200 import parallel as PD  # noqa: E402


def time_ctx(ctx, prec, steps=200):
    stream = torch.cuda.ExternalStream(ctx.stream, device=0)
    for _ in range(5):
        ctx.compute(prec, energy=False, forces=False, virial=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        ctx.compute(prec, energy=False, forces=False, virial=False)
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "si2m"
    prec = sys.argv[2] if len(sys.argv) > 2 else "double"
    worlds = [int(x) for x in sys.argv[3:]] or [1, 2, 4, 8]
    text, xyz, species, box, per, masses = bench.make_system(cfg)
    params = tb.parse_params(text)
    halo = params.r_cut_max + 1.0
    out = {"config": cfg, "precision": prec, "ranks": {}}
    t1 = None
    for world in worlds:
        group = PD.LocalGroup(world)
        dds = [None] * world
        gc = box[0] / world > 4 * halo + 1e-9
        if os.environ.get("RS_GC") == "0":
            gc = False

        def setup(r):
            d = PD.DomainDecomposition(params, 0, box, per, params.r_cut_max, 1.0, group, r,
                                       ghost_centers=gc)
            gid = PD.partition(xyz, box, world, r)
            d.setup(gid, xyz[gid], species[gid])
            dds[r] = d
        th = [threading.Thread(target=setup, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        ms = [time_ctx(d.ctx, prec) for d in dds]
        slow = dds[int(np.argmax(ms))].ctx
        slow.profile(True)
        for _ in range(50):
            slow.compute(prec, energy=False, forces=False, virial=False)
        pr = slow.profile_read(reset=True)
        slow.profile(False)
        stages = {k: v / max(pr["calls"], 1) for k, v in pr.items() if k.endswith("_ms")}
        counts = [d.counts for d in dds]
        if world == 1:
            t1 = ms[0]
        bound = t1 / (world * max(ms)) if t1 else None
        out["ranks"][world] = {"rank_ms": ms, "slowest_ms": max(ms), "bound": bound,
                               "owned": [c["owned"] for c in counts],
                               "centres": [c["centres"] for c in counts],
                               "local": [c["local"] for c in counts],
                               "ghost_centers": bool(gc), "slowest_rank_stages_ms": stages}
        print(world, f"slowest {max(ms):.4f} ms", f"bound {bound}", stages, flush=True)
        for d in dds:
            d.close()
        group.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
