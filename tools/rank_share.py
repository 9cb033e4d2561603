"""Per-rank compute of the x-slab decomposition, emulated on ONE
B200: a projection of the strong-scaling bound, not a multi-GPU measurement.

Only one GPU is available to this build, so `bench.py --gpus N` is unmeasured
at N > 1.  This tool builds every rank r of an N-way decomposition of the same
global system exactly as `bench.py --gpus N` does (Decomposition with
ghost_centers when the slabs are >= 4 halo wide, overlap=True), with the
ghost payload of the setup exchanged through host mailboxes (threads, like
tests/test_gpu_parallel.py — no kernel waits on another rank's).  Then, one
rank at a time and alone on the GPU, it times the rank's steady-state step
with CUDA events: the send-buffer gathers, phase 0 (interior centres), the
ghost scatters and phase 1 — everything `Decomposition.evaluate` issues except
the NCCL transfer itself (positions are static: the receive buffers keep what
one mailbox forward exchange after the setup delivered).  It also times phase 0 alone: the
window the forward exchange hides behind.

Reported per N: the max / mean rank step, T1 / (N x max rank step) (the
compute-side strong-scaling bound), the bytes each rank sends per step, and
the phase-0 window.  usage: python tools/rank_share.py [config] [steps] [N...]
"""
import json
import os
import queue
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import bench  # noqa: E402  (make_system: the bench's own synthetic input)
import paper_1607_02904_b200 as tb  # noqa: E402
import dd_model as P  # noqa: E402


class Mailbox:
    def __init__(self):
        self.q = {}
        self.lock = threading.Lock()

    def box(self, src, dst, tag):
        with self.lock:
            return self.q.setdefault((src, dst, tag), queue.Queue())


def make_rank(text, xyz, species, box, per, world, rank, mail, out, skin):
    params = tb.parse_params(text)
    halo = params.r_cut_max + skin
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        eng = P.GpuEngine(params, 0)
        dec = P.Decomposition.__new__(P.Decomposition)
        dec.engine, dec.group = eng, None
        dec.rank, dec.world = rank, world
        dec.box, dec.periodic = np.asarray(box, np.float64), np.asarray(per, np.uint8)
        gc = world > 1 and box[0] / world >= 4 * halo          # bench.py's rule
        if os.environ.get("RS_GC") == "0":                     # classic mode: reverse exchange
            gc = False
        # RS_OVERLAP=0: the one-phase step (graph-replayed evaluation after a
        # blocking exchange) instead of bench.py's overlapped split
        dec.ghost_centers = gc
        dec.overlap = os.environ.get("RS_OVERLAP", "1") != "0"
        dec.slab = P.Slab(rank, world, float(box[0]), halo)
        dec.slab_sel = P.Slab(rank, world, float(box[0]), 2 * halo if gc else halo)
        dec.left, dec.right = (rank - 1) % world, (rank + 1) % world
        dec.migrated = 0

        def exchange(sends, recvs):
            torch.cuda.current_stream().synchronize()
            for t, dst, tag in sends:
                mail.box(rank, dst, tag).put(t.cpu().clone())
            for t, src, tag in recvs:
                t.copy_(mail.box(src, rank, tag).get(timeout=600).to(t.device))
            torch.cuda.current_stream().synchronize()
        dec._exchange = exchange
        gid = P.partition(xyz, box, world, rank, halo)
        dec.setup(gid, xyz[gid], species[gid], params.r_cut_max, skin)
        # one real forward exchange (mailbox) fills the receive buffers the
        # timed steps scatter from: the ghosts then hold their owners' positions
        dec.forward()
        torch.cuda.current_stream().synchronize()
        out[rank] = (eng, dec, stream)


def time_rank(eng, dec, stream, precision, steps):
    """Steady-state step of one rank, NCCL transfer excluded; and phase 0 alone."""
    dec._exchange = lambda s, r: None
    dec._exchange_start = lambda s, r: []
    dec._exchange_finish = lambda reqs: None
    with torch.cuda.stream(stream):
        for _ in range(5):
            dec.evaluate(precision)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.nvtx.range_push("rs_steps")
        h0 = time.perf_counter()
        e0.record(stream)
        for _ in range(steps):
            dec.evaluate(precision)
        e1.record(stream)
        host_ms = (time.perf_counter() - h0) * 1e3 / steps     # enqueue rate of the host
        e1.synchronize()
        torch.cuda.nvtx.range_pop()
        step_ms = e0.elapsed_time(e1) / steps
        phase0_ms = 0.0
        if dec.world > 1:
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(steps)]
            for a, b in ev:                  # queued back to back, like the bench
                a.record(stream)
                eng.compute_phase(0, precision)
                b.record(stream)
                eng.compute_phase(1, precision)
            torch.cuda.synchronize()
            phase0_ms = sum(a.elapsed_time(b) for a, b in ev) / steps
        # stage split of the (one-phase) evaluation: profiling runs eagerly,
        # event-timed per stage (filter / setup / main force launch / tiers +
        # reduction) — the diagnostic behind the fixed per-step cost
        eng.ctx.profile(True)
        for _ in range(steps):
            dec.evaluate(precision)
        prof = eng.ctx.profile_read(reset=True)
        eng.ctx.profile(False)
        calls = max(prof["calls"], 1)
        stages = {k: prof[k] / calls for k in ("filter_ms", "setup_ms", "force_ms", "tail_ms")}
    return step_ms, phase0_ms, host_ms, stages


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "si2m"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    worlds = [int(x) for x in sys.argv[3:]] or [1, 2, 4, 8]
    text, xyz, species, box, per, _ = bench.make_system(cfg)
    skin = 1.0
    res = {"config": cfg, "n_atoms": len(xyz), "steps": steps, "precision": {},
           "overlap": os.environ.get("RS_OVERLAP", "1") != "0",
           "ghost_centres_allowed": os.environ.get("RS_GC") != "0",
           "note": "projection on ONE B200: each rank's step timed alone, NCCL transfer "
                   "excluded (tools/rank_share.py)"}
    for precision in os.environ.get("RS_PRECISIONS", "double,mixed").split(","):
        rows = {}
        t1 = None
        for world in worlds:
            mail, out = Mailbox(), {}
            th = [threading.Thread(target=make_rank,
                                   args=(text, xyz, species, box, per, world, r, mail, out, skin))
                  for r in range(world)]
            for t in th:
                t.start()
            for t in th:
                t.join()
            assert len(out) == world, "rank setup failed"
            per_rank = []
            only = os.environ.get("RS_RANKS")       # time a subset (ncu runs)
            for r in (range(world) if not only else range(min(int(only), world))):
                eng, dec, stream = out[r]
                step_ms, p0_ms, host_ms, stages = time_rank(eng, dec, stream, precision, steps)
                sent = 24 * (len(dec.send_left) + len(dec.send_right))
                per_rank.append({"rank": r, "owned": dec.n_owned, "ghosts": len(dec.ghost_gid),
                                 "centres": dec.n_centers, "interior": dec.n_interior,
                                 "step_ms": step_ms, "phase0_ms": p0_ms, "host_enqueue_ms": host_ms,
                                 "stages_one_phase": stages,
                                 "send_bytes_per_step": sent})
            gcent = bool(out[0][1].ghost_centers)
            for r in range(world):
                out[r][0].ctx.close()
            mx = max(p["step_ms"] for p in per_rank)
            if world == 1:
                t1 = mx
            row = {"ghost_centers": gcent,
                   "max_rank_step_ms": mx,
                   "mean_rank_step_ms": float(np.mean([p["step_ms"] for p in per_rank])),
                   "min_phase0_ms": min(p["phase0_ms"] for p in per_rank),
                   "max_send_bytes_per_step": max(p["send_bytes_per_step"] for p in per_rank),
                   "ranks": per_rank}
            if t1 is not None:
                row["compute_efficiency_bound"] = t1 / (world * mx)
            rows[str(world)] = row
            print(json.dumps({"precision": precision, "world": world,
                              "max_rank_step_ms": mx,
                              "eff": row.get("compute_efficiency_bound")}), flush=True)
        res["precision"][precision] = rows
    print(json.dumps(res))


if __name__ == "__main__":
    main()
