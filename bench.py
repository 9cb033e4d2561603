#!/usr/bin/env python
"""Benchmark of the B200 Tersoff force path (BASELINE.json metric: Tersoff
atom-steps/s on Si).

One step = one full evaluation of the hot path over the resident system:
short-list filter (paper Sec. 4.4) + fused zeta / bond-order / force kernel +
energy and virial reduction (+ deterministic gather when --deterministic).
The neighbor list is built once before timing, as a current list between
rebuilds (every ~25 steps at 1600 K).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--precision double|mixed|single]
                  [--config si2m|si32k|sic256k] [--impl ours|reference]

Prints one JSON line (rank 0).  `value` is device-resident throughput (CUDA
events on the context's stream, max over ranks); `e2e` is the same metric
through the reference-facing C-ABI call tsf_evaluate_forces with host
buffers (positions H2D and forces/energy/virial D2H inside the timed region).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Tersoff atom-steps/s (Si 32k/2M atoms)"
UNIT = "atom-steps/s"

CONFIGS = {
    # name: (cells, a0, jitter, params, description)
    "si2m": ((80, 80, 40), 5.431, 0.15, "si",
             "BASELINE cfg 4: Si diamond 80x80x40 = 2,048,000 atoms"),
    "si32k": ((20, 20, 10), 5.431, 0.15, "si", "BASELINE cfg 2 size: Si diamond 20x20x10 = 32,000 atoms"),
    "sic256k": ((32, 32, 32), 4.32, 0.10, "sic",
                "BASELINE cfg 3: 3C-SiC zincblende 32^3 = 262,144 atoms"),
    "liquid512k": ((40, 40, 40), 5.431, 0.0, "si",
                   "BASELINE cfg 5: liquid Si 40^3 cells = 512,000 atoms at 3000 K, the "
                   "committed snapshot tests/golden/liquid512k.tsfsnap (melted at 6000 K for "
                   "2 ps, held at 3000 K for 4 ps, dt 0.5 fs, velocity rescaling every 50 "
                   "steps; SURVEY.md 8d, tools/make_liquid_snapshot.py)"),
}
# --impl reference: the full workload; at ~1 s per step (2M atoms, 16
# threads) the timed steps are capped so a large --steps ends within minutes
REF_TIME_CAP_S = 240.0
DTYPES = {"double": "f64", "mixed": "f32 compute / f64 accumulate", "single": "f32"}
REF_OPTS = {"double": ("v1", "opt-d", 4), "mixed": ("v2", "opt-m", 8),
            "single": ("v2", "opt-s", 8)}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


LIQUID_SNAPSHOT = os.path.join(ROOT, "tests", "golden", "liquid512k.tsfsnap")


def _jitter(xyz, box, cfg):
    """The seeded uniform thermal-like jitter of the lattice configs, wrapped
    into the box (tests/systems.py baseline_cfg3/4 build the same arrays)."""
    jitter = CONFIGS[cfg][2]
    rng = np.random.default_rng(12345)
    return np.ascontiguousarray(np.mod(xyz + rng.uniform(-jitter, jitter, xyz.shape), box))


def _species_of(cfg, n, species):
    if CONFIGS[cfg][3] == "sic":
        text = open(os.path.join(ROOT, "tests", "golden", "SiC.tersoff")).read()
        return text, np.where(np.arange(n) % 8 < 4, 0, 1).astype(np.int32), [28.0855, 12.011]
    return None, np.ascontiguousarray(species, np.int32), [28.0855]


def make_system(cfg: str):
    """Synthetic input of the workload through the product's generators:
    diamond (or zincblende) lattice + seeded jitter, or, for the liquid, the
    committed TSFSNAP1 snapshot (tools/make_liquid_snapshot.py)."""
    import paper_1607_02904_b200 as tb
    if cfg.startswith("liquid"):
        s = tb.load_snapshot(LIQUID_SNAPSHOT)
        return (tb.builtin_silicon().serialize(), s.positions, s.species, s.box.lengths,
                s.box.periodic, list(s.species_masses))
    cells, a0 = CONFIGS[cfg][0], CONFIGS[cfg][1]
    s = tb.make_diamond_lattice(*cells, a0)
    xyz = _jitter(s.positions, s.box.lengths, cfg)
    text, species, masses = _species_of(cfg, s.natoms, s.species)
    return (text or tb.builtin_silicon().serialize(), xyz, species, s.box.lengths,
            s.box.periodic, masses)


def make_system_reference(cfg: str, R):
    """The same arrays without loading the product (the reference arm): the
    reference's own make_diamond_lattice (engine.cpp:28-58, via oracle/_ref)
    + the same numpy jitter, or the snapshot through the numpy reader."""
    from oracle.oracle import SI_TEXT
    if cfg.startswith("liquid"):
        from oracle import snapshot as osnap
        d = osnap.read(LIQUID_SNAPSHOT)
        return SI_TEXT, d["positions"], d["species"], d["box"], d["periodic"], list(d["masses"])
    cells, a0 = CONFIGS[cfg][0], CONFIGS[cfg][1]
    h = R.diamond_lattice(*cells, a0)
    xyz, _, species, box, per = R.system_arrays(h)
    R.free_system(h)
    xyz = _jitter(xyz, box, cfg)
    text, species, masses = _species_of(cfg, len(xyz), species)
    return text or SI_TEXT, xyz, species, box, per, masses


def algorithmic_work(xyz, species, box, offsets, nbrs, rows, ns):
    """P pairs inside their (si,sj,sj) cutoff and T triplets inside (si,sj,sk),
    on the short list, as the reference counts them:
    ALGO_FLOP = 75 P + 143 T, ALGO_TRANSC = 8 P + 4 T."""
    cnt = np.diff(offsets)
    i = np.repeat(np.arange(len(cnt)), cnt)
    d = xyz[nbrs] - xyz[i]
    d -= box * np.floor(d / box + 0.5)
    r2 = np.einsum("ij,ij->i", d, d)
    si, sj = species[i], species[nbrs]
    cutsq = rows[:, 15]
    pair_ok = r2 <= cutsq[(si * ns + sj) * ns + sj]
    P = int(pair_ok.sum())
    if ns == 1 and pair_ok.all():
        T = int(np.sum(cnt * (cnt - 1)))
    else:
        T = 0
        starts = offsets[:-1]
        for slot_j in range(int(cnt.max(initial=0))):
            has_j = cnt > slot_j
            ej = starts[has_j] + slot_j
            for slot_k in range(int(cnt.max(initial=0))):
                if slot_k == slot_j:
                    continue
                m = has_j & (cnt > slot_k)
                ej2 = starts[m] + slot_j
                ek = starts[m] + slot_k
                okj = pair_ok[ej2]
                row = (si[ej2] * ns + sj[ej2]) * ns + sj[ek]
                T += int(np.sum(okj & (r2[ek] <= cutsq[row])))
            del ej
    return P, T


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region: the
    sampler runs from before the warm-up; only samples stamped inside the
    timed window [t_lo, t_hi] (host wall clock) are kept (the nearest later
    one if the window is shorter than the 50 ms sampling period)."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), "--query-gpu=" + self.FIELDS,
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    @staticmethod
    def _stamp(text: str):
        import datetime
        try:
            return datetime.datetime.strptime(text.strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except ValueError:
            return None

    def stop(self, t_lo: float, t_hi: float):
        if self.p is None:
            return None
        time.sleep(0.12)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 8:
                rows.append((self._stamp(parts[0]), parts[1:]))
        os.unlink(self.f.name)
        inside = [r for ts, r in rows if ts is not None and t_lo <= ts <= t_hi]
        if not inside:
            later = [r for ts, r in rows if ts is not None and ts >= t_lo]
            inside = later[:1] or [r for _, r in rows][-1:]
        if not inside:
            return None
        sm = [float(r[0]) for r in inside if r[0].replace(".", "").isdigit()]
        reasons = set()
        for r in inside:
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                "sw_power_cap"), r[3:]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(inside[0][1]) if inside[0][1].replace(".", "").isdigit()
                else None,
                "samples": len(inside), "window_s": round(t_hi - t_lo, 3),
                "reasons": sorted(reasons)}


def load_peak(precision: str):
    path = os.path.join(ROOT, "profiles", "fp_peaks_b200.json")
    if os.path.exists(path):
        pk = json.load(open(path))
        key = "fp64_tflops" if precision == "double" else "fp32_tflops"
        return pk[key], f"measured ({os.path.relpath(path, ROOT)}: {key})"
    return (37.2 if precision == "double" else 74.4), "derived (148 SM x 1.965 GHz x FMA lanes)"


def load_ncu(cfg: str, precision: str, det: bool):
    """The main force kernel's ncu record for this workload (tools/ncu_traffic.sh
    -> profiles/ncu_traffic.json): DRAM read + write bytes per launch, and the
    pipe utilisation (fraction of peak sustained, time-weighted) — the north
    star's issue-rate view of the same kernel."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None, None
    tab = json.load(open(path))
    ent = tab.get(f"{cfg}/{precision}/{'det' if det else 'atomic'}") or {}
    force = ent.get("force")
    if not force:
        return None, None
    pipes = force.get("pipes_frac_of_peak")
    issue = None
    if pipes:
        issue = {"source": "ncu, profiles/ncu_traffic.json (tools/ncu_traffic.sh)", **pipes}
    return force["traffic_bytes"], issue


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref = unmodified /root/reference sources), all host threads."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle.oracle import Reference, reference_available
    if not reference_available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libtmdref.so not built (run __graft_entry__.build())"}))
        return
    R = Reference()
    text, xyz, species, box, per, masses = make_system_reference(args.config, R)
    n = len(xyz)
    ph = R.params(text)
    sh = R.system(xyz, species, masses, box, per)
    lh = R.neighbor_list(sh, R.lib.tmdref_params_r_cut_max(ph), 1.0)
    scheme, prec, width = REF_OPTS[args.precision]
    cores = os.cpu_count() or 1
    tw = time.perf_counter()
    for _ in range(args.warmup):
        R.evaluate(sh, lh, ph, n, scheme, prec, width, 16, cores, True, with_forces=False)
    t_step = (time.perf_counter() - tw) / args.warmup
    timed = min(args.steps, max(1, int(REF_TIME_CAP_S / max(t_step, 1e-9))))
    t0 = time.perf_counter()
    for _ in range(timed):
        R.evaluate(sh, lh, ph, n, scheme, prec, width, 16, cores, True, with_forces=False)
    t = time.perf_counter() - t0
    value = n * timed / t
    sample = (f"evaluate_forces({scheme}, width {width}, {prec}, workers={cores}) per step on "
              f"the full {n}-atom workload (same arrays as the GPU arm, built by the "
              f"reference's own generator); {timed} of {args.steps} steps timed"
              f"{' (time cap)' if timed < args.steps else ''}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / timed,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": DTYPES[args.precision], "data": "synthetic",
        "config": workload_config(args, n, world, None, None),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def workload_config(args, n, world, halo, parallelism):
    """The `config` object of both arms' lines: the workload, not the
    implementation (the driver compares the two arms' configs)."""
    jit = CONFIGS[args.config][2]
    return {
        "workload": CONFIGS[args.config][4] + (f", seeded uniform +-{jit:.2f} A jitter" if jit
                                               else "") +
                    ", skin 1.0 A; one filter + force/energy" +
                    ("" if getattr(args, "no_virial", False) else "/virial") + " evaluation per step",
        "n_atoms": n, "precision": args.precision,
        "deterministic": bool(args.deterministic),
        "parallelism": parallelism or (f"{world} x-slab domains" if world > 1 else "single GPU"),
        "l2": "inputs larger than L2 (positions + lists + forces > 126 MB at 2M atoms)"
              if n >= 1_000_000 else "inputs fit in L2",
    }


def cpu_baseline(text, xyz, species, box, per, masses):
    """compute_ref (paper Alg. 2, 1 thread) of the unmodified reference on the
    same system: one call (~10 s at 2M atoms)."""
    from oracle.oracle import Reference, reference_available
    if not reference_available():
        return None
    R = Reference()
    n = len(xyz)
    ph = R.params(text)
    sh = R.system(xyz, species, masses, box, per)
    lh = R.neighbor_list(sh, R.lib.tmdref_params_r_cut_max(ph), 1.0)
    t0 = time.perf_counter()
    R.compute_ref(sh, lh, ph, n, with_forces=False)
    t = time.perf_counter() - t0
    return {"value": n / t, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"compute_ref (1 thread) on the full {n}-atom system, one call, {t:.2f} s"}


def md_leg(tb, params, args, precision=None):
    """NVE MD steps through tsf_md_run on the workload's lattice at 1600 K
    (init_velocities seed 12345, dt 1 fs, skin 1 A, thermo every 100 steps):
    W warm-up steps, then max(100, K) timed steps including every rebuild."""
    import torch
    prec = precision or args.precision
    cells = CONFIGS[args.config][0]
    s = tb.make_diamond_lattice(*cells, CONFIGS[args.config][1])
    tb.init_velocities(s, 1600.0, 12345)
    ctx = tb.Context(params, 0)
    ctx.load(s)
    ctx.build_neighbor_list(params.r_cut_max, 1.0)
    ctx.md_set_state(s.velocities, s.species_masses)
    det = args.deterministic
    ctx.md_run(max(args.warmup, 20), 0.001, prec, det, 100)
    steps = max(100, args.steps)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.cuda.current_device())
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    thermo, rebuilds = ctx.md_run(steps, 0.001, prec, det, 100)
    e1.record(stream)
    e1.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    etot = thermo[:, 1] + thermo[:, 2]
    ctx.close()
    n = s.natoms
    return {"metric": "MD atom-steps/s", "value": n * steps / t, "unit": UNIT,
            "ms_per_step": 1e3 * t / steps, "steps": steps, "rebuilds": int(rebuilds),
            "ns_per_day": steps * 1e-6 / t * 86400.0, "precision": prec,
            "scatter": "deterministic gather" if det else "atomics",
            "workload": f"{CONFIGS[args.config][4]}, perfect lattice + init_velocities(1600 K, "
                        "seed 12345), dt 1 fs, skin 1 A, needs_rebuild every step, thermo "
                        "every 100 steps (tsf_md_run)",
            "rel_energy_drift": float(np.abs(etot - etot[0]).max() / abs(etot[0]))}


def md_leg_dd(tb, params, args, world, rank, local):
    """The MD leg across x slabs: tsf_dd_md_run (velocity Verlet, the
    needs_rebuild OR over ranks on the device, atom migration and ghost
    re-selection at rebuilds) on the workload's lattice at 1600 K; CUDA events
    on each rank's stream, max over ranks."""
    import torch
    from paper_1607_02904_b200 import parallel as PD
    cells = CONFIGS[args.config][0]
    s = tb.make_diamond_lattice(*cells, CONFIGS[args.config][1])
    tb.init_velocities(s, 1600.0, 12345)
    box = s.box.lengths
    halo = params.r_cut_max + 1.0
    if world > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{local}")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(PD.nccl_unique_id()), dtype=torch.uint8))
        torch.distributed.broadcast(uid, 0)
        transport, unique_id = "nccl", bytes(uid.cpu().numpy())
    else:
        transport, unique_id = PD.LocalGroup(1), None
    dd = PD.DomainDecomposition(params, local, box, s.box.periodic, params.r_cut_max, 1.0,
                                transport, rank, world=world, unique_id=unique_id,
                                masses=s.species_masses,
                                ghost_centers=box[0] / world > 4 * halo + 1e-9)
    gid = PD.partition(s.positions, box, world, rank)
    dd.setup(gid, s.positions[gid], s.species[gid], s.velocities[gid])
    det = args.deterministic
    dd.md_run(max(args.warmup, 20), 0.001, args.precision, det, 100)
    steps = max(100, args.steps)
    stream = torch.cuda.ExternalStream(dd.stream, device=local)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    thermo, rebuilds = dd.md_run(steps, 0.001, args.precision, det, 100)
    e1.record(stream)
    e1.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    if world > 1:
        tt = torch.tensor([t], device=f"cuda:{local}")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t = float(tt.item())
    migrated = dd.counts["migrated"]
    dd.close()
    etot = thermo[:, 1] + thermo[:, 2]
    n = s.natoms
    return {"metric": "MD atom-steps/s", "value": n * steps / t, "unit": UNIT,
            "ms_per_step": 1e3 * t / steps, "steps": steps, "rebuilds": int(rebuilds),
            "atoms_migrated_rank0": int(migrated),
            "ns_per_day": steps * 1e-6 / t * 86400.0, "precision": prec,
            "scatter": "deterministic gather" if det else "atomics",
            "workload": f"{CONFIGS[args.config][4]}, perfect lattice + init_velocities(1600 K, "
                        f"seed 12345), dt 1 fs, skin 1 A, {world} x slabs (tsf_dd_md_run: "
                        "ghost exchange every step, migration at rebuilds)",
            "rel_energy_drift": float(np.abs(etot - etot[0]).max() / abs(etot[0]))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--precision", default="double", choices=list(DTYPES))
    ap.add_argument("--config", default="si2m", choices=list(CONFIGS))
    ap.add_argument("--deterministic", action="store_true")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--no-md", action="store_true")
    # the reference's evaluate_forces returns energy and forces only; the
    # virial is this path's addition (A/B and forces-only workloads)
    ap.add_argument("--no-virial", action="store_true",
                    default=os.environ.get("TSF_BENCH_NO_VIRIAL") == "1")
    # the multi-GPU code path (GpuEngine + Decomposition) on one rank: a smoke
    # test of bench's N>1 branch where only one GPU is available
    ap.add_argument("--decompose", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import paper_1607_02904_b200 as tb
    from paper_1607_02904_b200 import _lib as L

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)

    text, xyz, species, box, per, masses = make_system(args.config)
    n = len(xyz)
    params = tb.parse_params(text)
    skin = 1.0
    use_dec = world > 1 or args.decompose
    if not use_dec:
        ctx = tb.Context(params, local)
        ctx.set_system(xyz, species, box, per)
        ctx.build_neighbor_list(params.r_cut_max, skin)
        soff, snb = ctx.export_neighbors("short")
        P, T = algorithmic_work(xyz, species, box, soff, snb, params.rows, params.species_count)
        stream = torch.cuda.ExternalStream(ctx.stream, device=local)

        def step():
            ctx.compute(args.precision, deterministic=args.deterministic, energy=False,
                        forces=False, virial=False, form_virial=not args.no_virial)
    else:
        # strong scaling: the same global system split into x slabs, one rank
        # per GPU, the C++ decomposition (csrc/tsf_dd.cu) over NCCL: ghost
        # positions forward (and, in classic mode, ghost forces back) every step
        from paper_1607_02904_b200 import parallel as PD
        halo = params.r_cut_max + skin
        ghost_centers = box[0] / world > 4 * halo + 1e-9
        if world > 1:
            uid = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{local}")
            if rank == 0:
                uid.copy_(torch.frombuffer(bytearray(PD.nccl_unique_id()), dtype=torch.uint8))
            torch.distributed.broadcast(uid, 0)
            transport, unique_id = "nccl", bytes(uid.cpu().numpy())
        else:       # --decompose: the same code path, one in-process rank
            transport, unique_id = PD.LocalGroup(1), None
        dec = PD.DomainDecomposition(params, local, box, per, params.r_cut_max, skin, transport,
                                     rank, world=world, unique_id=unique_id,
                                     ghost_centers=ghost_centers)
        gid = PD.partition(xyz, box, world, rank)
        dec.setup(gid, xyz[gid], species[gid])
        ctx = dec.ctx
        stream = torch.cuda.ExternalStream(dec.stream, device=local)
        # the whole job's algorithmic work (every centre once): the global short
        # list of a throw-away single context on this rank's GPU
        tmp = tb.Context(params, local)
        tmp.set_system(xyz, species, box, per)
        tmp.build_neighbor_list(params.r_cut_max, skin)
        soff, snb = tmp.export_neighbors("short")
        tmp.close()
        P, T = algorithmic_work(xyz, species, box, soff, snb, params.rows, params.species_count)
        del soff, snb

        def step():
            dec.evaluate(args.precision, args.deterministic)
    algo_flop = 75 * P + 143 * T
    if use_dec:
        parallelism = (f"{world} x-slab domains (C++ tsf_dd), ghost halo {halo:.1f} A, "
                       + ("ghost-centre mode: one forward exchange of positions per step, no "
                          "reverse force exchange" if ghost_centers else
                          "forward positions and reverse ghost forces each step")
                       + (" (NCCL P2P)" if world > 1 else " (one in-process rank)"))
    else:
        parallelism = "single GPU"

    clocks = ClockSampler(local)       # running before the warm-up
    # NVTX range around the steady state: ncu captures (tools/ncu_*.sh) use
    # --nvtx-include so input preparation (e.g. the liquid melt) is skipped
    torch.cuda.nvtx.range_push("bench_steps")
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    l0 = ctx.launches
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    t_lo = time.time()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize()
    t_hi = time.time()
    barrier()
    clk = clocks.stop(t_lo, t_hi)
    launches = ctx.launches - l0
    t = e0.elapsed_time(e1) / 1e3
    if world > 1:
        tt = torch.tensor([t], device=f"cuda:{local}")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t = float(tt.item())
    value = n * args.steps / t      # whole job: the global system, split over the ranks

    # per-stage timing pass (separate from the timed region)
    ctx.profile(True)
    for _ in range(args.steps):
        step()
    prof = ctx.profile_read(reset=True)
    ctx.profile(False)
    torch.cuda.nvtx.range_pop()
    calls = max(prof["calls"], 1)
    force_s = prof["force_ms"] / calls / 1e3
    # the roofline is taken over every force launch of the step — the main
    # launch plus the tier launches that take atoms over its lane-group width
    # (and the final fixed-order reduction, which cannot be timed apart): the
    # algorithmic work counts every atom, so the time must too
    stage_s = (prof["force_ms"] + prof["tail_ms"]) / calls / 1e3
    stage_total = prof["filter_ms"] + prof["setup_ms"] + prof["force_ms"] + prof["tail_ms"]
    peak, peak_src = load_peak(args.precision)
    # per GPU: the whole job's work over the ranks (x slabs of equal width)
    achieved = algo_flop / world / stage_s / 1e12
    ncu_traffic, ncu_issue = load_ncu(args.config, args.precision, args.deterministic)

    # e2e through the drop-in C-ABI call with host buffers
    e2e = None
    if not args.no_e2e and use_dec:
        # per rank: owned positions in from pinned host memory, decomposed
        # evaluation (ghost exchange both ways), owned forces back to the host
        own = dec.results()
        hx = torch.from_numpy(xyz[own["gid"]].copy()).pin_memory()
        hf = torch.empty((len(own["gid"]), 3), dtype=torch.float64).pin_memory()

        def call():
            dec.set_positions_ptr(hx.data_ptr())
            dec.evaluate(args.precision, args.deterministic)
            dec.forces_into(hf.data_ptr())
        for _ in range(args.warmup):
            call()
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            call()
        e1.record(stream)
        e1.synchronize()
        te = e0.elapsed_time(e1) / 1e3
        if world > 1:
            tt = torch.tensor([te], device=f"cuda:{local}")
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": n * args.steps / te, "unit": UNIT,
               "h2d_bytes_per_step": int(24 * n), "d2h_bytes_per_step": int(24 * n),
               "ms_per_step": 1e3 * te / args.steps,
               "call": "per rank: owned positions H2D (tsf_dd_set_positions, pinned), "
                       "tsf_dd_evaluate, owned forces D2H (tsf_dd_results); bytes summed over "
                       "ranks"}
    elif not args.no_e2e:
        lib = L.lib()
        hx = torch.from_numpy(xyz.copy()).pin_memory()
        hf = torch.empty((n, 3), dtype=torch.float64).pin_memory()
        sp_t = torch.from_numpy(np.ascontiguousarray(species, np.int32)).pin_memory()
        sp = sp_t.numpy()               # page-locked: species go straight to the device
        bx = np.ascontiguousarray(box, np.float64)
        pr = np.ascontiguousarray(per, np.uint8)
        energy = C.c_double()
        vir = np.zeros(6)
        pcode = {"double": 0, "mixed": 1, "single": 2}[args.precision]
        flags = L.TSF_DETERMINISTIC if args.deterministic else 0

        sp_ptr = [sp.ctypes.data_as(C.c_void_p)]

        def call():
            # species go with the first call only (NULL afterwards: the system's
            # species are resident, tsf_evaluate_forces)
            rc = lib.tsf_evaluate_forces(ctx._h, pcode, n, C.c_void_p(hx.data_ptr()),
                                         sp_ptr[0],
                                         bx.ctypes.data_as(C.c_void_p),
                                         pr.ctypes.data_as(C.c_void_p), 1.0, flags,
                                         C.byref(energy), C.c_void_p(hf.data_ptr()),
                                         vir.ctypes.data_as(C.c_void_p))
            if rc:
                raise RuntimeError(lib.tsf_last_error(ctx._h).decode())
            sp_ptr[0] = None
        for _ in range(args.warmup):
            call()
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            call()
        e1.record(stream)
        e1.synchronize()
        te = e0.elapsed_time(e1) / 1e3
        if world > 1:
            tt = torch.tensor([te], device=f"cuda:{local}")
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": n * world * args.steps / te, "unit": UNIT,
               # positions in (species resident after the first call);
               # forces, energy, virial out
               "h2d_bytes_per_step": int(hx.numel() * 8),
               "d2h_bytes_per_step": int(hf.numel() * 8 + 8 + 48),
               "ms_per_step": 1e3 * te / args.steps,
               "call": "tsf_evaluate_forces (include/tersoff_b200.h), pinned host buffers"}

    # the other precisions on the same resident system (device-resident only)
    variants = {}
    if world == 1 and not args.no_variants:
        for prec in [p for p in DTYPES if p != args.precision]:
            def vstep(prec=prec):
                ctx.compute(prec, deterministic=args.deterministic, energy=False, forces=False,
                            virial=False, form_virial=not args.no_virial)
            for _ in range(args.warmup):
                vstep()
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(args.steps):
                vstep()
            e1.record(stream)
            e1.synchronize()
            tv = e0.elapsed_time(e1) / 1e3
            ctx.profile(True)
            for _ in range(args.steps):
                vstep()
            pv = ctx.profile_read(reset=True)
            ctx.profile(False)
            kms = pv["force_ms"] / max(pv["calls"], 1)
            sms = (pv["force_ms"] + pv["tail_ms"]) / max(pv["calls"], 1)
            vpeak, _ = load_peak(prec)
            variants[prec] = {"value": n * args.steps / tv, "ms_per_step": 1e3 * tv / args.steps,
                              "dtype": DTYPES[prec], "kernel_ms": kms, "force_stage_ms": sms,
                              "roofline_frac": algo_flop / (sms * 1e-3) / 1e12 / vpeak}

    # MD-step leg (the paper's timing; Engine::run,
    # engine.cpp:174-199): GPU-resident velocity Verlet on cfg 4 at 1600 K —
    # kick, drift, the needs_rebuild test every step, list rebuilds, the
    # evaluation — timed with CUDA events on the context's stream
    md = None
    if not args.no_md and args.config in ("si2m", "si32k"):
        md = md_leg_dd(tb, params, args, world, rank, local) if use_dec else \
            md_leg(tb, params, args)
        if md and not use_dec and not args.no_variants:
            # the paper's other precisions on the same MD workload
            md["variants"] = {}
            for prec in [p for p in DTYPES if p != args.precision]:
                v = md_leg(tb, params, args, prec)
                md["variants"][prec] = {k: v[k] for k in ("value", "ms_per_step", "rebuilds",
                                                          "rel_energy_drift")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(text, xyz, species, box, per, masses)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": DTYPES[args.precision], "data": "synthetic",
            "config": workload_config(args, n, world, params.r_cut_max + skin, parallelism),
            "roofline": {
                "bound": "fp64" if args.precision == "double" else "fp32",
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": ncu_traffic,
                "algo_fraction": achieved / peak,
                "issue_rate": ncu_issue,
                "kernel": "k_force launches (main + tiers, with the final k_reduce)",
                "peak_source": peak_src,
                "algo_flop_per_launch": algo_flop, "pairs": P, "triplets": T,
                "algo_flop_formula": "75 P + 143 T (SURVEY.md 8d / Appendix A)",
                "kernel_ms": force_s * 1e3, "force_stage_ms": stage_s * 1e3,
                "stage_ms_per_step": {k: prof[k] / calls for k in
                                      ("filter_ms", "setup_ms", "force_ms", "tail_ms")},
                "force_share_of_step": prof["force_ms"] / stage_total if stage_total else None,
            },
            "cpu_baseline": cpu,
            "e2e": e2e,
            "md": md,
            "variants": variants,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(out))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
