"""The C++ domain decomposition (csrc/tsf_dd.cu, paper_1607_02904_b200.parallel)
on one B200: several ranks in one process over the LOCAL transport (one host
thread and one context per rank; messages are device-to-device copies ordered
by CUDA events — no kernel waits on another rank).

* a decomposed evaluation equals one context on the whole system (energy,
  virial, per-atom forces by global id), classic and ghost-centre modes,
  2 and 3 ranks, all precisions;
* the distributed NVE (tsf_dd_md_run: device-side rebuild decision, atom
  migration, ghost re-selection) follows the single-context tsf_md_run
  trajectory with the same rebuild schedule, with atoms crossing slab faces.
"""
import threading

import numpy as np
import pytest

import systems

pytestmark = pytest.mark.gpu


def run_ranks(world, fn):
    """fn(rank) in one thread per rank; re-raises the first failure."""
    out, errs = [None] * world, []

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if errs:
        raise errs[0]
    return out


def _lattice(tb, nx, ny, nz, jitter, seed):
    s = tb.make_diamond_lattice(nx, ny, nz)
    rng = np.random.default_rng(seed)
    xyz = np.mod(s.positions + rng.uniform(-jitter, jitter, s.positions.shape), s.box.lengths)
    return s, xyz


@pytest.mark.parametrize("world,ghost_centers", [(2, False), (3, False), (2, True), (3, True)])
def test_decomposed_evaluation_equals_one_context(tb, world, ghost_centers):
    from paper_1607_02904_b200.parallel import DomainDecomposition, LocalGroup, partition
    nx = 12 if ghost_centers else 8          # slabs wider than two ghost reaches
    s, xyz = _lattice(tb, nx, 3, 3, 0.12, 7)
    params = tb.builtin_silicon()
    ctx = tb.Context(params, 0)
    ctx.set_system(xyz, s.species, s.box.lengths, s.box.periodic)
    ctx.build_neighbor_list(params.r_cut_max, 1.0)
    ref = {p: ctx.compute(p, deterministic=True) for p in ("double", "mixed", "single")}
    ctx.close()
    group = LocalGroup(world)

    def rank_fn(r):
        gid = partition(xyz, s.box.lengths, world, r)
        dd = DomainDecomposition(params, 0, s.box.lengths, s.box.periodic, params.r_cut_max, 1.0,
                                 group, r, ghost_centers=ghost_centers)
        dd.setup(gid, xyz[gid], s.species[gid])
        res = {}
        for p in ("double", "mixed", "single"):
            for det in (True, False):
                dd.evaluate(p, det)
                res[(p, det)] = dd.results()
        counts = dd.counts
        dd.close()
        return res, counts

    outs = run_ranks(world, rank_fn)
    assert sum(c["owned"] for _, c in outs) == len(xyz)
    assert all(c["local"] > c["owned"] for _, c in outs)      # every rank holds ghosts
    for (p, det) in outs[0][0]:
        e_ref, f_ref, w_ref = ref[p]
        f = np.zeros_like(f_ref)
        for res, _ in outs:
            r = res[(p, det)]
            f[r["gid"]] = r["forces"]
        e = outs[0][0][(p, det)]["energy"]
        w = outs[0][0][(p, det)]["virial"]
        etol, ftol = (1e-12, 1e-10) if p == "double" else (1e-6, 1e-4 * max(1, np.abs(f_ref).max()))
        assert abs(e - e_ref) <= etol * abs(e_ref), (p, det, e, e_ref)
        assert np.abs(f - f_ref).max() <= ftol, (p, det)
        assert np.abs(w - w_ref).max() <= (1e-10 if p == "double" else 1e-5) * max(
            1.0, np.abs(w_ref).max())
        for res, _ in outs[1:]:                  # the global energy is the same on every rank
            assert res[(p, det)]["energy"] == e


@pytest.mark.parametrize("world,ghost_centers", [(1, False), (3, False), (3, True)])
def test_distributed_nve_follows_single_context(tb, world, ghost_centers):
    """60 steps at 3000 K: atoms migrate across the slab faces; the rebuild
    schedule is the single context's and positions agree to 1e-8 A."""
    from paper_1607_02904_b200.parallel import DomainDecomposition, LocalGroup, partition
    nx = 12 if ghost_centers else 8
    s = tb.make_diamond_lattice(nx, 3, 3)
    tb.init_velocities(s, 3000.0, 99)
    params = tb.builtin_silicon()
    steps = 60
    ctx = tb.Context(params, 0)
    ctx.load(s)
    ctx.build_neighbor_list(params.r_cut_max, 1.0)
    ctx.md_set_state(s.velocities, s.species_masses)
    thermo_ref, reb_ref = ctx.md_run(steps, 0.001, "double", True, 20)
    x_ref, v_ref = ctx.md_get_state()
    ctx.close()
    group = LocalGroup(world)

    def rank_fn(r):
        gid = partition(s.positions, s.box.lengths, world, r)
        dd = DomainDecomposition(params, 0, s.box.lengths, s.box.periodic, params.r_cut_max, 1.0,
                                 group, r, masses=s.species_masses, ghost_centers=ghost_centers)
        dd.setup(gid, s.positions[gid], s.species[gid], s.velocities[gid])
        thermo, reb = dd.md_run(steps, 0.001, "double", True, 20)
        res = dd.results(positions=True, velocities=True)
        counts = dd.counts
        dd.close()
        return thermo, reb, res, counts

    outs = run_ranks(world, rank_fn)
    thermo, reb = outs[0][0], outs[0][1]
    assert reb == reb_ref >= 1
    assert all(o[1] == reb for o in outs)
    if world > 1:
        assert sum(o[3]["migrated"] for o in outs) > 0
    x = np.zeros_like(x_ref)
    v = np.zeros_like(v_ref)
    for _, _, res, _ in outs:
        x[res["gid"]] = res["positions"]
        v[res["gid"]] = res["velocities"]
    d = x - x_ref
    d -= s.box.lengths * np.round(d / s.box.lengths)
    assert np.abs(d).max() < 1e-8
    assert np.abs(v - v_ref).max() < 1e-6
    np.testing.assert_allclose(thermo[:, 0], thermo_ref[:, 0])
    etot, etot_ref = thermo[:, 1] + thermo[:, 2], thermo_ref[:, 1] + thermo_ref[:, 2]
    assert np.abs(etot - etot_ref).max() <= 1e-9 * np.abs(etot_ref).max()


def test_decomposition_guards(tb):
    from paper_1607_02904_b200.parallel import DomainDecomposition, LocalGroup
    params = tb.builtin_silicon()
    s = tb.make_diamond_lattice(4, 3, 3)          # 21.7 A: two slabs of 10.9 < 2 x 4.2 ... ok
    with pytest.raises(tb.ConfigError, match="slabs"):
        DomainDecomposition(params, 0, s.box.lengths, s.box.periodic, params.r_cut_max, 1.0,
                            LocalGroup(3), 0)
    with pytest.raises(tb.ConfigError, match="periodic x"):
        DomainDecomposition(params, 0, s.box.lengths, np.array([0, 1, 1], np.uint8),
                            params.r_cut_max, 1.0, LocalGroup(2), 0)


def test_nccl_transport_single_rank(tb):
    """The NCCL transport (libnccl.so.2 resolved at run time): a one-rank
    communicator drives the same path — unique id, comm init, the device
    allreduce of energy/virial and of the rebuild flag in tsf_dd_md_run."""
    from paper_1607_02904_b200.parallel import DomainDecomposition, nccl_unique_id
    s = tb.make_diamond_lattice(4, 4, 4)
    tb.init_velocities(s, 1600.0, 5)
    params = tb.builtin_silicon()
    ctx = tb.Context(params, 0)
    ctx.load(s)
    ctx.build_neighbor_list(params.r_cut_max, 1.0)
    e_ref, f_ref, w_ref = ctx.compute("double", deterministic=True)
    ctx.md_set_state(s.velocities, s.species_masses)
    thermo_ref, reb_ref = ctx.md_run(40, 0.001, "double", True, 20)
    ctx.close()
    dd = DomainDecomposition(params, 0, s.box.lengths, s.box.periodic, params.r_cut_max, 1.0,
                             "nccl", 0, world=1, unique_id=nccl_unique_id(),
                             masses=s.species_masses)
    dd.setup(np.arange(s.natoms), s.positions, s.species, s.velocities)
    dd.evaluate("double", True)
    r = dd.results()
    assert abs(r["energy"] - e_ref) <= 1e-12 * abs(e_ref)
    f = np.zeros_like(f_ref)
    f[r["gid"]] = r["forces"]
    assert np.abs(f - f_ref).max() <= 1e-10
    thermo, reb = dd.md_run(40, 0.001, "double", True, 20)
    assert reb == reb_ref
    np.testing.assert_allclose(thermo[:, 1:], thermo_ref[:, 1:], rtol=1e-9)
    dd.close()
