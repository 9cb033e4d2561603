"""Multi-rank decomposition logic on CPU: world_size 2 and 3 over gloo.

The product's `paper_1607_02904_b200.parallel.Decomposition` (slab ownership,
ghost selection, forward position / reverse force exchange, result gather)
runs unchanged; the engine is the CPU oracle restricted to owned centres
(`n_center`).  The decomposed energy, forces and virial must equal the
single-process oracle: the x-slab split in the global frame is exact up to
summation order.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import systems


class OracleEngine:
    """Engine interface of parallel.GpuEngine, backed by the CPU oracle."""

    def __init__(self, oracle, params_text):
        from oracle.oracle import parse_param_text
        self.oracle = oracle
        self.op = parse_param_text(params_text)
        self.device = torch.device("cpu")

    def load(self, xyz, species, box, periodic, n_owned, n_centers=None, n_interior=-1):
        self.xyz = np.array(xyz, np.float64)
        self.species = np.asarray(species, np.int32)
        self.box, self.per, self.n_owned = np.asarray(box), np.asarray(periodic), n_owned
        self.n_centers = n_owned if n_centers is None else n_centers

    def build(self, cutoff, skin):
        self.off, self.nb = self.oracle.build_neighbor_list(self.xyz, self.box, self.per, cutoff,
                                                            skin)
        self.skin, self.ref = skin, self.xyz.copy()

    # velocity Verlet pieces with tsf_md_kick's arithmetic (k_kick, tsf_md.cu):
    # separate roundings, wrap_1d (box.hpp:41-46), needs_rebuild's exact
    # minimum image (neighbor.cpp:134-141); owned atoms only
    MVV2E = 1.0364269e-4

    def md_set_state(self, vel, masses):
        self.vel = np.array(vel, np.float64).reshape(-1, 3)
        self.masses = np.asarray(masses, np.float64)

    def md_get_state(self):
        return self.xyz.copy(), self.vel.copy()

    def kick(self, dt, drift=True, kicks=1):
        o = slice(0, self.n_owned)
        m = self.masses[self.species[o]][:, None]
        k = (0.5 * dt) / (m * self.MVV2E)
        f = self.f[o]
        v = self.vel[o]
        for _ in range(kicks):
            v = v + f * k
        self.vel[o] = v
        if not drift:
            return False
        x = self.xyz[o] + v * dt
        L = self.box
        for ax in range(3):
            if self.per[ax]:
                c = x[:, ax] - L[ax] * np.floor(x[:, ax] / L[ax])
                c = np.where(c < 0.0, c + L[ax], c)
                x[:, ax] = np.where(c >= L[ax], c - L[ax], c)
        self.xyz[o] = x
        d = x - self.ref[o]
        for ax in range(3):
            if self.per[ax]:
                far = np.abs(d[:, ax]) > 0.25 * L[ax]
                d[far, ax] = d[far, ax] - L[ax] * np.floor(d[far, ax] / L[ax] + 0.5)
        r2 = d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1] + d[:, 2] * d[:, 2]
        return bool(np.any(r2 > 0.25 * self.skin * self.skin))

    def kinetic(self):
        o = slice(0, self.n_owned)
        m = self.masses[self.species[o]]
        v = self.vel[o]
        return float(np.sum(0.5 * m * (v * v).sum(axis=1) * self.MVV2E))

    def gather_positions(self, idx, out=None):
        t = torch.from_numpy(self.xyz[idx.numpy()].copy())
        return out.copy_(t) if out is not None else t

    def scatter_positions(self, lo, t):
        self.xyz[lo:lo + len(t)] = t.numpy()

    def compute(self, precision="double", deterministic=False):
        # forces from every centre (ghost centres included), energy and
        # virial from the owned centres only — tsf_set_centers' semantics
        r = self.oracle.compute_ref(self.op, self.xyz, self.species, self.box, self.per, self.off,
                                    self.nb, n_center=self.n_centers)
        self.f = r["forces"].copy()
        if self.n_centers != self.n_owned:
            r = self.oracle.compute_ref(self.op, self.xyz, self.species, self.box, self.per,
                                        self.off, self.nb, n_center=self.n_owned)
        self.ev = np.concatenate([[r["energy"]], r["virial"]])

    def compute_phase(self, phase, precision="double", deterministic=False):
        if phase == 1:             # the oracle has no split: the whole step in phase 1
            self.compute(precision, deterministic)

    def ghost_forces(self, lo, m, out=None):
        t = torch.from_numpy(self.f[lo:lo + m].copy())
        return out.copy_(t) if out is not None else t

    def add_forces(self, idx, t):
        self.f[idx.numpy()] += t.numpy()

    def results(self):
        return torch.from_numpy(self.ev.copy()), torch.from_numpy(self.f.copy())


def _case(cells):
    import paper_1607_02904_b200 as tb
    return systems.perturbed(tb, cells, 0.15, 17, skin=0.5)


def _worker(rank, world, port, cells, shift, out_path, ghost_centers=False, overlap=False,
            rev_split=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        from dd_model import Decomposition, partition
        c = _case(cells)
        halo = 3.2 + c.skin
        gid = partition(c.xyz, c.box, world, rank, halo)
        dec = Decomposition(OracleEngine(Oracle(), c.params_text), c.box, c.periodic, halo,
                            ghost_centers=ghost_centers, overlap=overlap)
        dec.setup(gid, c.xyz[gid], c.species[gid], 3.2, c.skin)
        if rev_split:
            # the reverse add's fallback (an atom sent both ways): one add per side
            dec._rev_fused = False
        if shift is not None:
            # move owned atoms a little: the forward exchange must refresh ghosts
            moved = np.mod(c.xyz + shift, c.box)
            dec.engine.scatter_positions(0, torch.from_numpy(moved[dec.gid]))
        dec.evaluate()
        e, f, w = dec.gather_results(len(c.xyz))
        if rank == 0:
            np.savez(out_path, e=e, f=f, w=w, n_owned=dec.n_owned, n_ghost=len(dec.ghost_gid))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world,cells,shifted,ghost_centers,overlap", [
    (2, 4, False, False, False), (2, 4, True, False, False), (3, 5, False, False, False),
    (2, 6, True, True, False), (3, 9, False, True, False),
    (2, 5, True, False, True), (2, 6, True, True, True)])
def test_decomposed_equals_single_process(oracle, tmp_path, world, cells, shifted, ghost_centers,
                                          overlap, rev_split=False):
    """Classic mode (reverse force exchange) and ghost-centre mode (layer-1
    ghosts act as centres, no reverse exchange) both give the single-process
    energy, forces and virial."""
    from oracle.oracle import parse_param_text
    c = _case(cells)
    shift = np.array([0.03, -0.02, 0.01]) if shifted else None
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, _free_port(), cells, shift, out, ghost_centers, overlap,
                            rev_split), nprocs=world, join=True)
    res = np.load(out)
    op = parse_param_text(c.params_text)
    off, nb = oracle.build_neighbor_list(c.xyz, c.box, c.periodic, op.r_cut_max, c.skin)
    xyz = np.mod(c.xyz + shift, c.box) if shifted else c.xyz
    ref = oracle.compute_ref(op, xyz, c.species, c.box, c.periodic, off, nb)
    assert res["n_ghost"] > 0
    assert abs(res["e"] - ref["energy"]) <= 1e-12 * abs(ref["energy"])
    assert np.abs(res["f"] - ref["forces"]).max() <= 1e-10
    assert np.abs(res["w"] - ref["virial"]).max() <= 1e-10 * np.abs(ref["virial"]).max()


def test_reverse_exchange_split_add(oracle, tmp_path):
    """Classic mode with the reverse add issued per side (the fallback when an
    atom is sent both ways) equals the fused single add."""
    test_decomposed_equals_single_process(oracle, tmp_path, 3, 5, True, False, False, True)


def test_slab_geometry_guards():
    from dd_model import Slab
    s = Slab(rank=1, world=4, length=40.0, halo=3.0)
    assert (s.lo, s.hi) == (10.0, 20.0)
    x = np.array([10.0, 12.9, 13.1, 17.0, 19.99, 39.9])
    assert s.near_left(x).tolist() == [True, True, False, False, False, False]
    assert s.near_right(x).tolist() == [False, False, False, True, True, False]
    assert Slab(0, 4, 40.0, 3.0).owner(np.array([-0.5, 0.0, 9.99, 10.0, 39.99, 40.0])).tolist() == \
        [3, 0, 0, 1, 3, 0]


def _nve_worker(rank, world, port, steps, out_path, nx=5, ghost_centers=False, overlap=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1607_02904_b200 as tb
        from oracle.oracle import Oracle
        from dd_model import Decomposition, SlabNVE, partition
        c = _nve_case(nx)
        s = tb.make_diamond_lattice(nx, 2, 2)
        tb.init_velocities(s, 3000.0, 7)
        halo = 3.2 + c.skin
        gid = partition(c.xyz, c.box, world, rank, halo)
        dec = Decomposition(OracleEngine(Oracle(), c.params_text), c.box, c.periodic, halo,
                            ghost_centers=ghost_centers, overlap=overlap)
        dec.setup(gid, c.xyz[gid], c.species[gid], 3.2, c.skin)
        nve = SlabNVE(dec, [28.0855], 3.2, c.skin)
        nve.set_velocities(s.velocities[dec.gid])   # dec.gid: this rank's storage order
        samples = nve.run(steps, dt=0.001, thermo_every=10)
        g, x, v = nve.owned_state()
        parts = [None] * world
        dist.all_gather_object(parts, (g, x, v))
        migrated = [None] * world
        dist.all_gather_object(migrated, dec.migrated)
        if rank == 0:
            n = len(c.xyz)
            X, V = np.zeros((n, 3)), np.zeros((n, 3))
            for g, x, v in parts:
                X[g], V[g] = x, v
            np.savez(out_path, x=X, v=V, samples=np.array(samples), rebuilds=nve.rebuilds,
                     migrated=sum(migrated))
    finally:
        dist.destroy_process_group()


def _nve_case(nx=5):
    import paper_1607_02904_b200 as tb
    s = tb.make_diamond_lattice(nx, 2, 2)
    return systems.Case(f"nve_{nx}x2x2", s.positions, s.species, s.box.lengths, s.box.periodic,
                        0.5, systems.si_text(tb))


@pytest.mark.parametrize("world,nx,ghost_centers,overlap", [
    (2, 5, False, False), (3, 5, False, False), (2, 6, True, False), (2, 6, True, True)])
def test_slab_nve_matches_single_domain(tmp_path, world, nx, ghost_centers, overlap):
    """SlabNVE (kick/drift of owned atoms, ghost exchange, rebuild vote,
    migration at rebuilds) on a hot 160-atom lattice over 2 and 3 gloo ranks
    follows the single-domain run of the same driver: atoms cross slab faces
    and migrate, the rebuild schedule is identical, and positions, velocities
    and energies agree to summation-order rounding."""
    steps = 60
    res = {}
    for w in (1, world):
        out = str(tmp_path / f"nve{w}.npz")
        mp.spawn(_nve_worker, args=(w, _free_port(), steps, out, nx, ghost_centers, overlap),
                 nprocs=w, join=True)
        res[w] = np.load(out)
    a, b = res[1], res[world]
    assert int(a["rebuilds"]) >= 2 and int(b["rebuilds"]) == int(a["rebuilds"])
    assert int(b["migrated"]) > 0                  # atoms did change owners
    box = _nve_case(nx).box
    dx = b["x"] - a["x"]
    dx -= box * np.round(dx / box)
    assert np.abs(dx).max() < 1e-9
    assert np.abs(b["v"] - a["v"]).max() < 1e-7
    np.testing.assert_allclose(b["samples"], a["samples"], rtol=1e-10, atol=1e-9)
    # energy is conserved by the distributed integrator
    e = b["samples"][:, 1] + b["samples"][:, 2]
    assert np.abs(e - e[0]).max() < 1e-3 * abs(e[0])
