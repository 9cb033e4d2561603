"""TEST INFRASTRUCTURE ONLY — the x-slab decomposition algorithm as a Python
model over torch.distributed (round 1's host-side implementation).  The
product is the C++ decomposition behind the C-ABI (csrc/tsf_dd.cu,
`tsf_dd_*`, wrapped by paper_1607_02904_b200/parallel.py); this model stays as
the CPU reference of the same algorithm: tests/test_parallel.py runs it with
gloo and the CPU oracle as the engine (world size 2 and 3), and
tests/test_gpu_dd.py checks the C++ path against single-domain results.

x-slab spatial domain decomposition of the Tersoff path.

The reference has no distribution at all; this is the B200-native
multi-GPU form of the paper's LAMMPS runs (Fig. 9): one process per
GPU, torch.distributed (NCCL over NVLink) for the two exchange steps a
many-body force evaluation needs:

  forward  ghost positions: atoms within r_cut_max + skin of a slab face are
           copied to the neighbour slab every step;
  reverse  ghost forces: the (i, j, k) terms of an owned centre put forces on
           ghosts; those go back to the owners and are added (Newton's third
           law across the face).

Everything stays in the GLOBAL frame and the global periodic box: ghosts keep
their owners' wrapped coordinates, so every displacement is the reference's
minimum image bit for bit, and a rank's neighbour lists are exactly the
global lists restricted to its owned atoms.  Only owned atoms act as centres
(`tsf_set_owned`), so each (i, j, k) term is computed once, by the owner of i.

Engines: `GpuEngine` (libtersoff_b200.so, device tensors, NCCL) is the
product.  The same `Decomposition` logic is exercised on CPU with gloo and an
oracle engine in tests/test_parallel.py.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from paper_1607_02904_b200 import _lib as L
from paper_1607_02904_b200.api import Context, ConfigError

TAG_FWD_LEFT, TAG_FWD_RIGHT, TAG_REV_RIGHT, TAG_REV_LEFT = 11, 12, 13, 14
TAG_FWD_LEFT2, TAG_FWD_RIGHT2 = 15, 16      # ghost-centre mode: layer-2 ghosts


@dataclass
class Slab:
    rank: int
    world: int
    length: float          # box length along x
    halo: float            # r_cut_max + skin

    @property
    def width(self) -> float:
        return self.length / self.world

    @property
    def lo(self) -> float:
        return self.rank * self.width

    @property
    def hi(self) -> float:
        return (self.rank + 1) * self.width

    def owner(self, x: np.ndarray) -> np.ndarray:
        """Owning rank of wrapped x coordinates."""
        xw = np.mod(x, self.length)
        return np.minimum((xw / self.width).astype(np.int64), self.world - 1)

    def near_left(self, x: np.ndarray) -> np.ndarray:
        """Owned atoms the left neighbour needs: within halo of the left face."""
        return np.mod(x - self.lo, self.length) <= self.halo

    def near_right(self, x: np.ndarray) -> np.ndarray:
        return np.mod(self.hi - x, self.length) <= self.halo


class GpuEngine:
    """Device-resident engine: one context per rank on the caller's stream."""

    def __init__(self, params, device: int):
        self.ctx = Context(params, device)
        self.device = torch.device("cuda", device)
        self._lib = L.lib()
        # One stream orders torch's work (allocations, NCCL P2P, .item()) and
        # the C-ABI's kernels.  torch's legacy default stream has the handle 0,
        # which tsf_set_stream reads as "the context's own stream" — a
        # non-blocking stream that does NOT order against it — so the engine
        # then makes a dedicated stream torch's current one.
        stream = torch.cuda.current_stream(device)
        if stream.cuda_stream == 0:
            stream = torch.cuda.Stream(device)
            torch.cuda.set_stream(stream)
        self.stream = stream
        self.ctx._ok(self._lib.tsf_set_stream(self.ctx._h, C.c_void_p(stream.cuda_stream)))

    def _p(self, t: torch.Tensor):
        return C.c_void_p(t.data_ptr())

    def load(self, xyz: np.ndarray, species: np.ndarray, box, periodic, n_owned: int,
             n_centers: int = None, n_interior: int = -1):
        self.ctx.set_system(xyz, species, box, periodic)
        n_centers = n_owned if n_centers is None else n_centers
        self.ctx._ok(self._lib.tsf_set_centers(self.ctx._h, n_owned, n_centers))
        self.ctx.set_interior(n_interior)

    def compute_phase(self, phase: int, precision: str = "double", deterministic: bool = False):
        self.ctx.compute_phase(phase, precision, deterministic)

    def build(self, cutoff: float, skin: float):
        self.ctx.build_neighbor_list(cutoff, skin)

    def gather_positions(self, idx: torch.Tensor, out: torch.Tensor = None) -> torch.Tensor:
        if out is None:
            out = torch.empty((len(idx), 3), dtype=torch.float64, device=self.device)
        if len(idx):
            self.ctx._ok(self._lib.tsf_gather_positions(self.ctx._h, self._p(idx), len(idx),
                                                        self._p(out)))
        return out

    def scatter_positions(self, lo: int, xyz: torch.Tensor):
        if len(xyz):
            self.ctx._ok(self._lib.tsf_scatter_positions(self.ctx._h, lo, len(xyz), self._p(xyz)))

    def compute(self, precision: str = "double", deterministic: bool = False):
        self.ctx.compute(precision, deterministic=deterministic, energy=False, forces=False,
                         virial=False)

    def ghost_forces(self, lo: int, m: int, out: torch.Tensor = None) -> torch.Tensor:
        if out is None:
            out = torch.empty((m, 3), dtype=torch.float64, device=self.device)
        if m:
            self.ctx._ok(self._lib.tsf_gather_forces(self.ctx._h, lo, m, self._p(out)))
        return out

    def add_forces(self, idx: torch.Tensor, f: torch.Tensor):
        if len(idx):
            self.ctx._ok(self._lib.tsf_add_forces(self.ctx._h, self._p(idx), len(idx), self._p(f)))

    def results(self):
        ev = torch.empty(7, dtype=torch.float64, device=self.device)
        f = torch.empty((self.ctx.n, 3), dtype=torch.float64, device=self.device)
        self.ctx._ok(self._lib.tsf_results_device(self.ctx._h, self._p(ev), self._p(f)))
        return ev, f

    # ---- velocity Verlet pieces (SlabNVE) ----
    def md_set_state(self, velocities: np.ndarray, masses):
        self.ctx.md_set_state(velocities, masses)

    def md_get_state(self):
        """Local positions and velocities, user order (owned atoms first)."""
        return self.ctx.md_get_state()

    def kick(self, dt: float, drift: bool = True, kicks: int = 1) -> bool:
        return self.ctx.md_kick(dt, drift, kicks, check=drift)

    def kinetic(self) -> float:
        return self.ctx.md_kinetic()


class Decomposition:
    """One rank's view: owned atoms (global ids), ghost blocks, send lists.

    ghost_centers=False (classic): ghosts within halo = r_cut_max + skin of a
    face; only owned atoms are centres; the forces their terms put on ghosts
    go back to the owners (reverse exchange).
    ghost_centers=True: ghosts within 2 halo; the first layer (within halo)
    also acts as centres (tsf_set_centers), so every term that puts force on
    an owned atom is evaluated locally — one exchange per step instead of two,
    for ~2 halo / slab of redundant compute; energy and virial stay with the
    owners.  Local layout: [owned | layer-1 from left | layer-1 from right |
    layer-2 from left | layer-2 from right]."""

    def __init__(self, engine, box, periodic, halo: float, group=None,
                 ghost_centers: bool = False, overlap: bool = False):
        self.engine = engine
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.box = np.asarray(box, np.float64)
        self.periodic = np.asarray(periodic, np.uint8)
        self.ghost_centers = bool(ghost_centers)
        # overlap: the forward exchange is in flight while the interior
        # centres (no ghost within halo: slots [0, n_interior)) are computed
        self.overlap = bool(overlap)
        reach = 2.0 * halo if self.ghost_centers else halo      # ghost selection distance
        if self.world > 1:
            if not self.periodic[0]:
                raise ConfigError("slab decomposition needs a periodic x axis")
            if self.box[0] / self.world < 2.0 * reach:
                raise ConfigError(f"{self.world} slabs of {self.box[0] / self.world:.3f} A are "
                                  f"thinner than 2 x {reach:.3f} A")
        self.slab = Slab(self.rank, self.world, float(self.box[0]), float(halo))
        self.slab_sel = Slab(self.rank, self.world, float(self.box[0]), float(reach))
        self.left = (self.rank - 1) % self.world
        self.right = (self.rank + 1) % self.world
        self.migrated = 0      # atoms received from neighbours by migrate()

    # ---- exchange helpers ------------------------------------------------
    def _device(self):
        return getattr(self.engine, "device", torch.device("cpu"))

    def _exchange_start(self, sends, recvs):
        """sends: [(tensor, dst, tag)], recvs: [(tensor, src, tag)] in a fixed
        order on every rank (NCCL matches per pair in issue order, gloo by tag).
        Returns the pending requests (NCCL: enqueued behind the current stream)."""
        ops = [dist.P2POp(dist.isend, t, d, self.group, tag) for t, d, tag in sends if t.numel()]
        ops += [dist.P2POp(dist.irecv, t, s, self.group, tag) for t, s, tag in recvs if t.numel()]
        return dist.batch_isend_irecv(ops) if ops else []

    def _exchange_finish(self, reqs):
        for req in reqs:
            req.wait()

    def _exchange(self, sends, recvs):
        self._exchange_finish(self._exchange_start(sends, recvs))

    def _swap_counts(self, n_left, n_right):
        """Send count(s) left and right, return what the left and right
        neighbours sent (ints, or tuples when tuples were sent)."""
        dev = self._device()
        k = len(n_left) if isinstance(n_left, (tuple, list)) else 1
        send_l = torch.tensor(n_left if k > 1 else [n_left], dtype=torch.int64, device=dev)
        send_r = torch.tensor(n_right if k > 1 else [n_right], dtype=torch.int64, device=dev)
        from_r = torch.zeros(k, dtype=torch.int64, device=dev)
        from_l = torch.zeros(k, dtype=torch.int64, device=dev)
        self._exchange([(send_l, self.left, TAG_FWD_LEFT), (send_r, self.right, TAG_FWD_RIGHT)],
                       [(from_r, self.right, TAG_FWD_LEFT), (from_l, self.left, TAG_FWD_RIGHT)])
        if k > 1:
            return tuple(int(x) for x in from_l.tolist()), tuple(int(x) for x in from_r.tolist())
        return int(from_l.item()), int(from_r.item())

    # ---- setup at a (re)build -------------------------------------------
    def setup(self, gid: np.ndarray, xyz: np.ndarray, species: np.ndarray, cutoff: float,
              skin: float):
        """gid/xyz/species: this rank's owned atoms (global ids, global frame).
        Owned atoms are stored by (boundary, gid): interior ones — farther
        than one halo from both faces, so no ghost in their lists — first.
        self.last_order is the permutation applied to the inputs."""
        if self.world > 1 and self.overlap:
            boundary = self.slab.near_left(xyz[:, 0]) | self.slab.near_right(xyz[:, 0])
            order = np.lexsort((gid, boundary))
            self.n_interior = int((~boundary).sum())
        else:
            order = np.argsort(gid, kind="stable")
            self.n_interior = -1
        self.last_order = order
        self.gid = np.ascontiguousarray(gid[order], np.int64)
        xyz = np.ascontiguousarray(xyz[order], np.float64)
        species = np.ascontiguousarray(species[order], np.int32)
        self.n_owned = len(self.gid)
        dev = self._device()
        self.n_gl1 = self.n_gr1 = 0              # layer-1 ghosts (ghost_centers)
        self.nl1 = self.nr1 = 0                  # layer-1 atoms among those sent
        if self.world == 1:
            self.send_left = self.send_right = np.zeros(0, np.int64)
            self.n_gl = self.n_gr = 0
            gxyz = np.zeros((0, 3))
            gsp = np.zeros(0, np.int32)
            self.ghost_gid = np.zeros(0, np.int64)
        else:
            def select(near_sel, near_l1):
                idx = np.nonzero(near_sel(xyz[:, 0]))[0]
                l1 = near_l1(xyz[idx, 0])
                return idx[np.argsort(~l1, kind="stable")], int(l1.sum())   # layer 1 first
            self.send_left, self.nl1 = select(self.slab_sel.near_left, self.slab.near_left)
            self.send_right, self.nr1 = select(self.slab_sel.near_right, self.slab.near_right)
            (self.n_gl, self.n_gl1), (self.n_gr, self.n_gr1) = self._swap_counts(
                (len(self.send_left), self.nl1), (len(self.send_right), self.nr1))
            if not self.ghost_centers:
                self.n_gl1 = self.n_gr1 = 0
            # ghost payload: global id, species, xyz (as float64 rows)
            def pack(idx):
                return torch.from_numpy(np.column_stack([self.gid[idx].astype(np.float64),
                                                         species[idx].astype(np.float64),
                                                         xyz[idx]])).to(dev)
            from_l = torch.zeros((self.n_gl, 5), dtype=torch.float64, device=dev)
            from_r = torch.zeros((self.n_gr, 5), dtype=torch.float64, device=dev)
            self._exchange([(pack(self.send_left), self.left, TAG_FWD_LEFT),
                            (pack(self.send_right), self.right, TAG_FWD_RIGHT)],
                           [(from_r, self.right, TAG_FWD_LEFT), (from_l, self.left, TAG_FWD_RIGHT)])
            ghosts = torch.cat(self._layout(from_l, from_r)).cpu().numpy()
            self.ghost_gid = ghosts[:, 0].astype(np.int64)
            gsp = ghosts[:, 1].astype(np.int32)
            gxyz = np.ascontiguousarray(ghosts[:, 2:5])
        self.local_xyz = np.concatenate([xyz, gxyz])
        self.local_species = np.concatenate([species, gsp]).astype(np.int32)
        self.n_centers = self.n_owned + self.n_gl1 + self.n_gr1
        self.engine.load(self.local_xyz, self.local_species, self.box, self.periodic,
                         self.n_owned, self.n_centers, self.n_interior)
        self.engine.build(cutoff, skin)
        self.t_send_left = torch.from_numpy(self.send_left.astype(np.int32)).to(dev)
        self.t_send_right = torch.from_numpy(self.send_right.astype(np.int32)).to(dev)
        # per-step buffers and exchange lists, allocated once per setup (the
        # step's host work is then a handful of launches and one P2P batch
        # per direction — it must stay below the GPU time of a step at 8 GPUs)
        def buf(m):
            return torch.empty((m, 3), dtype=torch.float64, device=dev)
        nl, nr = len(self.send_left), len(self.send_right)
        # forward exchange: ONE gather launch fills [to left | to right], the
        # receives land straight in local ghost order, ONE scatter launch
        # writes them (small launches were a third of a rank's step at 8 GPUs,
        # tools/rank_share.py)
        self.t_send = torch.cat([self.t_send_left, self.t_send_right])
        self._pos_send = buf(nl + nr)
        self._ghost_in = buf(self.n_gl + self.n_gr)
        send_l, send_r = self._pos_send[:nl], self._pos_send[nl:]
        if self.ghost_centers:
            # a sender's lists hold layer 1 first; [l1 | l2] goes out as two
            # messages per side so that the receiver's four blocks are in place
            ll1, lr1 = self.nl1, self.nr1
            g = self._ghost_in
            a, b = self.n_gl1, self.n_gl1 + self.n_gr1
            c = b + (self.n_gl - self.n_gl1)
            from_l1, from_r1, from_l2, from_r2 = g[:a], g[a:b], g[b:c], g[c:]
            self._fwd_sends = [(send_l[:ll1], self.left, TAG_FWD_LEFT),
                               (send_l[ll1:], self.left, TAG_FWD_LEFT2),
                               (send_r[:lr1], self.right, TAG_FWD_RIGHT),
                               (send_r[lr1:], self.right, TAG_FWD_RIGHT2)]
            self._fwd_recvs = [(from_r1, self.right, TAG_FWD_LEFT),
                               (from_r2, self.right, TAG_FWD_LEFT2),
                               (from_l1, self.left, TAG_FWD_RIGHT),
                               (from_l2, self.left, TAG_FWD_RIGHT2)]
        else:
            from_l, from_r = self._ghost_in[:self.n_gl], self._ghost_in[self.n_gl:]
            self._fwd_sends = [(send_l, self.left, TAG_FWD_LEFT),
                               (send_r, self.right, TAG_FWD_RIGHT)]
            self._fwd_recvs = [(from_r, self.right, TAG_FWD_LEFT),
                               (from_l, self.left, TAG_FWD_RIGHT)]
        # reverse exchange (classic mode): one gather of the ghost forces
        # [left | right] and, unless an atom is sent both ways (slabs of
        # exactly 2 halo), one add over [from left | from right]
        self._f_ghost = buf(self.n_gl + self.n_gr)
        self._f_to = buf(nl + nr)
        self._rev_fused = len(np.intersect1d(self.send_left, self.send_right)) == 0

    # ---- one force evaluation ------------------------------------------
    def forward(self):
        """Refresh ghost positions from their owners."""
        if self.world == 1:
            return
        self.engine.gather_positions(self.t_send, out=self._pos_send)
        self._exchange(self._fwd_sends, self._fwd_recvs)
        self.engine.scatter_positions(self.n_owned, self._ghost_in)

    def _layout(self, from_l, from_r):
        """Received ghost rows in local order: classic [left | right];
        ghost_centers [layer-1 left | layer-1 right | layer-2 left | layer-2 right]."""
        if not self.ghost_centers:
            return [from_l, from_r]
        return [from_l[: self.n_gl1], from_r[: self.n_gr1], from_l[self.n_gl1:],
                from_r[self.n_gr1:]]

    def reverse(self):
        """Send ghost forces home and add them to the owners' forces (classic
        mode; with ghost_centers the owned forces are already complete)."""
        if self.world == 1 or self.ghost_centers:
            return
        f_g = self.engine.ghost_forces(self.n_owned, self.n_gl + self.n_gr, out=self._f_ghost)
        f_gl, f_gr = f_g[:self.n_gl], f_g[self.n_gl:]
        nl = len(self.send_left)
        to_l, to_r = self._f_to[:nl], self._f_to[nl:]
        # my right ghosts are the right neighbour's send_left; my left ghosts its send_right
        self._exchange([(f_gr, self.right, TAG_REV_RIGHT), (f_gl, self.left, TAG_REV_LEFT)],
                       [(to_l, self.left, TAG_REV_RIGHT), (to_r, self.right, TAG_REV_LEFT)])
        if self._rev_fused:
            self.engine.add_forces(self.t_send, self._f_to)
        else:
            self.engine.add_forces(self.t_send_left, to_l)
            self.engine.add_forces(self.t_send_right, to_r)

    def evaluate(self, precision: str = "double", deterministic: bool = False):
        if self.overlap and self.world > 1:
            # ghosts in flight while the interior centres compute (phase 0;
            # a no-op when the engine cannot split yet — phase 1 then does it all)
            self.engine.gather_positions(self.t_send, out=self._pos_send)
            reqs = self._exchange_start(self._fwd_sends, self._fwd_recvs)
            self.engine.compute_phase(0, precision, deterministic)
            self._exchange_finish(reqs)
            self.engine.scatter_positions(self.n_owned, self._ghost_in)
            self.engine.compute_phase(1, precision, deterministic)
        else:
            self.forward()
            self.engine.compute(precision, deterministic)
        self.reverse()

    # ---- atom migration at a rebuild ----------------------
    def migrate(self, xyz: np.ndarray, vel: np.ndarray, cutoff: float, skin: float):
        """Owned atoms that left the slab go to the neighbour that owns them
        now (with species and velocity), arrivals join; ghosts are re-selected
        and the lists rebuilt (setup).  xyz / vel: this rank's owned atoms in
        the order of self.gid.  Returns the new owned velocities (self.gid
        order)."""
        species = self.local_species[: self.n_owned]
        if self.world == 1:
            self.setup(self.gid, xyz, species, cutoff, skin)
            return np.asarray(vel, np.float64)[self.last_order]
        owner = self.slab.owner(xyz[:, 0])
        to_l = owner == self.left
        to_r = (owner == self.right) & ~to_l
        stay = owner == self.rank
        if not np.all(stay | to_l | to_r):
            raise ConfigError("an atom moved farther than one slab between list builds")
        dev = self._device()

        def pack(m):
            return torch.from_numpy(np.column_stack([
                self.gid[m].astype(np.float64), species[m].astype(np.float64), xyz[m],
                vel[m]])).to(dev)
        n_l, n_r = self._swap_counts(int(to_l.sum()), int(to_r.sum()))
        from_l = torch.zeros((n_l, 8), dtype=torch.float64, device=dev)
        from_r = torch.zeros((n_r, 8), dtype=torch.float64, device=dev)
        self._exchange([(pack(to_l), self.left, TAG_FWD_LEFT), (pack(to_r), self.right, TAG_FWD_RIGHT)],
                       [(from_r, self.right, TAG_FWD_LEFT), (from_l, self.left, TAG_FWD_RIGHT)])
        arr = torch.cat([from_l, from_r]).cpu().numpy()
        self.migrated += len(arr)
        gid = np.concatenate([self.gid[stay], arr[:, 0].astype(np.int64)])
        sp = np.concatenate([species[stay], arr[:, 1].astype(np.int32)])
        x = np.concatenate([xyz[stay], arr[:, 2:5]])
        v = np.concatenate([vel[stay], arr[:, 5:8]])
        self.setup(gid, x, sp, cutoff, skin)
        return v[self.last_order]

    def gather_results(self, total_atoms: int):
        """Energy/virial summed over ranks and global-order forces on rank 0
        (a check/report path, not the per-step loop)."""
        ev, f = self.engine.results()
        if self.world > 1:
            dist.all_reduce(ev, group=self.group)
        owned = f[: self.n_owned].double().cpu().numpy()
        parts = [None] * self.world if self.world > 1 else [(self.gid, owned)]
        if self.world > 1:
            dist.all_gather_object(parts, (self.gid, owned), group=self.group)
        forces = np.zeros((total_atoms, 3))
        for gid, fo in parts:
            forces[gid] = fo
        e = ev.cpu().numpy()
        return float(e[0]), forces, e[1:7].copy()


class SlabNVE:
    """Velocity-Verlet NVE across the slab decomposition — the MD step of
    SURVEY.md 8d/8e: every rank integrates its owned atoms (tsf_md_kick),
    ghosts follow by the forward exchange, forces come back by the reverse
    exchange, the rebuild decision is the OR over ranks of the reference's
    needs_rebuild test, and at a rebuild atoms migrate to their new owners
    before ghosts and lists are rebuilt.  Thermo (potential, kinetic energy)
    is summed over ranks.  The closing half-kick of a step is deferred into
    the next opening kick when no sample intervenes, as in tsf_md_run."""

    def __init__(self, dec: "Decomposition", masses, cutoff: float, skin: float,
                 precision: str = "double", deterministic: bool = False):
        self.dec = dec
        self.masses = np.asarray(masses, np.float64)
        self.cutoff, self.skin = float(cutoff), float(skin)
        self.precision, self.deterministic = precision, deterministic
        self.rebuilds = 0
        self._evaluated = False

    def set_velocities(self, vel_owned: np.ndarray):
        """Velocities of the owned atoms, in the order of dec.gid."""
        eng = self.dec.engine
        v = np.zeros((self.dec.n_owned + len(self.dec.ghost_gid), 3))
        v[: self.dec.n_owned] = vel_owned
        eng.md_set_state(v, self.masses)

    def _allreduce(self, values):
        t = torch.tensor(values, dtype=torch.float64, device=self.dec._device())
        if self.dec.world > 1:
            dist.all_reduce(t, group=self.dec.group)
        return t.cpu().numpy()

    def _sample(self, step):
        ev, _ = self.dec.engine.results()
        pe, ke = self._allreduce([float(ev[0].item()), self.dec.engine.kinetic()])
        return (step, float(pe), float(ke))

    def run(self, steps: int, dt: float = 0.001, thermo_every: int = 100):
        dec, eng = self.dec, self.dec.engine
        if not self._evaluated:
            dec.evaluate(self.precision, self.deterministic)
            self._evaluated = True
        samples = [self._sample(0)]
        pending = False
        for s in range(1, steps + 1):
            moved = eng.kick(dt, drift=True, kicks=2 if pending else 1)
            if self._allreduce([1.0 if moved else 0.0])[0] > 0:
                x, v = eng.md_get_state()
                n = dec.n_owned
                vel = dec.migrate(x[:n], v[:n], self.cutoff, self.skin)
                self.set_velocities(vel)
                self.rebuilds += 1
            dec.evaluate(self.precision, self.deterministic)
            if s % thermo_every == 0 or s == steps:
                eng.kick(dt, drift=False)
                samples.append(self._sample(s))
                pending = False
            else:
                pending = True
        return samples

    def owned_state(self):
        """(gid, positions, velocities) of this rank's owned atoms."""
        x, v = self.dec.engine.md_get_state()
        n = self.dec.n_owned
        return self.dec.gid.copy(), x[:n].copy(), v[:n].copy()


def partition(xyz: np.ndarray, box, world: int, rank: int, halo: float) -> np.ndarray:
    """Global ids owned by `rank` (x slabs of equal width)."""
    return np.nonzero(Slab(rank, world, float(box[0]), halo).owner(xyz[:, 0]) == rank)[0]
