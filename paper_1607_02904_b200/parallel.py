"""Multi-GPU x-slab domain decomposition: a thin ctypes
surface over the C++ decomposition in libtersoff_b200.so (csrc/tsf_dd.cu,
`tsf_dd_*` in include/tersoff_b200.h).

One process (or, with the LOCAL transport, one host thread) per rank; each
rank owns the atoms of one slab of the periodic x axis and keeps ghosts
within one halo (r_cut_max + skin) of its faces — two halos with
`ghost_centers`.  Ghost selection, the per-step ghost-position exchange, the
reverse ghost-force exchange, atom migration at rebuilds and the distributed
velocity-Verlet loop all run on the device in C++; this module only moves
host arrays in and out.

Transports:
  * NCCL between processes (`nccl_unique_id()` on rank 0, broadcast by the
    caller, e.g. over torch.distributed);
  * LOCAL: several ranks in one process sharing a `LocalGroup`, one host
    thread per rank — the multi-rank path on one GPU.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .api import CudaError, ConfigError, NumericError, Context, PRECISIONS, _ptr

GHOST_CENTERS = 0x1


def _dd_check(rc: int):
    if rc == L.TSF_OK:
        return
    msg = L.lib().tsf_dd_error_message().decode()
    if rc == L.TSF_ERR_NUMERIC:
        raise NumericError(msg)
    if rc == L.TSF_ERR_CONFIG:
        raise ConfigError(msg)
    raise CudaError(msg)


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0; distribute it to every rank)."""
    buf = (C.c_uint8 * 128)()
    _dd_check(L.lib().tsf_dd_nccl_unique_id(buf))
    return bytes(buf)


class LocalGroup:
    """The in-process transport's group: `world` ranks of one process."""

    def __init__(self, world: int):
        self.world = world
        self._h = C.c_void_p()
        _dd_check(L.lib().tsf_dd_group_create(world, C.byref(self._h)))

    def close(self):
        if self._h:
            L.lib().tsf_dd_group_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class DomainDecomposition:
    """One rank of the C++ decomposition.

    transport: a LocalGroup (in-process ranks) or "nccl" (then `world`,
    `rank` and `unique_id` from nccl_unique_id() on rank 0)."""

    def __init__(self, params, device: int, box, periodic, cutoff: float, skin: float,
                 transport, rank: int, world: int | None = None, unique_id: bytes | None = None,
                 masses=None, ghost_centers: bool = False):
        self.ctx = Context(params, device)
        self.rank = rank
        lib = L.lib()
        box = np.ascontiguousarray(box, np.float64)
        per = np.ascontiguousarray(periodic, np.uint8)
        m = None if masses is None else np.ascontiguousarray(masses, np.float64)
        mode = GHOST_CENTERS if ghost_centers else 0
        self._h = C.c_void_p()
        if isinstance(transport, LocalGroup):
            self.world = transport.world
            self._group = transport
            rc = lib.tsf_dd_create_local(self.ctx._h, transport._h, rank, float(cutoff),
                                         float(skin), _ptr(box), _ptr(per),
                                         _ptr(m) if m is not None else None, mode,
                                         C.byref(self._h))
        elif transport == "nccl":
            if unique_id is None or world is None:
                raise ConfigError("the NCCL transport needs world and the rank-0 unique id")
            self.world = world
            idb = (C.c_uint8 * 128).from_buffer_copy(unique_id)
            rc = lib.tsf_dd_create_nccl(self.ctx._h, world, rank, idb, float(cutoff),
                                        float(skin), _ptr(box), _ptr(per),
                                        _ptr(m) if m is not None else None, mode,
                                        C.byref(self._h))
        else:
            raise ConfigError(f"unknown transport {transport!r}")
        _dd_check(rc)

    def setup(self, gid, xyz, species, velocities=None):
        """This rank's owned atoms (global ids, global-frame positions)."""
        gid = np.ascontiguousarray(gid, np.int64)
        xyz = np.ascontiguousarray(xyz, np.float64).reshape(-1, 3)
        sp = np.ascontiguousarray(species, np.int32)
        v = None if velocities is None else np.ascontiguousarray(velocities,
                                                                   np.float64).reshape(-1, 3)
        _dd_check(L.lib().tsf_dd_setup(self._h, len(gid), _ptr(gid), _ptr(xyz), _ptr(sp),
                                       _ptr(v) if v is not None else None))

    def set_positions(self, xyz):
        """Owned positions in gid order (as results() returns them); pinned
        host memory goes straight over PCIe."""
        x = np.ascontiguousarray(xyz, np.float64).reshape(-1, 3)
        _dd_check(L.lib().tsf_dd_set_positions(self._h, _ptr(x)))

    def set_positions_ptr(self, ptr: int):
        """As set_positions, from a raw host pointer (e.g. a pinned tensor)."""
        _dd_check(L.lib().tsf_dd_set_positions(self._h, C.c_void_p(ptr)))

    @property
    def stream(self) -> int:
        return self.ctx.stream

    def evaluate(self, precision="double", deterministic=False):
        p = PRECISIONS[precision] if isinstance(precision, str) else int(precision)
        _dd_check(L.lib().tsf_dd_evaluate(self._h, p, L.TSF_DETERMINISTIC if deterministic else 0))

    def rebuild(self):
        _dd_check(L.lib().tsf_dd_rebuild(self._h))

    def md_run(self, steps, dt=0.001, precision="double", deterministic=False, thermo_every=100):
        p = PRECISIONS[precision] if isinstance(precision, str) else int(precision)
        cap = steps // thermo_every + 3
        thermo = np.zeros((cap, 3))
        ns, nreb = C.c_int64(0), C.c_int64(0)
        _dd_check(L.lib().tsf_dd_md_run(self._h, p, steps, dt,
                                        L.TSF_DETERMINISTIC if deterministic else 0,
                                        thermo_every, _ptr(thermo), cap, C.byref(ns),
                                        C.byref(nreb)))
        return thermo[:ns.value], nreb.value

    @property
    def counts(self) -> dict:
        c = np.zeros(8, np.int64)
        _dd_check(L.lib().tsf_dd_counts(self._h, _ptr(c)))
        keys = ("owned", "centres", "local", "sent_left", "sent_right", "rebuilds", "migrated",
                "ghost_centers")
        return dict(zip(keys, (int(x) for x in c)))

    def results(self, positions=False, velocities=False):
        """(energy, virial[6]) summed over ranks, and this rank's owned atoms
        in gid order: gid, forces (+ positions / velocities on request)."""
        n = self.counts["owned"]
        ev = np.zeros(7)
        gid = np.zeros(n, np.int64)
        f = np.zeros((n, 3))
        x = np.zeros((n, 3)) if positions else None
        v = np.zeros((n, 3)) if velocities else None
        _dd_check(L.lib().tsf_dd_results(self._h, _ptr(ev), _ptr(gid),
                                         _ptr(x) if x is not None else None, _ptr(f),
                                         _ptr(v) if v is not None else None))
        out = {"energy": float(ev[0]), "virial": ev[1:7].copy(), "gid": gid, "forces": f}
        if positions:
            out["positions"] = x
        if velocities:
            out["velocities"] = v
        return out

    def forces_into(self, ptr: int):
        """Owned forces (gid order) straight into host memory at `ptr` (e.g. a
        pinned tensor of n_owned x 3 doubles)."""
        _dd_check(L.lib().tsf_dd_results(self._h, None, None, None, C.c_void_p(ptr), None))

    def close(self):
        if self._h:
            L.lib().tsf_dd_destroy(self._h)
            self._h = C.c_void_p()
        self.ctx.close()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def partition(xyz: np.ndarray, box, world: int, rank: int) -> np.ndarray:
    """Global ids owned by `rank`: x slabs of equal width (tsf_dd's owner rule)."""
    L_ = float(box[0])
    x = np.mod(xyz[:, 0], L_)
    owner = np.minimum((x / (L_ / world)).astype(np.int64), world - 1)
    return np.nonzero(owner == rank)[0]
