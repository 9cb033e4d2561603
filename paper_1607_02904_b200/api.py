"""Python surface of the B200 Tersoff path, shaped like the reference's ``tersoffmd``
module (proj/python/bindings.cpp:69-289, proj/python/tersoffmd/__init__.py).

Thin: every force evaluation, neighbor build, filter and rebuild check runs in
``libtersoff_b200.so`` on the GPU through the C-ABI (include/tersoff_b200.h).
Host-side numpy is used only for state bookkeeping (arrays in, arrays out,
kinetic energy of the velocities the caller owns).
"""
from __future__ import annotations

import ctypes as C
import os
import time
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L

MVV2E = 1.0364269e-4          # proj/include/tmd/units.hpp:10
K_BOLTZMANN = 8.617333e-5     # proj/include/tmd/units.hpp:13


# --------------------------------------------------------------------------
# errors (proj/include/tmd/error.hpp:9-21; bindings.cpp:72-74)
# --------------------------------------------------------------------------
class ConfigError(ValueError):
    pass


class ParseError(ValueError):
    pass


class NumericError(ArithmeticError):
    pass


class CudaError(RuntimeError):
    pass


def _raise(rc: int, msg: str, parse: bool = False):
    if rc == L.TSF_ERR_CONFIG:
        if parse and not msg.startswith("cannot open"):
            raise ParseError(msg)
        raise ConfigError(msg)
    if rc == L.TSF_ERR_NUMERIC:
        raise NumericError(msg)
    if rc == L.TSF_ERR_CUDA:
        raise CudaError(msg)
    raise RuntimeError(msg)


def _check(rc: int, ctx=None, parse: bool = False):
    if rc != L.TSF_OK:
        lib = L.lib()
        msg = (lib.tsf_last_error(ctx) if ctx else lib.tsf_error_message()).decode()
        _raise(rc, msg, parse)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# --------------------------------------------------------------------------
# parameter table (params.hpp:40-75)
# --------------------------------------------------------------------------
class ParamTable:
    def __init__(self, handle):
        self._h = handle
        self._lib = L.lib()

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.tsf_params_free(self._h)
            self._h = None

    @property
    def species_count(self) -> int:
        return self._lib.tsf_params_species_count(self._h)

    @property
    def species_names(self) -> list:
        return [self._lib.tsf_params_species_name(self._h, s).decode()
                for s in range(self.species_count)]

    def species_id(self, name: str) -> int:
        return self._lib.tsf_params_species_id(self._h, name.encode())

    @property
    def r_cut_max(self) -> float:
        return self._lib.tsf_params_r_cut_max(self._h)

    @property
    def rows(self) -> np.ndarray:
        """FlatParams<double> rows, (S^3, 16) (params.hpp:88-115)."""
        s = self.species_count
        out = np.zeros((s ** 3, 16))
        _check(self._lib.tsf_params_flat_rows(self._h, _ptr(out), out.size))
        return out

    def serialize(self) -> str:
        n = self._lib.tsf_params_serialize(self._h, None, 0)
        buf = C.create_string_buffer(n + 1)
        self._lib.tsf_params_serialize(self._h, buf, n + 1)
        return buf.value.decode()

    def __repr__(self):
        return f"<ParamTable of {self.species_count} species, r_cut_max {self.r_cut_max:f}>"


def builtin_silicon() -> ParamTable:
    h = C.c_void_p()
    _check(L.lib().tsf_params_builtin_silicon(C.byref(h)), parse=True)
    return ParamTable(h)


def load_params(path: str) -> ParamTable:
    h = C.c_void_p()
    _check(L.lib().tsf_params_load(str(path).encode(), C.byref(h)), parse=True)
    return ParamTable(h)


def parse_params(text: str) -> ParamTable:
    h = C.c_void_p()
    raw = text.encode()
    _check(L.lib().tsf_params_parse(raw, len(raw), b"<string>", C.byref(h)), parse=True)
    return ParamTable(h)


# --------------------------------------------------------------------------
# system state (box.hpp:11-24, system.hpp:14-27)
# --------------------------------------------------------------------------
@dataclass
class SimulationBox:
    lx: float = 0.0
    ly: float = 0.0
    lz: float = 0.0
    periodic_x: bool = True
    periodic_y: bool = True
    periodic_z: bool = True

    @property
    def lengths(self) -> np.ndarray:
        return np.array([self.lx, self.ly, self.lz], dtype=np.float64)

    @property
    def periodic(self) -> np.ndarray:
        return np.array([self.periodic_x, self.periodic_y, self.periodic_z], dtype=np.uint8)


@dataclass
class AtomSystem:
    positions: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    velocities: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    forces: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    species: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    species_masses: list = field(default_factory=list)
    box: SimulationBox = field(default_factory=SimulationBox)

    def __post_init__(self):
        self.positions = np.ascontiguousarray(self.positions, dtype=np.float64).reshape(-1, 3)
        n = len(self.positions)
        self.velocities = np.ascontiguousarray(
            self.velocities if len(self.velocities) else np.zeros((n, 3)), dtype=np.float64)
        self.forces = np.ascontiguousarray(
            self.forces if len(self.forces) else np.zeros((n, 3)), dtype=np.float64)
        self.species = np.ascontiguousarray(
            self.species if len(self.species) else np.zeros(n, np.int32), dtype=np.int32)

    @property
    def natoms(self) -> int:
        return len(self.positions)

    def copy(self) -> "AtomSystem":
        return AtomSystem(self.positions.copy(), self.velocities.copy(), self.forces.copy(),
                          self.species.copy(), list(self.species_masses),
                          SimulationBox(**vars(self.box)))

    def validate(self):
        """system.cpp:10-26"""
        n = self.natoms
        if len(self.velocities) != n or len(self.forces) != n or len(self.species) != n:
            raise ConfigError("atom state arrays disagree on atom count")
        if not (self.box.lx > 0 and self.box.ly > 0 and self.box.lz > 0):
            raise ConfigError("simulation box edges must be positive")
        for a, s in enumerate(self.species):
            if s < 0 or s >= len(self.species_masses):
                raise ConfigError(f"atom {a} has species id {s} without a mass entry")
        for s, m in enumerate(self.species_masses):
            if not m > 0:
                raise ConfigError(f"species {s} has non-positive mass")

    def __repr__(self):
        return f"<AtomSystem of {self.natoms} atoms>"


def make_diamond_lattice(nx, ny, nz, a0=5.431, species_id=0, mass=28.0855) -> AtomSystem:
    """engine.cpp:28-58"""
    if not mass > 0:
        raise ConfigError("species mass must be positive")
    lib = L.lib()
    n = lib.tsf_diamond_lattice_size(nx, ny, nz)
    xyz = np.zeros((max(n, 0), 3))
    sp = np.zeros(max(n, 0), np.int32)
    box = np.zeros(3)
    _check(lib.tsf_make_diamond_lattice(nx, ny, nz, a0, species_id, _ptr(xyz), _ptr(sp),
                                        _ptr(box)))
    return AtomSystem(xyz, species=sp, species_masses=[mass] * (species_id + 1),
                      box=SimulationBox(*box))


def perturbed_lattice(params: ParamTable, cells: int, jitter: float, seed: int) -> AtomSystem:
    """verify.cpp:83-104"""
    lib = L.lib()
    n = cells ** 3 * 8
    xyz = np.zeros((n, 3))
    sp = np.zeros(n, np.int32)
    masses = np.zeros(params.species_count)
    box = np.zeros(3)
    _check(lib.tsf_perturbed_lattice(params._h, cells, jitter, seed, _ptr(xyz), _ptr(sp),
                                     _ptr(masses), _ptr(box)))
    return AtomSystem(xyz, species=sp, species_masses=list(masses), box=SimulationBox(*box))


def init_velocities(system: AtomSystem, temperature: float, seed: int) -> None:
    """engine.cpp:64-116 (mt19937_64 Box-Muller, COM removal, exact rescale)."""
    m = np.ascontiguousarray(system.species_masses, dtype=np.float64)
    v = np.zeros((system.natoms, 3))
    _check(L.lib().tsf_init_velocities(system.natoms, _ptr(system.species), _ptr(m),
                                       temperature, seed, _ptr(v)))
    system.velocities = v


def kinetic_energy(system: AtomSystem) -> float:
    m = np.asarray(system.species_masses)[system.species]
    return float(np.sum(0.5 * m * np.sum(system.velocities ** 2, axis=1) * MVV2E))


def temperature(system: AtomSystem) -> float:
    if system.natoms == 0:
        return 0.0
    return 2.0 * kinetic_energy(system) / (3.0 * system.natoms * K_BOLTZMANN)


def total_momentum(system: AtomSystem):
    m = np.asarray(system.species_masses)[system.species]
    p = (system.velocities * m[:, None]).sum(axis=0)
    return float(p[0]), float(p[1]), float(p[2])


# --------------------------------------------------------------------------
# on-disk snapshots (tsf_snapshot_*; format in csrc/tsf_snapshot.cpp)
# --------------------------------------------------------------------------
SNAP_F32_COORDS = 0x1
SNAP_VELOCITIES = 0x2


def save_snapshot(path: str, system: AtomSystem, float32_coords: bool = False,
                  velocities: bool = False) -> str:
    """Write `system` (positions, species, masses, box[, velocities]) with a
    SHA-256 trailer; returns the hex digest.  With float32_coords the stored
    state is the float32-rounded one — reload the file to get it."""
    ns = len(system.species_masses)
    m = np.ascontiguousarray(system.species_masses, dtype=np.float64)
    flags = (SNAP_F32_COORDS if float32_coords else 0) | (SNAP_VELOCITIES if velocities else 0)
    sha = (C.c_uint8 * 32)()
    _check(L.lib().tsf_snapshot_write(
        os.fsencode(path), system.natoms, _ptr(system.positions), _ptr(system.species), ns,
        _ptr(m), _ptr(system.box.lengths), _ptr(system.box.periodic),
        _ptr(system.velocities) if velocities else None, flags, sha))
    return bytes(sha).hex()


def snapshot_info(path: str) -> dict:
    """Header of a snapshot after its checksum is verified."""
    n, ns, fl = C.c_int64(), C.c_int(), C.c_uint32()
    sha = (C.c_uint8 * 32)()
    _check(L.lib().tsf_snapshot_info(os.fsencode(path), C.byref(n), C.byref(ns), C.byref(fl),
                                     sha))
    return {"natoms": n.value, "species_count": ns.value, "flags": fl.value,
            "sha256": bytes(sha).hex()}


def load_snapshot(path: str) -> AtomSystem:
    """Read a snapshot (checksum verified) into an AtomSystem."""
    info = snapshot_info(path)
    n, ns = info["natoms"], info["species_count"]
    xyz, vel = np.zeros((n, 3)), np.zeros((n, 3))
    sp = np.zeros(n, np.int32)
    m, box = np.zeros(ns), np.zeros(3)
    per = np.zeros(3, np.uint8)
    _check(L.lib().tsf_snapshot_read(os.fsencode(path), _ptr(xyz), _ptr(sp), _ptr(m), _ptr(box),
                                     _ptr(per), _ptr(vel)))
    return AtomSystem(xyz, vel, species=sp, species_masses=list(m),
                      box=SimulationBox(*box, *(bool(p) for p in per)))


# --------------------------------------------------------------------------
# device context
# --------------------------------------------------------------------------
PRECISIONS = {"ref": 0, "opt-d": 0, "double": 0, "opt-m": 1, "mixed": 1, "opt-s": 2, "single": 2}
PRECISION_NAMES = {0: "opt-d", 1: "opt-m", 2: "opt-s"}
SCHEMES = ("auto", "ref", "scalar-opt", "v1", "v2", "v3")


def default_device() -> int:
    return int(os.environ.get("LOCAL_RANK", os.environ.get("TSF_DEVICE", "0")))


class Context:
    """A device context: one CUDA stream with the system, lists and force
    buffers resident in HBM.  ``params=None`` gives a list-only context."""

    def __init__(self, params: ParamTable | None, device: int | None = None):
        self._lib = L.lib()
        self.params = params
        self.device = default_device() if device is None else device
        h = C.c_void_p()
        _check(self._lib.tsf_create(params._h if params is not None else None, self.device,
                                    C.byref(h)))
        self._h = h
        self.n = -1
        self._list_ref = None

    def close(self):
        if getattr(self, "_h", None):
            self._lib.tsf_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def _ok(self, rc):
        _check(rc, self._h)

    @property
    def stream(self) -> int:
        return self._lib.tsf_stream(self._h) or 0

    @property
    def launches(self) -> int:
        return self._lib.tsf_launch_count(self._h)

    @property
    def near_refreshes(self) -> int:
        """Near-list refreshes by the force-path filter since creation."""
        return self._lib.tsf_near_refreshes(self._h)

    def profile(self, on: bool = True):
        self._ok(self._lib.tsf_profile_enable(self._h, int(on)))

    def profile_read(self, reset: bool = True):
        """Accumulated per-stage ms: filter, setup, force kernel, tail; and the call count."""
        ms = np.zeros(4)
        calls = C.c_int64(0)
        self._ok(self._lib.tsf_profile_read(self._h, _ptr(ms), C.byref(calls), int(reset)))
        return {"filter_ms": ms[0], "setup_ms": ms[1], "force_ms": ms[2], "tail_ms": ms[3],
                "calls": calls.value}

    def set_system(self, positions, species, box_lengths, periodic=(1, 1, 1)):
        xyz = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
        sp = np.ascontiguousarray(species, dtype=np.int32)
        box = np.ascontiguousarray(box_lengths, dtype=np.float64)
        per = np.ascontiguousarray(periodic, dtype=np.uint8)
        if len(sp) != len(xyz):
            raise ConfigError("atom state arrays disagree on atom count")
        self._ok(self._lib.tsf_set_system(self._h, len(xyz), _ptr(xyz), _ptr(sp), _ptr(box),
                                          _ptr(per)))
        self.n = len(xyz)

    def load(self, system: AtomSystem):
        self.set_system(system.positions, system.species, system.box.lengths, system.box.periodic)

    def set_positions(self, positions):
        xyz = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
        if len(xyz) != self.n:
            raise ConfigError("position array does not match the system size")
        self._ok(self._lib.tsf_set_positions(self._h, _ptr(xyz)))

    def get_positions(self) -> np.ndarray:
        out = np.zeros((self.n, 3))
        self._ok(self._lib.tsf_get_positions(self._h, _ptr(out)))
        return out

    def build_neighbor_list(self, cutoff: float | None = None, skin: float = 1.0):
        if cutoff is None:
            cutoff = self.params.r_cut_max
        self._ok(self._lib.tsf_build_neighbor_list(self._h, float(cutoff), float(skin)))
        self._list_ref = None

    def set_neighbor_list(self, offsets, neighbors, cutoff: float, skin: float):
        off = np.ascontiguousarray(offsets, dtype=np.int32)
        nb = np.ascontiguousarray(neighbors, dtype=np.int32)
        if len(off) != self.n + 1:
            raise ConfigError("neighbor offsets must have natoms + 1 entries")
        if len(nb) == 0:
            nb = np.zeros(1, np.int32)
        self._ok(self._lib.tsf_set_neighbor_list(self._h, _ptr(off), _ptr(nb), float(cutoff),
                                                 float(skin)))

    def needs_rebuild(self) -> bool:
        out = C.c_int(0)
        self._ok(self._lib.tsf_needs_rebuild(self._h, C.byref(out)))
        return bool(out.value)

    def export_neighbors(self, which: str = "skin"):
        sel = L.TSF_LIST_SKIN if which == "skin" else L.TSF_LIST_SHORT
        tot = self._lib.tsf_neighbor_entries(self._h, sel)
        if tot < 0:
            self._ok(int(-tot))
        off = np.zeros(self.n + 1, np.int32)
        nb = np.zeros(max(tot, 1), np.int32)
        self._ok(self._lib.tsf_export_neighbors(self._h, sel, _ptr(off), _ptr(nb), len(nb)))
        return off, nb[:tot]

    def compute(self, precision="double", deterministic=False, filter=True, energy=True,
                forces=True, virial=True, form_virial=True):
        """Evaluate on the current system and list.  Returns (E, F, W) with
        None for outputs not requested; requesting nothing keeps the results on
        the device and does not synchronize.  The virial is not formed when it
        is not requested next to E or F, or when form_virial is False
        (TSF_NO_VIRIAL: the device results then hold zeros for it)."""
        p = PRECISIONS[precision] if isinstance(precision, str) else int(precision)
        fn = (self._lib.tsf_compute_f64, self._lib.tsf_compute_mixed,
              self._lib.tsf_compute_f32)[p]
        flags = (L.TSF_DETERMINISTIC if deterministic else 0) | (0 if filter else L.TSF_NO_FILTER)
        if not form_virial:
            flags |= L.TSF_NO_VIRIAL
        e = C.c_double(0.0)
        f = np.zeros((self.n, 3)) if forces else None
        w = np.zeros(6) if virial else None
        self._ok(fn(self._h, flags, C.byref(e) if energy else None,
                    _ptr(f) if forces else None, _ptr(w) if virial else None))
        return (e.value if energy else None), f, w

    def md_set_state(self, velocities, masses):
        v = np.ascontiguousarray(velocities, dtype=np.float64).reshape(-1, 3)
        m = np.ascontiguousarray(masses, dtype=np.float64)
        self._ok(self._lib.tsf_md_set_state(self._h, _ptr(v), _ptr(m)))

    def md_scale_velocities(self, factor: float):
        self._ok(self._lib.tsf_md_scale_velocities(self._h, float(factor)))

    def md_kick(self, dt: float, drift: bool = True, kicks: int = 1, check: bool = True):
        """One velocity-Verlet piece (tsf_md_kick): `kicks` half-kicks, then
        with drift the position update, wrap and the rebuild test; returns
        whether some owned atom moved more than skin/2 since the list build."""
        moved = C.c_int(0)
        self._ok(self._lib.tsf_md_kick(self._h, float(dt), int(bool(drift)), int(kicks),
                                       C.byref(moved) if check else None))
        return bool(moved.value)

    def set_interior(self, n_interior: int):
        """User atoms [0, n_interior) have no ghost within cutoff + skin;
        the next list build lets evaluations split (tsf_set_interior)."""
        self._ok(self._lib.tsf_set_interior(self._h, int(n_interior)))

    def compute_phase(self, phase: int, precision: str = "double", deterministic: bool = False):
        """Half of a split evaluation (tsf_compute_phase): 0 the interior
        centres, 1 the rest and the reductions.  Results via the device."""
        p = PRECISIONS[precision] if isinstance(precision, str) else int(precision)
        flags = L.TSF_DETERMINISTIC if deterministic else 0
        self._ok(self._lib.tsf_compute_phase(self._h, p, flags, int(phase)))

    def md_kinetic(self) -> float:
        """Kinetic energy of the owned atoms, eV."""
        ke = C.c_double(0.0)
        self._ok(self._lib.tsf_md_kinetic(self._h, C.byref(ke)))
        return ke.value

    def md_get_state(self):
        x = np.zeros((self.n, 3))
        v = np.zeros((self.n, 3))
        self._ok(self._lib.tsf_md_get_state(self._h, _ptr(x), _ptr(v)))
        return x, v

    def md_run(self, steps, dt=0.001, precision="double", deterministic=False,
               thermo_every=100):
        p = PRECISIONS[precision] if isinstance(precision, str) else int(precision)
        cap = steps // thermo_every + 3
        thermo = np.zeros((cap, 3))
        ns, nreb = C.c_int64(0), C.c_int64(0)
        flags = L.TSF_DETERMINISTIC if deterministic else 0
        self._ok(self._lib.tsf_md_run(self._h, p, steps, dt, flags, thermo_every, _ptr(thermo),
                                      cap, C.byref(ns), C.byref(nreb)))
        return thermo[:ns.value], nreb.value


_contexts: dict = {}


def _context_for(params: ParamTable | None, device: int | None = None) -> Context:
    dev = default_device() if device is None else device
    key = (id(params) if params is not None else None, dev)
    ent = _contexts.get(key)
    if ent is not None and (params is None or ent[1]() is params):
        return ent[0]
    ctx = Context(params, dev)
    _contexts[key] = (ctx, weakref.ref(params) if params is not None else (lambda: None))
    return ctx


# --------------------------------------------------------------------------
# neighbor lists (neighbor.hpp:15-54)
# --------------------------------------------------------------------------
class NeighborList:
    """Full, ascending CSR list within cutoff + skin, built on the GPU."""

    def __init__(self, offsets, neighbors, skin, build_cutoff, reference_positions):
        self.offsets = offsets
        self.neighbors = neighbors
        self.skin = skin
        self.build_cutoff = build_cutoff
        self.reference_positions = reference_positions

    @property
    def natoms(self) -> int:
        return len(self.offsets) - 1

    @property
    def pair_count(self) -> int:
        return len(self.neighbors)

    def segment(self, i: int) -> np.ndarray:
        if not 0 <= i < self.natoms:
            raise IndexError("atom index out of range")
        return self.neighbors[self.offsets[i]:self.offsets[i + 1]].copy()

    def __repr__(self):
        return f"<NeighborList of {self.natoms} atoms, {self.pair_count} entries>"


def build_neighbor_list(system: AtomSystem, cutoff: float, skin: float = 0.0) -> NeighborList:
    ctx = _context_for(None)
    ctx.load(system)
    ctx.build_neighbor_list(cutoff, skin)
    off, nb = ctx.export_neighbors("skin")
    return NeighborList(off, nb, float(skin), float(cutoff) + float(skin),
                        system.positions.copy())


def needs_rebuild(lst: NeighborList, system: AtomSystem) -> bool:
    ctx = _context_for(None)
    ctx.set_system(lst.reference_positions, system.species, system.box.lengths,
                   system.box.periodic)
    ctx.set_neighbor_list(lst.offsets, lst.neighbors, lst.build_cutoff - lst.skin, lst.skin)
    ctx.set_positions(system.positions)
    return ctx.needs_rebuild()


def _resolve_options(scheme, precision, width, k_max, workers):
    """Option validation of evaluate_forces (potential_opt.cpp:51-138).  The
    CPU lane width, worker count and k_max have no GPU meaning (the group width
    follows the short-list occupancy; the derivative cache is the group) but
    are validated the same way."""
    if scheme not in SCHEMES:
        raise ConfigError(f"unknown scheme '{scheme}' (expected auto, ref, scalar-opt, v1, v2, "
                          "or v3)")
    if precision not in PRECISIONS:
        raise ConfigError(f"unknown precision '{precision}' (expected ref, double (opt-d), "
                          "single (opt-s), or mixed (opt-m))")
    if k_max < 0:
        raise ConfigError("k_max must be non-negative")
    if workers < 1:
        raise ConfigError("worker count must be at least 1")
    if width not in (0, 1, 4, 8, 16):
        raise ConfigError(f"unsupported backend width {width} (supported: 1, 4, 8, 16)")
    p = PRECISIONS[precision]
    if scheme in ("ref", "scalar-opt") and p != 0:
        raise ConfigError(f"scheme {scheme} runs in double precision only")
    return p


def evaluate_forces(system: AtomSystem, lst: NeighborList, params: ParamTable,
                    scheme: str = "auto", precision: str = "opt-d", width: int = 0,
                    k_max: int = 16, filter: bool = True, workers: int = 1,
                    deterministic: bool = True, virial: bool = False):
    """evaluate_forces (potential_opt.hpp:105-106) on the GPU: (energy, forces[, virial])."""
    p = _resolve_options(scheme, precision, width, k_max, workers)
    ctx = _context_for(params)
    ctx.load(system)
    if lst.natoms != system.natoms:
        raise ConfigError("neighbor list and system disagree on atom count")
    if ctx._list_ref is None or ctx._list_ref() is not lst:
        ctx.set_neighbor_list(lst.offsets, lst.neighbors, lst.build_cutoff - lst.skin, lst.skin)
        ctx._list_ref = weakref.ref(lst)
    e, f, w = ctx.compute(p, deterministic=deterministic, filter=filter, virial=virial)
    return (e, f, w) if virial else (e, f)


# --------------------------------------------------------------------------
# NVE driver (engine.hpp:16-93), GPU-resident
# --------------------------------------------------------------------------
def run_nve(system: AtomSystem, params: ParamTable, steps: int, dt: float = 0.001,
            skin: float = 1.0, scheme: str = "auto", precision: str = "opt-d", width: int = 0,
            k_max: int = 16, workers: int = 1, thermo_every: int = 100,
            rebuild_check_every: int = 1, deterministic: bool = False):
    p = _resolve_options(scheme, precision, width, k_max, workers)
    if steps < 0:
        raise ConfigError("steps must be non-negative")
    if not dt > 0:
        raise ConfigError("dt must be positive")
    if skin < 0:
        raise ConfigError("skin must be non-negative")
    if rebuild_check_every != 1:
        raise ConfigError("the GPU engine checks list staleness every step")
    system.validate()
    if system.species.max(initial=-1) >= params.species_count:
        raise ConfigError("system uses a species id the parameter table does not define")
    ctx = Context(params)
    ctx.load(system)
    ctx.build_neighbor_list(params.r_cut_max, skin)
    ctx.md_set_state(system.velocities, system.species_masses)
    ctx.compute(p, deterministic=deterministic, energy=False, forces=False, virial=False)
    t0 = time.perf_counter()
    thermo, rebuilds = ctx.md_run(steps, dt, p, deterministic, thermo_every)
    wall = time.perf_counter() - t0
    n = system.natoms
    samples = []
    for step, pe, ke in thermo:
        samples.append({"step": int(step), "time_ps": step * dt,
                        "temp_K": 2.0 * ke / (3.0 * n * K_BOLTZMANN) if n else 0.0,
                        "pe_eV": pe, "ke_eV": ke, "etot_eV": pe + ke})
    x, v = ctx.md_get_state()
    _, fcur, _ = ctx.compute(p, deterministic=deterministic, energy=False, virial=False)
    final = system.copy()
    final.positions, final.velocities, final.forces = x, v, fcur
    ns_day = (steps * dt * 1e-3) / wall * 86400.0 if steps > 0 and wall > 0 else 0.0
    rows = ["step,time_ps,temp_K,pe_eV,ke_eV,etot_eV"]
    for s in samples:
        rows.append(",".join([str(s["step"])] + [repr(float(s[k])) for k in
                                                  ("time_ps", "temp_K", "pe_eV", "ke_eV",
                                                   "etot_eV")]))
    rows += [f"scheme,{'gpu-group'}", f"width,{width or (4 if p == 0 else 8)}",
             f"precision,{PRECISION_NAMES[p]}", f"ns_per_day,{ns_day!r}"]
    ctx.close()
    return {"samples": samples, "wall_seconds": wall, "ns_per_day": ns_day,
            "scheme": "gpu-group", "precision": PRECISION_NAMES[p],
            "width": width or (4 if p == 0 else 8), "neighbor_rebuilds": rebuilds,
            "csv": "\n".join(rows) + "\n", "system": final}


def melt(system: AtomSystem, params: ParamTable, hot_temperature: float = 6000.0,
         hot_ps: float = 2.0, temperature: float = 3000.0, hold_ps: float = 4.0,
         dt: float = 0.0005, rescale_every: int = 50, seed: int = 12345,
         precision: str = "double") -> AtomSystem:
    """Liquid fixture generator (SURVEY.md 8d cfg 5): Maxwell-Boltzmann at
    `hot_temperature`, hold there for `hot_ps`, then at `temperature` for
    `hold_ps`, velocity-Verlet with velocity rescaling every `rescale_every`
    steps — GPU-resident (tsf_md_run + tsf_md_scale_velocities)."""
    work = system.copy()
    init_velocities(work, hot_temperature, seed)
    ctx = Context(params)
    ctx.load(work)
    ctx.build_neighbor_list(params.r_cut_max, 1.0)
    ctx.md_set_state(work.velocities, work.species_masses)
    n = work.natoms
    for target, ps in ((hot_temperature, hot_ps), (temperature, hold_ps)):
        blocks = max(1, int(round(ps / dt / rescale_every)))
        for _ in range(blocks):
            thermo, _ = ctx.md_run(rescale_every, dt, precision, False, rescale_every)
            t_now = 2.0 * thermo[-1, 2] / (3.0 * n * K_BOLTZMANN)
            if t_now > 0:
                ctx.md_scale_velocities(np.sqrt(target / t_now))
    x, v = ctx.md_get_state()
    ctx.close()
    out = work.copy()
    out.positions, out.velocities = x, v
    out.forces = np.zeros_like(x)
    return out
