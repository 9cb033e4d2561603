"""TEST INFRASTRUCTURE ONLY — ctypes front end for the CPU oracle.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The
product package (``paper_1607_02904_b200``) never imports it.

Two checkers live behind it:

* ``Oracle``    — ``oracle/_build/liboracle.so``, our plain-C restatement of
  the reference algorithm (``oracle/tersoff_oracle.c``), always available.
* ``Reference`` — ``oracle/_ref/libtmdref.so``, the UNMODIFIED reference
  library compiled from ``/root/reference/proj/src`` by ``oracle/Makefile``
  with a C-ABI shim (``oracle/ref_shim.cpp``).  Built in the dev container
  and shipped as a binary; absent ⇒ ``reference_available()`` is False.

``parse_param_text`` restates the reference parser
(``proj/src/params.cpp:119-192``, ``:74-92``) in Python so the oracle does not
depend on the product's C++ parser.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtmdref.so")

# ParamField column order, proj/include/tmd/params.hpp:78-83
FIELDS = ["A", "B", "lam1", "lam2", "lam3", "beta", "eta", "c", "d", "h", "gamma",
          "m", "R", "D", "cut", "cutsq"]
# file column order, proj/include/tmd/params.hpp:62-66
FILE_FIELDS = ["m", "gamma", "lambda3", "c", "d", "h", "eta", "beta", "lambda2", "B",
               "R", "D", "lambda1", "A"]

SI_TEXT = ("Si Si Si 3.0 1.0 1.3258 4.8381 2.0417 0.0000 22.956 "
           "0.33675 1.3258 95.373 3.0 0.2 3.2394 3264.7\n")  # params.cpp:228-234


class OracleParseError(ValueError):
    pass


@dataclass
class OracleParams:
    species: list
    rows: np.ndarray          # (S^3, 16) float64, FlatParams<double> layout
    r_cut_max: float

    @property
    def ns(self) -> int:
        return len(self.species)


def parse_param_text(text: str) -> OracleParams:
    """Restatement of parse_param_text + ParamTable validation."""
    toks = []
    for line in text.split("\n"):
        line = line.split("#", 1)[0]
        toks.extend(t for t in line.replace("\t", " ").replace("\r", " ").split(" ") if t)
    if not toks:
        raise OracleParseError("no entries found")
    if len(toks) % 17:
        raise OracleParseError("truncated entry")
    species: list = []

    def intern(name):
        if name not in species:
            species.append(name)
        return species.index(name)

    raw = []
    for t in range(0, len(toks), 17):
        ids = [intern(toks[t]), intern(toks[t + 1]), intern(toks[t + 2])]
        try:
            num = [float(x) for x in toks[t + 3:t + 17]]
        except ValueError as exc:
            raise OracleParseError(str(exc)) from None
        if num[0] != math.floor(num[0]):
            raise OracleParseError("field 'm' must be an integer")
        raw.append((ids, dict(zip(FILE_FIELDS, num))))
    s = len(species)
    table = [None] * (s ** 3)
    for ids, e in raw:
        idx = (ids[0] * s + ids[1]) * s + ids[2]
        if table[idx] is not None:
            raise OracleParseError("duplicate entry")
        table[idx] = e
    if any(e is None for e in table):
        raise OracleParseError("missing entry")
    rows = np.zeros((s ** 3, 16))
    for idx, e in enumerate(table):
        m = int(e["m"])
        if not all(math.isfinite(v) for v in e.values()):
            raise OracleParseError("field is not finite")
        if m not in (1, 3) or not e["D"] > 0 or not e["R"] > e["D"] or not e["eta"] > 0 \
                or e["beta"] < 0 or e["d"] == 0 or e["A"] < 0 or e["B"] < 0 or e["gamma"] < 0:
            raise OracleParseError("field constraint violated")
        cut = e["R"] + e["D"]
        rows[idx] = [e["A"], e["B"], e["lambda1"], e["lambda2"], e["lambda3"], e["beta"],
                     e["eta"], e["c"], e["d"], e["h"], e["gamma"], float(m), e["R"], e["D"],
                     cut, cut * cut]
    return OracleParams(species, rows, float(rows[:, 14].max()))


def build(quiet: bool = True) -> None:
    """Compile oracle/_build (always) and oracle/_ref (when the reference is present)."""
    subprocess.run(["make", "-C", HERE, "all"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


# --------------------------------------------------------------------------
# our C restatement
# --------------------------------------------------------------------------
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


class OracleNumericError(ArithmeticError):
    pass


class OracleConfigError(ValueError):
    pass


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.orc_compute_ref.argtypes = [C.c_int64, C.c_int64, _dp, _ip, _dp, _up, C.c_int, _dp, _ip, _ip,
                                      C.POINTER(C.c_double), C.POINTER(C.c_longdouble), _dp,
                                      _dp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.orc_compute_ref.restype = C.c_int
        L.orc_build_neighbor_list.argtypes = [C.c_int64, _dp, _dp, _up, C.c_double, C.c_double,
                                              _ip, C.POINTER(C.POINTER(C.c_int32)),
                                              C.POINTER(C.c_int64)]
        L.orc_build_neighbor_list.restype = C.c_int
        L.orc_brute_neighbor_list.argtypes = [C.c_int64, _dp, _dp, _up, C.c_double, _ip,
                                              C.POINTER(C.POINTER(C.c_int32)),
                                              C.POINTER(C.c_int64)]
        L.orc_brute_neighbor_list.restype = C.c_int
        L.orc_filter.argtypes = [C.c_int64, _dp, _dp, _up, _ip, _ip, C.c_double, _ip, _ip]
        L.orc_filter.restype = C.c_int64
        L.orc_needs_rebuild.argtypes = [C.c_int64, _dp, _dp, _dp, _up, C.c_double]
        L.orc_needs_rebuild.restype = C.c_int
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_cutoff_fc.argtypes = [C.c_double, C.c_double, C.c_double,
                                    C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.orc_bond_order.argtypes = [C.c_double, _dp, C.POINTER(C.c_double),
                                     C.POINTER(C.c_double)]
        L.orc_zeta_term.argtypes = [_dp, C.c_double, _dp, C.c_double, _dp,
                                    C.POINTER(C.c_double), _dp, _dp, _dp]
        self.lib = L

    @staticmethod
    def _geom(xyz, box, periodic):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
        box = np.ascontiguousarray(box, dtype=np.float64)
        per = np.ascontiguousarray(periodic, dtype=np.uint8)
        return xyz, box, per

    def _csr(self, fn, n, *args):
        off = np.zeros(n + 1, dtype=np.int32)
        ptr = C.POINTER(C.c_int32)()
        tot = C.c_int64(0)
        rc = fn(n, *args, off, C.byref(ptr), C.byref(tot))
        if rc == 2:
            raise OracleConfigError("neighbor build rejected its inputs")
        if rc != 0:
            raise RuntimeError(f"oracle neighbor build failed rc={rc}")
        nb = np.ctypeslib.as_array(ptr, shape=(tot.value,)).copy() if tot.value else \
            np.zeros(0, dtype=np.int32)
        self.lib.orc_free(C.cast(ptr, C.c_void_p))
        return off, nb

    def build_neighbor_list(self, xyz, box, periodic, cutoff, skin):
        xyz, box, per = self._geom(xyz, box, periodic)
        return self._csr(self.lib.orc_build_neighbor_list, len(xyz), xyz.ravel(), box, per,
                         float(cutoff), float(skin))

    def brute_neighbor_list(self, xyz, box, periodic, bc):
        xyz, box, per = self._geom(xyz, box, periodic)
        return self._csr(self.lib.orc_brute_neighbor_list, len(xyz), xyz.ravel(), box, per,
                         float(bc))

    def filter(self, xyz, box, periodic, offsets, nbrs, r_cut_max):
        xyz, box, per = self._geom(xyz, box, periodic)
        n = len(xyz)
        oo = np.zeros(n + 1, dtype=np.int32)
        on = np.zeros(max(len(nbrs), 1), dtype=np.int32)
        w = self.lib.orc_filter(n, xyz.ravel(), box, per, np.ascontiguousarray(offsets, np.int32),
                                np.ascontiguousarray(nbrs, np.int32), float(r_cut_max), oo, on)
        return oo, on[:w].copy()

    def needs_rebuild(self, xyz, ref_xyz, box, periodic, skin) -> bool:
        xyz, box, per = self._geom(xyz, box, periodic)
        ref = np.ascontiguousarray(ref_xyz, dtype=np.float64).reshape(-1)
        return bool(self.lib.orc_needs_rebuild(len(xyz), xyz.ravel(), ref, box, per,
                                               float(skin)))

    def compute_ref(self, params: OracleParams, xyz, species, box, periodic, offsets, nbrs,
                    n_center=None):
        """Returns dict(energy, energy_ld, forces (n,3), virial (6,)).  With
        n_center, only atoms [0, n_center) are central atoms."""
        xyz, box, per = self._geom(xyz, box, periodic)
        n = len(xyz)
        f = np.zeros(3 * n)
        vir = np.zeros(6)
        e = C.c_double(0)
        eld = C.c_longdouble(0)
        bi, bj = C.c_int64(-1), C.c_int64(-1)
        rc = self.lib.orc_compute_ref(n, n if n_center is None else n_center, xyz.ravel(), np.ascontiguousarray(species, np.int32),
                                      box, per, params.ns, np.ascontiguousarray(params.rows.ravel()),
                                      np.ascontiguousarray(offsets, np.int32),
                                      np.ascontiguousarray(nbrs, np.int32) if len(nbrs) else
                                      np.zeros(1, np.int32),
                                      C.byref(e), C.byref(eld), f, vir, C.byref(bi), C.byref(bj))
        if rc == 3:
            raise OracleNumericError(f"non-finite pair term for atoms {bi.value},{bj.value}")
        if rc != 0:
            raise RuntimeError(f"oracle compute failed rc={rc}")
        return {"energy": e.value, "energy_ld": float(eld.value), "forces": f.reshape(n, 3),
                "virial": vir}

    # scalar pieces for known-answer tests
    def cutoff_fc(self, r, R, D):
        v, d = C.c_double(), C.c_double()
        self.lib.orc_cutoff_fc(r, R, D, C.byref(v), C.byref(d))
        return v.value, d.value

    def bond_order(self, zeta, row):
        v, d = C.c_double(), C.c_double()
        self.lib.orc_bond_order(zeta, np.ascontiguousarray(row, np.float64), C.byref(v),
                                C.byref(d))
        return v.value, d.value


# --------------------------------------------------------------------------
# the unmodified reference, through oracle/ref_shim.cpp
# --------------------------------------------------------------------------
def reference_available() -> bool:
    return os.path.exists(REF_SO)


class RefError(Exception):
    pass


class Reference:
    def __init__(self, path: str = REF_SO):
        L = C.CDLL(path)
        vp, pp = C.c_void_p, C.POINTER(C.c_void_p)
        L.tmdref_last_error.restype = C.c_char_p
        L.tmdref_params_parse.argtypes = [C.c_char_p, pp]
        L.tmdref_params_r_cut_max.argtypes = [vp]
        L.tmdref_params_r_cut_max.restype = C.c_double
        L.tmdref_params_free.argtypes = [vp]
        L.tmdref_system_new.argtypes = [C.c_int64, _dp, _ip, C.c_int, _dp, _dp, _up, pp]
        L.tmdref_system_free.argtypes = [vp]
        L.tmdref_system_size.argtypes = [vp]
        L.tmdref_system_size.restype = C.c_int64
        L.tmdref_system_get.argtypes = [vp, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p]
        L.tmdref_system_set_positions.argtypes = [vp, _dp]
        L.tmdref_system_set_velocities.argtypes = [vp, _dp]
        L.tmdref_diamond_lattice.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int32,
                                             C.c_double, pp]
        L.tmdref_perturbed_lattice.argtypes = [vp, C.c_int, C.c_double, C.c_uint64, pp]
        L.tmdref_init_velocities.argtypes = [vp, C.c_double, C.c_uint64]
        L.tmdref_list_build.argtypes = [vp, C.c_double, C.c_double, pp]
        L.tmdref_list_free.argtypes = [vp]
        L.tmdref_list_entries.argtypes = [vp]
        L.tmdref_list_entries.restype = C.c_int64
        L.tmdref_list_export.argtypes = [vp, _ip, _ip]
        L.tmdref_needs_rebuild.argtypes = [vp, vp]
        L.tmdref_filter.argtypes = [vp, vp, C.c_double, C.c_int, C.c_void_p, C.c_void_p]
        L.tmdref_filter.restype = C.c_int64
        L.tmdref_compute_ref.argtypes = [vp, vp, vp, C.POINTER(C.c_double), C.c_void_p]
        L.tmdref_evaluate.argtypes = [vp, vp, vp, C.c_char_p, C.c_char_p, C.c_int, C.c_int,
                                      C.c_int, C.c_int, C.POINTER(C.c_double), C.c_void_p]
        L.tmdref_fd_forces.argtypes = [vp, vp, vp, C.c_double, _dp]
        L.tmdref_run_nve.argtypes = [vp, vp, C.c_long, C.c_double, C.c_double, C.c_char_p,
                                     C.c_char_p, C.c_int, C.c_int, C.c_int,
                                     C.POINTER(C.c_double), C.POINTER(C.c_double),
                                     C.POINTER(C.c_double), C.POINTER(C.c_int), pp]
        self.lib = L

    def _check(self, rc):
        if rc:
            raise RefError(rc, self.lib.tmdref_last_error().decode())

    # handles are plain ints; callers free them with the *_free helpers
    def params(self, text: str):
        h = C.c_void_p()
        self._check(self.lib.tmdref_params_parse(text.encode(), C.byref(h)))
        return h

    def system(self, xyz, species, masses, box, periodic):
        xyz = np.ascontiguousarray(xyz, np.float64).reshape(-1)
        h = C.c_void_p()
        m = np.ascontiguousarray(masses, np.float64)
        self._check(self.lib.tmdref_system_new(len(xyz) // 3, xyz,
                                               np.ascontiguousarray(species, np.int32),
                                               len(m), m, np.ascontiguousarray(box, np.float64),
                                               np.ascontiguousarray(periodic, np.uint8),
                                               C.byref(h)))
        return h

    def system_arrays(self, h):
        n = self.lib.tmdref_system_size(h)
        xyz = np.zeros((n, 3))
        vel = np.zeros((n, 3))
        sp = np.zeros(n, np.int32)
        box = np.zeros(3)
        per = np.zeros(3, np.uint8)
        self.lib.tmdref_system_get(h, xyz.ctypes.data, vel.ctypes.data, sp.ctypes.data,
                                   box.ctypes.data, per.ctypes.data)
        return xyz, vel, sp, box, per

    def diamond_lattice(self, nx, ny, nz, a0=5.431, species_id=0, mass=28.0855):
        h = C.c_void_p()
        self._check(self.lib.tmdref_diamond_lattice(nx, ny, nz, a0, species_id, mass,
                                                    C.byref(h)))
        return h

    def perturbed_lattice(self, params_h, cells, jitter, seed):
        h = C.c_void_p()
        self._check(self.lib.tmdref_perturbed_lattice(params_h, cells, jitter, seed,
                                                      C.byref(h)))
        return h

    def init_velocities(self, sys_h, temperature, seed):
        self._check(self.lib.tmdref_init_velocities(sys_h, temperature, seed))

    def neighbor_list(self, sys_h, cutoff, skin):
        h = C.c_void_p()
        self._check(self.lib.tmdref_list_build(sys_h, cutoff, skin, C.byref(h)))
        return h

    def list_csr(self, list_h, n):
        tot = self.lib.tmdref_list_entries(list_h)
        off = np.zeros(n + 1, np.int32)
        nb = np.zeros(max(tot, 1), np.int32)
        self.lib.tmdref_list_export(list_h, off, nb)
        return off, nb[:tot]

    def filter_csr(self, list_h, sys_h, r_cut_max, n, apply=True):
        tot = self.lib.tmdref_filter(list_h, sys_h, r_cut_max, int(apply), None, None)
        off = np.zeros(n + 1, np.int32)
        nb = np.zeros(max(tot, 1), np.int32)
        self.lib.tmdref_filter(list_h, sys_h, r_cut_max, int(apply), off.ctypes.data,
                               nb.ctypes.data)
        return off, nb[:tot]

    def compute_ref(self, sys_h, list_h, params_h, n, with_forces=True):
        e = C.c_double()
        f = np.zeros((n, 3)) if with_forces else None
        self._check(self.lib.tmdref_compute_ref(sys_h, list_h, params_h, C.byref(e),
                                                f.ctypes.data if with_forces else None))
        return e.value, f

    def evaluate(self, sys_h, list_h, params_h, n, scheme="auto", precision="opt-d",
                 width=0, k_max=16, workers=1, filter=True, with_forces=True):
        e = C.c_double()
        f = np.zeros((n, 3)) if with_forces else None
        self._check(self.lib.tmdref_evaluate(sys_h, list_h, params_h, scheme.encode(),
                                             precision.encode(), width, k_max, workers,
                                             int(filter), C.byref(e),
                                             f.ctypes.data if with_forces else None))
        return e.value, f

    def run_nve(self, sys_h, params_h, steps, dt=0.001, skin=1.0, scheme="auto",
                precision="opt-d", width=0, workers=1, thermo_every=100):
        wall, e0, e1 = C.c_double(), C.c_double(), C.c_double()
        reb = C.c_int()
        fin = C.c_void_p()
        self._check(self.lib.tmdref_run_nve(sys_h, params_h, steps, dt, skin, scheme.encode(),
                                            precision.encode(), width, workers, thermo_every,
                                            C.byref(wall), C.byref(e0), C.byref(e1),
                                            C.byref(reb), C.byref(fin)))
        return {"wall_seconds": wall.value, "etot_first": e0.value, "etot_last": e1.value,
                "rebuilds": reb.value, "final": fin}

    def free_system(self, h):
        self.lib.tmdref_system_free(h)

    def free_list(self, h):
        self.lib.tmdref_list_free(h)

    def free_params(self, h):
        self.lib.tmdref_params_free(h)
