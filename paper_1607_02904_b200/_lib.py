"""Loader for the sm_100a extension ``libtersoff_b200.so`` (C-ABI: include/tersoff_b200.h).

The library is built in-tree (``make -C paper_1607_02904_b200/csrc``).  If it
is missing we try to build it once; if that fails the import fails loudly —
there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# TSF_LIBRARY: an alternative build of the same sources (side-by-side experiments)
LIB_PATH = os.environ.get("TSF_LIBRARY") or os.path.join(HERE, "libtersoff_b200.so")
CSRC = os.path.join(HERE, "csrc")

TSF_OK, TSF_ERR_INTERNAL, TSF_ERR_CONFIG, TSF_ERR_NUMERIC, TSF_ERR_CUDA = 0, 1, 2, 3, 4
TSF_DETERMINISTIC = 0x1
TSF_NO_FILTER = 0x2
TSF_NO_VIRIAL = 0x4
TSF_LIST_SKIN, TSF_LIST_SHORT = 0, 1

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the extension for sm_100a; returns the .so path."""
    cmd = ["make", "-C", CSRC, "-j8"]
    if force:
        subprocess.run(["make", "-C", CSRC, "clean"], check=True, stdout=subprocess.DEVNULL)
    subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL)
    return LIB_PATH


_vp = C.c_void_p
_pp = C.POINTER(C.c_void_p)
_d = C.c_double
_dptr = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)

# (name, restype, argtypes) — every symbol declared in include/tersoff_b200.h
PROTOTYPES = [
    ("tsf_error_message", C.c_char_p, []),
    ("tsf_last_error", C.c_char_p, [_vp]),
    ("tsf_version", C.c_char_p, []),
    ("tsf_params_parse", C.c_int, [C.c_char_p, C.c_size_t, C.c_char_p, _pp]),
    ("tsf_params_load", C.c_int, [C.c_char_p, _pp]),
    ("tsf_params_builtin_silicon", C.c_int, [_pp]),
    ("tsf_params_free", None, [_vp]),
    ("tsf_params_species_count", C.c_int, [_vp]),
    ("tsf_params_species_name", C.c_char_p, [_vp, C.c_int]),
    ("tsf_params_species_id", C.c_int, [_vp, C.c_char_p]),
    ("tsf_params_r_cut_max", C.c_double, [_vp]),
    ("tsf_params_flat_rows", C.c_int, [_vp, _vp, C.c_size_t]),
    ("tsf_params_serialize", C.c_int64, [_vp, C.c_char_p, C.c_size_t]),
    ("tsf_diamond_lattice_size", C.c_int64, [C.c_int, C.c_int, C.c_int]),
    ("tsf_make_diamond_lattice", C.c_int, [C.c_int, C.c_int, C.c_int, _d, C.c_int32, _vp, _vp,
                                          _vp]),
    ("tsf_perturbed_lattice", C.c_int, [_vp, C.c_int, _d, C.c_uint64, _vp, _vp, _vp, _vp]),
    ("tsf_init_velocities", C.c_int, [C.c_int64, _vp, _vp, _d, C.c_uint64, _vp]),
    ("tsf_snapshot_write", C.c_int, [C.c_char_p, C.c_int64, _vp, _vp, C.c_int, _vp, _vp, _vp,
                                     _vp, C.c_uint32, _vp]),
    ("tsf_snapshot_info", C.c_int, [C.c_char_p, _i64p, C.POINTER(C.c_int),
                                    C.POINTER(C.c_uint32), _vp]),
    ("tsf_snapshot_read", C.c_int, [C.c_char_p, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("tsf_create", C.c_int, [_vp, C.c_int, _pp]),
    ("tsf_destroy", None, [_vp]),
    ("tsf_stream", _vp, [_vp]),
    ("tsf_set_system", C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, _vp]),
    ("tsf_set_positions", C.c_int, [_vp, _vp]),
    ("tsf_get_positions", C.c_int, [_vp, _vp]),
    ("tsf_build_neighbor_list", C.c_int, [_vp, _d, _d]),
    ("tsf_set_neighbor_list", C.c_int, [_vp, _vp, _vp, _d, _d]),
    ("tsf_needs_rebuild", C.c_int, [_vp, C.POINTER(C.c_int)]),
    ("tsf_neighbor_entries", C.c_int64, [_vp, C.c_int]),
    ("tsf_export_neighbors", C.c_int, [_vp, C.c_int, _vp, _vp, C.c_int64]),
    ("tsf_compute_f64", C.c_int, [_vp, C.c_uint32, _vp, _vp, _vp]),
    ("tsf_compute_mixed", C.c_int, [_vp, C.c_uint32, _vp, _vp, _vp]),
    ("tsf_compute_f32", C.c_int, [_vp, C.c_uint32, _vp, _vp, _vp]),
    ("tsf_evaluate_forces", C.c_int, [_vp, C.c_int, C.c_int64, _vp, _vp, _vp, _vp, _d,
                                      C.c_uint32, _vp, _vp, _vp]),
    ("tsf_math_probe", C.c_int, [_vp, C.c_int, C.c_int64, _vp, _vp]),
    ("tsf_launch_count", C.c_int64, [_vp]),
    ("tsf_near_refreshes", C.c_int64, [_vp]),
    ("tsf_profile_enable", C.c_int, [_vp, C.c_int]),
    ("tsf_profile_read", C.c_int, [_vp, _vp, _i64p, C.c_int]),
    ("tsf_set_stream", C.c_int, [_vp, _vp]),
    ("tsf_set_owned", C.c_int, [_vp, C.c_int64]),
    ("tsf_set_centers", C.c_int, [_vp, C.c_int64, C.c_int64]),
    ("tsf_set_interior", C.c_int, [_vp, C.c_int64]),
    ("tsf_compute_phase", C.c_int, [_vp, C.c_int, C.c_uint32, C.c_int]),
    ("tsf_gather_positions", C.c_int, [_vp, _vp, C.c_int64, _vp]),
    ("tsf_scatter_positions", C.c_int, [_vp, C.c_int64, C.c_int64, _vp]),
    ("tsf_gather_forces", C.c_int, [_vp, C.c_int64, C.c_int64, _vp]),
    ("tsf_add_forces", C.c_int, [_vp, _vp, C.c_int64, _vp]),
    ("tsf_results_device", C.c_int, [_vp, _vp, _vp]),
    ("tsf_dd_error_message", C.c_char_p, []),
    ("tsf_dd_nccl_unique_id", C.c_int, [_vp]),
    ("tsf_dd_create_nccl", C.c_int, [_vp, C.c_int, C.c_int, _vp, _d, _d, _vp, _vp, _vp,
                                     C.c_uint32, _pp]),
    ("tsf_dd_group_create", C.c_int, [C.c_int, _pp]),
    ("tsf_dd_group_destroy", None, [_vp]),
    ("tsf_dd_create_local", C.c_int, [_vp, _vp, C.c_int, _d, _d, _vp, _vp, _vp, C.c_uint32,
                                      _pp]),
    ("tsf_dd_destroy", None, [_vp]),
    ("tsf_dd_setup", C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, _vp]),
    ("tsf_dd_evaluate", C.c_int, [_vp, C.c_int, C.c_uint32]),
    ("tsf_dd_rebuild", C.c_int, [_vp]),
    ("tsf_dd_md_run", C.c_int, [_vp, C.c_int, C.c_int64, _d, C.c_uint32, C.c_int, _vp,
                                C.c_int64, _i64p, _i64p]),
    ("tsf_dd_set_positions", C.c_int, [_vp, _vp]),
    ("tsf_dd_counts", C.c_int, [_vp, _vp]),
    ("tsf_dd_results", C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    ("tsf_md_scale_velocities", C.c_int, [_vp, C.c_double]),
    ("tsf_md_kick", C.c_int, [_vp, _d, C.c_int, C.c_int, C.POINTER(C.c_int)]),
    ("tsf_md_kinetic", C.c_int, [_vp, _dptr]),
    ("tsf_md_set_state", C.c_int, [_vp, _vp, _vp]),
    ("tsf_md_get_state", C.c_int, [_vp, _vp, _vp]),
    ("tsf_md_run", C.c_int, [_vp, C.c_int, C.c_int64, _d, C.c_uint32, C.c_int, _vp, C.c_int64,
                             _i64p, _i64p]),
]


def lib():
    """The loaded extension (builds it on first use if absent)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                try:
                    build()
                except Exception as exc:  # noqa: BLE001
                    raise ImportError(
                        f"paper_1607_02904_b200: CUDA extension {LIB_PATH} is missing and could "
                        f"not be built ({exc}); there is no CPU fallback") from exc
            L = C.CDLL(LIB_PATH)
            for name, res, args in PROTOTYPES:
                # an alternative build (TSF_LIBRARY, A/B experiments) may predate a symbol
                if os.environ.get("TSF_LIBRARY") and not hasattr(L, name):
                    continue
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib
