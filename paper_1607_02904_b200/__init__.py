"""B200-native Tersoff force/energy path (arXiv 1607.02904), drop-in for the
reference's ``evaluate_forces`` (proj/include/tmd/potential_opt.hpp:105-106).

The compute path is ``libtersoff_b200.so`` (hand-written sm_100a CUDA behind the
C-ABI in ``include/tersoff_b200.h``); this package is a thin ctypes surface
shaped like the reference's ``tersoffmd`` Python module.
"""
from .api import (  # noqa: F401
    AtomSystem,
    ConfigError,
    Context,
    CudaError,
    NeighborList,
    NumericError,
    ParamTable,
    ParseError,
    SimulationBox,
    build_neighbor_list,
    builtin_silicon,
    evaluate_forces,
    init_velocities,
    kinetic_energy,
    load_params,
    make_diamond_lattice,
    melt,
    needs_rebuild,
    parse_params,
    perturbed_lattice,
    run_nve,
    load_snapshot,
    save_snapshot,
    snapshot_info,
    temperature,
    total_momentum,
)
from ._lib import LIB_PATH, build  # noqa: F401

__version__ = "0.1.0"
