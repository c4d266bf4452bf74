"""B200-native HPCCG conjugate-gradient hot path (arXiv 2602.21897 artifact).

Hand-written sm_100a CUDA kernels and a C++ host runtime in
``_lib/libtw_hpccg.so`` behind the C ABI ``include/tw_hpccg.h``; this package
is the Python face that mirrors the reference's operator API
(``hpccg.py``).  There is no CPU fallback.
"""
from . import _native
from .hpccg import (CgBackend, CgOptions, CgResult, CgSolver, ConfigError, ContractViolation,
                    CudaError, EllMatrix, EmulatedRankGroup, Event, NcclError, Runtime, Tile,
                    cg_monolithic, cg_solve, cg_tasks, default_runtime, dot_range, dump_csr,
                    ell_from_csr, gen_stencil_matrix, halo_exchange, load_csr, make_tile_plan,
                    parse_csr, rhs_splitmix, rhs_xorshift, slab_partition, slab_plan, spmv_dot,
                    spmv_range, task_dag_edges, update_p, update_xr_rr, waxpby_range)

__all__ = [
    "CgBackend", "CgOptions", "CgResult", "CgSolver", "ConfigError", "ContractViolation",
    "CudaError", "EllMatrix", "EmulatedRankGroup", "Event", "NcclError", "Runtime", "Tile",
    "cg_monolithic", "cg_solve", "cg_tasks", "default_runtime", "dot_range", "dump_csr",
    "ell_from_csr", "gen_stencil_matrix", "halo_exchange", "load_csr", "make_tile_plan",
    "parse_csr", "rhs_splitmix", "rhs_xorshift", "slab_partition", "slab_plan", "spmv_dot",
    "spmv_range", "task_dag_edges", "update_p", "update_xr_rr", "waxpby_range",
    "_native",
]
