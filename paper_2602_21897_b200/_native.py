"""ctypes binding of libtw_hpccg.so (include/tw_hpccg.h).

The shared library is built in-tree by ``paper_2602_21897_b200/csrc/Makefile``
(``__graft_entry__.build()``).  There is no fallback: if the library is
missing, importing the bound functions raises ``NativeLibraryMissing``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libtw_hpccg.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "tw_hpccg.h")

TW_OK, TW_ERR_CONFIG, TW_ERR_CONTRACT, TW_ERR_CUDA, TW_ERR_NCCL = 0, 1, 2, 3, 4
TW_CG_MONOLITHIC, TW_CG_TASKS = 0, 1
TW_DISPATCH_STREAMS, TW_DISPATCH_PERSISTENT, TW_DISPATCH_AUTO, TW_DISPATCH_CHAIN = 0, 1, 2, 3
TW_K1_REGISTER, TW_K1_TMA_GATHER, TW_K1_STAGED, TW_K1_STAGED_TABLE = 0, 1, 2, 3
TW_TRANSPORT_NONE, TW_TRANSPORT_NCCL, TW_TRANSPORT_PEER, TW_TRANSPORT_LOOPBACK = 0, 1, 2, 3
TW_XUPD_AUTO, TW_XUPD_K2, TW_XUPD_K3, TW_XUPD_K3_PAIRS = 0, 1, 2, 3
TW_L2KEEP_AUTO, TW_L2KEEP_ON, TW_L2KEEP_OFF = 0, 1, 2


class NativeLibraryMissing(ImportError):
    pass


class TwError(RuntimeError):
    code = -1


class ConfigError(TwError):
    """Malformed input: the reference's tw::ConfigError (types.hpp:30-33)."""
    code = TW_ERR_CONFIG


class ContractViolation(TwError):
    """API misuse: the reference's tw::ContractViolation (types.hpp:23-26)."""
    code = TW_ERR_CONTRACT


class CudaError(TwError):
    code = TW_ERR_CUDA


class NcclError(TwError):
    code = TW_ERR_NCCL


_ERRS = {1: ConfigError, 2: ContractViolation, 3: CudaError, 4: NcclError}

i64 = C.c_int64
vp = C.c_void_p
dp = C.POINTER(C.c_double)
DONE_CB = C.CFUNCTYPE(None, C.c_void_p)  # tw_event_bind_async callback
lp = C.POINTER(C.c_int64)


class EllInfo(C.Structure):
    _fields_ = [("nx", i64), ("ny", i64), ("nz", i64), ("z_begin", i64), ("z_end", i64),
                ("n_global", i64), ("n_rows", i64), ("row_offset", i64), ("col_offset", i64),
                ("x_len", i64), ("nnz", i64), ("n_slices", i64), ("ell_entries", i64),
                ("max_width", C.c_int32), ("slice_rows", C.c_int32)]


class SlabPlan(C.Structure):
    _fields_ = [(k, i64) for k in ("nx", "ny", "nz", "z_begin", "z_end", "plane", "n_rows",
                                   "row_offset", "col_offset", "x_len", "diag_shift", "nnz",
                                   "interior_r0", "interior_r1", "send_lo", "recv_lo",
                                   "send_hi", "recv_hi")] + [("ghost_lo", C.c_int32),
                                                             ("ghost_hi", C.c_int32)]


class CgOptionsC(C.Structure):
    _fields_ = [("variant", C.c_int), ("tiles", C.c_int), ("stream_pool_capacity", C.c_uint),
                ("use_graph", C.c_int), ("iteration_marks", C.c_int), ("tol", C.c_double),
                ("dispatch", C.c_int), ("x_update", C.c_int), ("l2_keep", C.c_int),
                ("dag_spmv_slices", C.c_int64), ("dag_vec_rows", C.c_int64)]


class CgMode(C.Structure):
    _fields_ = [(k, C.c_int32) for k in ("variant", "tiles", "dispatch", "use_graph", "k1_form",
                                         "k1_l2_keep", "x_in_k3", "transport", "nranks",
                                         "kernels_per_iteration", "collectives_per_iteration")]


TW_K1_NAMES = {0: "spmv_kernel (register path)", 1: "spmv_tma_kernel (TMA matrix, gathered x)",
               2: "spmv_tma_staged_kernel (closed-form x runs)",
               3: "spmv_tma_staged_kernel (run-table x runs)"}


# (name, restype, argtypes) for every symbol include/tw_hpccg.h declares.
SIGNATURES = [
    ("tw_last_error_string", C.c_char_p, []),
    ("tw_abi_version", C.c_int, []),
    ("tw_ctx_create", C.c_int, [C.c_int, C.c_uint, C.POINTER(vp)]),
    ("tw_ctx_destroy", C.c_int, [vp]),
    ("tw_ctx_compute_stream", C.c_int, [vp, C.POINTER(vp)]),
    ("tw_ctx_synchronize", C.c_int, [vp]),
    ("tw_ctx_device_info", C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("tw_comm_unique_id", C.c_int, [C.c_char_p]),
    ("tw_ctx_init_comm", C.c_int, [vp, C.c_int, C.c_int, C.c_char_p]),
    ("tw_ctx_comm_info", C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("tw_ctx_init_emulated_rank", C.c_int, [vp, C.c_int, C.c_int]),
    ("tw_malloc", C.c_int, [vp, C.POINTER(vp), i64]),
    ("tw_free", C.c_int, [vp, vp]),
    ("tw_malloc_host", C.c_int, [C.POINTER(vp), i64]),
    ("tw_free_host", C.c_int, [vp]),
    ("tw_memcpy", C.c_int, [vp, vp, vp, i64, vp]),
    ("tw_slab_plan", C.c_int, [i64, i64, i64, i64, i64, C.POINTER(SlabPlan)]),
    ("tw_slab_partition", C.c_int, [i64, C.c_int, C.c_int, lp, lp]),
    ("tw_gen_stencil_ell", C.c_int, [vp, i64, i64, i64, i64, i64, C.POINTER(vp)]),
    ("tw_ell_from_csr", C.c_int, [vp, i64, lp, lp, dp, C.POINTER(vp)]),
    ("tw_ell_info", C.c_int, [vp, C.POINTER(EllInfo)]),
    ("tw_ell_to_csr", C.c_int, [vp, lp, lp, dp]),
    ("tw_ell_to_csr_rows", C.c_int, [vp, i64, i64, C.c_int, lp, lp, dp]),
    ("tw_ell_destroy", C.c_int, [vp]),
    ("tw_spmv_range", C.c_int, [vp, vp, vp, i64, i64, vp]),
    ("tw_spmv_dot", C.c_int, [vp, vp, vp, i64, i64, vp, vp]),
    ("tw_dot_range", C.c_int, [vp, vp, vp, i64, i64, vp, vp]),
    ("tw_waxpby_range", C.c_int, [vp, C.c_double, vp, C.c_double, vp, vp, i64, i64, vp]),
    ("tw_make_tile_plan", C.c_int, [vp, C.c_int, lp, lp, lp, lp]),
    ("tw_rhs_xorshift", C.c_int, [vp, C.c_uint64, i64, i64, vp, vp]),
    ("tw_rhs_splitmix", C.c_int, [vp, C.c_uint64, i64, i64, vp, vp]),
    ("tw_cg_options_default", None, [C.POINTER(CgOptionsC)]),
    ("tw_cg_create", C.c_int, [vp, vp, C.POINTER(CgOptionsC), C.c_int, C.POINTER(vp)]),
    ("tw_cg_destroy", C.c_int, [vp]),
    ("tw_cg_set_rhs", C.c_int, [vp, vp, C.c_int]),
    ("tw_cg_iterate", C.c_int, [vp, C.c_int]),
    ("tw_cg_wait", C.c_int, [vp]),
    ("tw_cg_iterations_done", C.c_int, [vp, C.POINTER(C.c_int)]),
    ("tw_cg_history", C.c_int, [vp, dp, C.c_int]),
    ("tw_cg_solution", C.c_int, [vp, dp]),
    ("tw_cg_vectors", C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]),
    ("tw_cg_iteration_marks", C.c_int, [vp, dp, C.c_int]),
    ("tw_cg_iteration_times", C.c_int, [vp, dp, C.c_int]),
    ("tw_cg_task_edges", C.c_int, [vp, C.c_char_p, i64, C.POINTER(i64)]),
    ("tw_cg_enable_kernel_timing", C.c_int, [vp, C.c_int]),
    ("tw_cg_kernel_times", C.c_int, [vp, dp, dp, dp, C.POINTER(C.c_int)]),
    ("tw_task_dag_edges", C.c_int, [i64, C.c_int, lp, lp, lp, lp, i64, i64, C.c_int, C.c_int,
                                    C.c_int, C.c_char_p, i64, C.POINTER(i64)]),
    ("tw_cg_launches_per_iteration", C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("tw_cg_mode", C.c_int, [vp, C.POINTER(CgMode)]),
    ("tw_cg_group_set_rhs", C.c_int, [C.POINTER(vp), C.c_int, C.POINTER(vp), C.c_int]),
    ("tw_cg_group_iterate", C.c_int, [C.POINTER(vp), C.c_int, C.c_int]),
    ("tw_halo_exchange", C.c_int, [vp, vp, vp]),
    ("tw_ell_x_staged", C.c_int, [vp, C.POINTER(C.c_int)]),
    ("tw_ell_set_x_staged", C.c_int, [vp, C.c_int, C.POINTER(C.c_int)]),
    ("tw_update_xr_rr", C.c_int, [vp, vp, vp, vp, vp, vp, i64, i64, vp, vp]),
    ("tw_update_p", C.c_int, [vp, vp, vp, vp, i64, i64, vp]),
    ("tw_stream_acquire", C.c_int, [vp, C.POINTER(vp)]),
    ("tw_stream_release", C.c_int, [vp, vp]),
    ("tw_event_create", C.c_int, [C.POINTER(vp)]),
    ("tw_event_destroy", C.c_int, [vp]),
    ("tw_event_record", C.c_int, [vp, vp]),
    ("tw_event_query", C.c_int, [vp, C.POINTER(C.c_int)]),
    ("tw_event_wait", C.c_int, [vp, vp]),
    ("tw_stream_wait_event", C.c_int, [vp, vp]),
    ("tw_event_bind_async", C.c_int, [vp, vp, DONE_CB, vp]),
    ("tw_cg_group_enable_peer", C.c_int, [C.POINTER(vp), C.c_int]),
    ("tw_cg_group_iterate_concurrent", C.c_int, [C.POINTER(vp), C.c_int, C.c_int, C.c_int]),
    ("tw_cg_peer_export", C.c_int, [vp, C.c_char_p]),
    ("tw_cg_peer_connect", C.c_int, [vp, C.c_char_p]),
    ("tw_cg_peer_ping_send", C.c_int, [vp]),
    ("tw_cg_peer_ping_check", C.c_int, [vp, C.c_int, C.POINTER(C.c_int)]),
    ("tw_cg_solve", C.c_int, [vp, vp, vp, C.c_int, C.POINTER(CgOptionsC), dp, dp,
                              C.POINTER(C.c_int)]),
]

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libtw_hpccg.so once; raise loudly when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("TW_HPCCG_LIB", path)  # tuning variants built by scripts/
    if not os.path.exists(path):
        raise NativeLibraryMissing(
            f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the HPCCG path)")
    lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != TW_OK:
        msg = load().tw_last_error_string().decode(errors="replace")
        raise _ERRS.get(rc, TwError)(msg)


HEADERS = (HEADER, os.path.join(os.path.dirname(HEADER), "tw_hpccg_emulation.h"))


def declared_symbols(headers=HEADERS) -> list[str]:
    """Every function name include/tw_hpccg.h and tw_hpccg_emulation.h declare."""
    import re
    if isinstance(headers, str):
        headers = (headers,)
    text = "".join(open(h).read() for h in headers)
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tw_[a-z0-9_]+)\s*\(", text)))
