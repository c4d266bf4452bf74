"""Reference-facing host API of the B200 HPCCG path.

Mirrors the reference's operator interface (proj/include/taskweave/
{csr,kernels,cg}.hpp) with the same names, argument meaning and error
behaviour, over the C ABI of ``include/tw_hpccg.h``:

==========================  =====================================================
reference                   here
==========================  =====================================================
``Runtime`` (runtime.hpp)   ``Runtime`` -- device context, compute stream, stream
                            pool (QueuePool capacity), optional NCCL communicator
``CsrMatrix`` (csr.hpp)     ``EllMatrix`` -- sliced ELL resident in HBM
``gen_stencil_matrix``      ``gen_stencil_matrix(nx, ny, nz, rt=None, ...)``
``spmv_range``              ``spmv_range(A, x, y, r0, r1)``
``dot_range``               ``dot_range(a, b, i0, i1)``
``waxpby_range``            ``waxpby_range(alpha, x, beta, y, w, i0, i1)``
``make_tile_plan``          ``make_tile_plan(A, tiles)``
``cg_monolithic``           ``cg_monolithic(rt, A, b, iterations, opt)``
``cg_tasks``                ``cg_tasks(rt, A, b, iterations, opt)``
``CgOptions`` / ``CgResult``  same fields (``backend`` is always the CUDA device)
==========================  =====================================================

Vectors handed to the kernel functions are device buffers: torch CUDA float64
tensors, or ``DeviceBuffer`` objects from ``Runtime.alloc``.  Errors raise
``ConfigError`` (bad input) or ``ContractViolation`` (API misuse), as the
reference's exceptions do.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Any

import numpy as np

from . import _native as N
from ._native import ConfigError, ContractViolation, CudaError, NcclError  # noqa: F401


def _lib():
    return N.load()


def _ptr(v: Any) -> int:
    """Device pointer of a torch tensor / DeviceBuffer / int."""
    if v is None:
        return 0
    if isinstance(v, int):
        return v
    if hasattr(v, "data_ptr"):
        if getattr(v, "dtype", None) is not None and "float64" not in str(v.dtype) and \
                "int" not in str(v.dtype):
            raise ContractViolation(f"expected a float64 device tensor, got {v.dtype}")
        if hasattr(v, "is_cuda") and not v.is_cuda:
            raise ContractViolation("expected a CUDA tensor")
        return int(v.data_ptr())
    if isinstance(v, DeviceBuffer):
        return v.ptr
    raise ContractViolation(f"not a device buffer: {type(v)!r}")


class DeviceBuffer:
    """Raw device allocation owned by a Runtime (for callers without torch)."""

    def __init__(self, rt: "Runtime", nbytes: int):
        self.rt, self.nbytes = rt, nbytes
        p = C.c_void_p()
        N.check(_lib().tw_malloc(rt.h, C.byref(p), nbytes))
        self.ptr = int(p.value or 0)

    def __del__(self):
        try:
            if getattr(self, "ptr", 0) and self.rt.h:
                _lib().tw_free(self.rt.h, C.c_void_p(self.ptr))
                self.ptr = 0
        except Exception:
            pass

    def upload(self, arr: np.ndarray) -> "DeviceBuffer":
        arr = np.ascontiguousarray(arr)
        if arr.nbytes > self.nbytes:
            raise ContractViolation("upload larger than the buffer")
        N.check(_lib().tw_memcpy(self.rt.h, C.c_void_p(self.ptr), arr.ctypes.data_as(C.c_void_p),
                                 arr.nbytes, None))
        self.rt.synchronize()
        return self

    def download(self, dtype=np.float64, count: int | None = None) -> np.ndarray:
        count = self.nbytes // np.dtype(dtype).itemsize if count is None else count
        out = np.empty(count, dtype)
        self.rt.synchronize()
        N.check(_lib().tw_memcpy(self.rt.h, out.ctypes.data_as(C.c_void_p), C.c_void_p(self.ptr),
                                 out.nbytes, None))
        self.rt.synchronize()
        return out


class Runtime:
    """Device context: the tw::Runtime + sim::Device pair of the reference
    (runtime.hpp:25-55, sim_device.hpp:91-166) on a real B200."""

    def __init__(self, device: int = 0, stream_pool_capacity: int = 4):
        h = C.c_void_p()
        N.check(_lib().tw_ctx_create(device, stream_pool_capacity, C.byref(h)))
        self.h = h
        self.device = device
        s = C.c_void_p()
        N.check(_lib().tw_ctx_compute_stream(self.h, C.byref(s)))
        self.compute_stream = int(s.value or 0)

    def acquire_stream(self) -> int:
        """QueuePool::acquire: a pooled stream (blocks while all are out)."""
        s = C.c_void_p()
        N.check(_lib().tw_stream_acquire(self.h, C.byref(s)))
        return int(s.value or 0)

    def release_stream(self, stream: int) -> None:
        N.check(_lib().tw_stream_release(self.h, C.c_void_p(stream)))

    def close(self):
        if getattr(self, "h", None):
            N.check(_lib().tw_ctx_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def synchronize(self):
        N.check(_lib().tw_ctx_synchronize(self.h))

    @property
    def sm_count(self) -> int:
        d, s = C.c_int(), C.c_int()
        N.check(_lib().tw_ctx_device_info(self.h, C.byref(d), C.byref(s)))
        return s.value

    def alloc(self, count: int, dtype=np.float64) -> DeviceBuffer:
        return DeviceBuffer(self, int(count) * np.dtype(dtype).itemsize)

    # multi-GPU
    @staticmethod
    def comm_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        N.check(_lib().tw_comm_unique_id(buf))
        return buf.raw

    def init_comm(self, rank: int, nranks: int, uid: bytes | None):
        uid = uid if uid is not None else bytes(128)
        N.check(_lib().tw_ctx_init_comm(self.h, rank, nranks, C.c_char_p(uid)))

    def init_emulated_rank(self, rank: int, nranks: int):
        """Make this context emulated rank `rank` of an `nranks` group on one
        device (tw_ctx_init_emulated_rank); see EmulatedRankGroup."""
        N.check(_lib().tw_ctx_init_emulated_rank(self.h, rank, nranks))

    @property
    def rank(self) -> int:
        r, n = C.c_int(), C.c_int()
        N.check(_lib().tw_ctx_comm_info(self.h, C.byref(r), C.byref(n)))
        return r.value

    @property
    def nranks(self) -> int:
        r, n = C.c_int(), C.c_int()
        N.check(_lib().tw_ctx_comm_info(self.h, C.byref(r), C.byref(n)))
        return n.value


_default_rt: Runtime | None = None


def default_runtime() -> Runtime:
    global _default_rt
    if _default_rt is None:
        _default_rt = Runtime(0)
    return _default_rt




class Event:
    """A device event with the reference's record / query / wait and the
    task-aware bind_event_async (tw_event_*)."""

    def __init__(self):
        h = C.c_void_p()
        N.check(_lib().tw_event_create(C.byref(h)))
        self.h = h
        self._cbs = []  # keep bound callbacks alive until they fire

    def record(self, stream: int) -> None:
        N.check(_lib().tw_event_record(self.h, C.c_void_p(stream)))

    def query(self) -> bool:
        d = C.c_int()
        N.check(_lib().tw_event_query(self.h, C.byref(d)))
        return bool(d.value)

    def wait(self, rt: Runtime) -> None:
        N.check(_lib().tw_event_wait(rt.h, self.h))

    def block_stream(self, stream: int) -> None:
        """Later work on `stream` waits for this event (device edge)."""
        N.check(_lib().tw_stream_wait_event(C.c_void_p(stream), self.h))

    def bind_async(self, rt: Runtime, done) -> None:
        """done() runs on the context's polling thread once the event completes."""
        cb = N.DONE_CB(lambda _arg: done())
        self._cbs.append(cb)
        N.check(_lib().tw_event_bind_async(rt.h, self.h, cb, None))

    def close(self):
        if getattr(self, "h", None):
            N.check(_lib().tw_event_destroy(self.h))
            self.h = None


@dataclass
class Tile:
    """tw::bench::Tile (cg.hpp:55-62); band in global columns."""
    r0: int
    r1: int
    band_lo: int
    band_hi: int


class EllMatrix:
    """The device-resident replacement of CsrMatrix (csr.hpp:9-17)."""

    def __init__(self, rt: Runtime, handle: C.c_void_p):
        self.rt, self.h = rt, handle
        info = N.EllInfo()
        N.check(_lib().tw_ell_info(self.h, C.byref(info)))
        self.info = info

    def __del__(self):
        try:
            if getattr(self, "h", None) and getattr(self.rt, "h", None):
                _lib().tw_ell_destroy(self.h)
                self.h = None
        except Exception:
            pass

    @property
    def n(self) -> int:
        """Rows owned by this rank (all rows on one GPU)."""
        return int(self.info.n_rows)

    @property
    def n_global(self) -> int:
        return int(self.info.n_global)

    def nnz(self) -> int:
        return int(self.info.nnz)

    @property
    def x_len(self) -> int:
        return int(self.info.x_len)

    @property
    def x_staged(self) -> bool:
        """The single-domain CG's K1 reads this matrix in its x-staged form."""
        v = C.c_int()
        N.check(_lib().tw_ell_x_staged(self.h, C.byref(v)))
        return bool(v.value)

    def set_x_staged(self, enable: bool) -> bool:
        """Build or drop the x-staged form (K1's 16-bit columns); returns
        whether the matrix carries it afterwards."""
        v = C.c_int()
        N.check(_lib().tw_ell_set_x_staged(self.h, int(enable), C.byref(v)))
        return bool(v.value)

    def to_csr(self):
        """(row_ptr int64[n+1], col_idx int64[nnz], values f64[nnz]), global columns."""
        n, nnz = self.n, self.nnz()
        rp = np.empty(n + 1, np.int64)
        ci = np.empty(nnz, np.int64)
        va = np.empty(nnz, np.float64)
        N.check(_lib().tw_ell_to_csr(self.h, rp.ctypes.data_as(N.lp), ci.ctypes.data_as(N.lp),
                                     va.ctypes.data_as(N.dp)))
        return rp, ci, va

    def to_csr_rows(self, r0: int, r1: int, staged: bool = False):
        """Rows [r0, r1) as (row_ptr relative to r0, col_idx global, values);
        staged=True decodes the 16-bit x-staged columns the CG's K1 reads."""
        cap = self.info.max_width * (r1 - r0)
        rp = np.empty(r1 - r0 + 1, np.int64)
        ci = np.empty(cap, np.int64)
        va = np.empty(cap, np.float64)
        N.check(_lib().tw_ell_to_csr_rows(self.h, r0, r1, int(staged), rp.ctypes.data_as(N.lp),
                                          ci.ctypes.data_as(N.lp), va.ctypes.data_as(N.dp)))
        k = int(rp[-1])
        return rp, ci[:k], va[:k]

    def validate(self):
        """CsrMatrix::validate (csr.cpp:13-27) on the converted structure."""
        rp, ci, _ = self.to_csr()
        if rp[0] != 0 or np.any(np.diff(rp) < 0) or rp[-1] != len(ci):
            raise ConfigError("ell: row structure inconsistent")
        if len(ci) and (ci.min() < 0 or ci.max() >= self.n_global):
            raise ConfigError("ell: column index out of range")


def gen_stencil_matrix(nx: int, ny: int, nz: int, rt: Runtime | None = None,
                       z_begin: int = 0, z_end: int | None = None) -> EllMatrix:
    """gen_stencil_matrix (csr.cpp:29-59), generated on the device."""
    rt = rt or default_runtime()
    h = C.c_void_p()
    N.check(_lib().tw_gen_stencil_ell(rt.h, nx, ny, nz, z_begin, nz if z_end is None else z_end,
                                      C.byref(h)))
    return EllMatrix(rt, h)


def ell_from_csr(row_ptr, col_idx, values, rt: Runtime | None = None) -> EllMatrix:
    """CsrMatrix (host arrays) -> device ELL; validation as csr.cpp:13-27."""
    rt = rt or default_runtime()
    rp = np.ascontiguousarray(row_ptr, np.int64)
    ci = np.ascontiguousarray(col_idx, np.int64)
    va = np.ascontiguousarray(values, np.float64)
    if len(ci) != len(va):
        raise ConfigError("csr: row_ptr[n] disagrees with stored entries")
    if len(rp) < 1:
        raise ConfigError("csr: row_ptr must hold n+1 offsets")
    if rp[-1] != len(ci):
        raise ConfigError("csr: row_ptr[n] disagrees with stored entries")
    h = C.c_void_p()
    N.check(_lib().tw_ell_from_csr(rt.h, len(rp) - 1, rp.ctypes.data_as(N.lp),
                                   ci.ctypes.data_as(N.lp), va.ctypes.data_as(N.dp), C.byref(h)))
    return EllMatrix(rt, h)


CSR_HEADER = "# taskweave csr v1"


def dump_csr(A: "EllMatrix | tuple", out=None) -> str:
    """dump_csr (csr.cpp:61-74): header, "n nnz", then row_ptr, col_idx and
    values lines, doubles at 17 significant digits (round-trips exactly).
    ``A`` is a device EllMatrix or a (row_ptr, col_idx, values) tuple."""
    rp, ci, va = A.to_csr() if isinstance(A, EllMatrix) else A
    lines = [CSR_HEADER, f"{len(rp) - 1} {int(rp[-1])}",
             " ".join(str(int(v)) for v in rp), " ".join(str(int(v)) for v in ci),
             " ".join("%.17g" % v for v in va)]
    text = "\n".join(lines) + "\n"
    if out is not None:
        out.write(text)
    return text


def parse_csr(text: str):
    """load_csr's parser + CsrMatrix::validate (csr.cpp:13-27, 76-98) on the
    host: returns (row_ptr, col_idx, values); ConfigError on bad input."""
    head, _, rest = text.partition("\n")
    if head.rstrip("\r") != CSR_HEADER:
        raise ConfigError("csr load: missing 'taskweave csr v1' header")
    tok = rest.split()
    try:
        n, nnz = int(tok[0]), int(tok[1])
    except (IndexError, ValueError):
        raise ConfigError("csr load: bad size line") from None
    if n < 0 or nnz < 0:
        raise ConfigError("csr: row_ptr must hold n+1 offsets")
    pos = 2

    def take(count, conv, what):
        nonlocal pos
        if pos + count > len(tok):
            raise ConfigError(f"csr load: truncated {what}")
        try:
            vals = [conv(t) for t in tok[pos:pos + count]]
        except ValueError:
            raise ConfigError(f"csr load: truncated {what}") from None
        pos += count
        return vals
    rp = np.array(take(n + 1, int, "row_ptr"), np.int64)
    ci = np.array(take(nnz, int, "col_idx"), np.int64)
    va = np.array(take(nnz, float, "values"), np.float64)
    if rp[0] != 0:
        raise ConfigError("csr: row_ptr must start at 0")
    bad = np.nonzero(np.diff(rp) < 0)[0]
    if len(bad):
        raise ConfigError(f"csr: row_ptr decreases at row {int(bad[0])}")
    if rp[-1] != nnz:
        raise ConfigError("csr: row_ptr[n] disagrees with stored entries")
    if nnz and (ci.min() < 0 or ci.max() >= n):
        c = int(ci[(ci < 0) | (ci >= n)][0])
        raise ConfigError(f"csr: column index {c} out of range")
    return rp, ci, va


def load_csr(src, rt: "Runtime | None" = None) -> "EllMatrix":
    """load_csr (csr.cpp:76-98) straight into a device EllMatrix."""
    text = src if isinstance(src, str) else src.read()
    rp, ci, va = parse_csr(text)
    return ell_from_csr(rp, ci, va, rt=rt)


def spmv_range(A: EllMatrix, x, y, r0: int, r1: int, stream: int | None = None) -> None:
    """y[r0:r1] = A x over local rows (kernels.cpp:5-13); bit-identical."""
    N.check(_lib().tw_spmv_range(A.h, C.c_void_p(_ptr(x)), C.c_void_p(_ptr(y)), r0, r1,
                                 C.c_void_p(stream or 0)))


def spmv_dot(A: EllMatrix, p, Ap, r0: int, r1: int, stream: int | None = None) -> float:
    """Fused K1: Ap = A p on [r0, r1) and returns p.Ap over the same rows."""
    out = A.rt.alloc(1)
    N.check(_lib().tw_spmv_dot(A.h, C.c_void_p(_ptr(p)), C.c_void_p(_ptr(Ap)), r0, r1,
                               C.c_void_p(out.ptr), C.c_void_p(stream or 0)))
    return float(out.download()[0])


def halo_exchange(A: EllMatrix, x, stream: int | None = None) -> None:
    """exchange_externals: ghost planes of the slab vector x (x_len
    entries) from the neighbouring ranks (NCCL, collective)."""
    N.check(_lib().tw_halo_exchange(A.h, C.c_void_p(_ptr(x)), C.c_void_p(stream or 0)))


def update_xr_rr(alpha: float, x, p, r, Ap, i0: int, i1: int, rt: Runtime | None = None) -> float:
    """Fused K2 standalone: x += alpha p; r -= alpha Ap on [i0, i1); returns
    r.r over the range (alpha staged in a device scalar)."""
    rt = rt or default_runtime()
    sc = rt.alloc(2)
    sc.upload(np.array([alpha, 0.0]))
    N.check(_lib().tw_update_xr_rr(rt.h, C.c_void_p(sc.ptr), C.c_void_p(_ptr(x)), C.c_void_p(_ptr(p)),
                                   C.c_void_p(_ptr(r)), C.c_void_p(_ptr(Ap)), i0, i1,
                                   C.c_void_p(sc.ptr + 8), None))
    return float(sc.download()[1])


def update_p(beta: float, r, p, i0: int, i1: int, rt: Runtime | None = None) -> None:
    """Fused K3 standalone: p = r + beta p on [i0, i1)."""
    rt = rt or default_runtime()
    sc = rt.alloc(1)
    sc.upload(np.array([beta]))
    N.check(_lib().tw_update_p(rt.h, C.c_void_p(sc.ptr), C.c_void_p(_ptr(r)), C.c_void_p(_ptr(p)),
                               i0, i1, None))
    rt.synchronize()


def dot_range(a, b, i0: int, i1: int, rt: Runtime | None = None) -> float:
    """dot_range (kernels.cpp:15-20) as a fixed-order device reduction."""
    rt = rt or default_runtime()
    out = rt.alloc(1)
    N.check(_lib().tw_dot_range(rt.h, C.c_void_p(_ptr(a)), C.c_void_p(_ptr(b)), i0, i1,
                                C.c_void_p(out.ptr), None))
    return float(out.download()[0])


def waxpby_range(alpha: float, x, beta: float, y, w, i0: int, i1: int,
                 rt: Runtime | None = None) -> None:
    """w = alpha x + beta y on [i0, i1) (kernels.cpp:22-26); bit-identical."""
    rt = rt or default_runtime()
    N.check(_lib().tw_waxpby_range(rt.h, alpha, C.c_void_p(_ptr(x)), beta, C.c_void_p(_ptr(y)),
                                   C.c_void_p(_ptr(w)), i0, i1, None))


def make_tile_plan(A: EllMatrix, tiles: int) -> list[Tile]:
    """make_tile_plan (cg.cpp:348-370); ConfigError for tiles < 1 or > rows."""
    arrs = [np.empty(max(tiles, 1), np.int64) for _ in range(4)]
    N.check(_lib().tw_make_tile_plan(A.h, tiles, *[a.ctypes.data_as(N.lp) for a in arrs]))
    return [Tile(int(arrs[0][t]), int(arrs[1][t]), int(arrs[2][t]), int(arrs[3][t]))
            for t in range(tiles)]


def slab_plan(nx: int, ny: int, nz: int, z_begin: int, z_end: int) -> N.SlabPlan:
    """z-slab geometry of the owned planes [z_begin, z_end) (host only)."""
    out = N.SlabPlan()
    N.check(_lib().tw_slab_plan(nx, ny, nz, z_begin, z_end, C.byref(out)))
    return out


def slab_partition(nz: int, rank: int, nranks: int) -> tuple[int, int]:
    """Strong-scaling split: planes [nz r / R, nz (r+1) / R)."""
    a, b = C.c_int64(), C.c_int64()
    N.check(_lib().tw_slab_partition(nz, rank, nranks, C.byref(a), C.byref(b)))
    return a.value, b.value


def task_dag_edges(n_rows: int, tiles: list[Tile] | tuple, iterations: int,
                   diag_shift: int = 0, plane: int = 0, ghost_lo: bool = False,
                   ghost_hi: bool = False) -> list[tuple[str, str]]:
    """Logical block-task DAG of cg_tasks (cg.cpp:166-334) inferred on the
    host from the tasks' access regions -- the edges the reference's depsys
    records (dep_system.cpp:22-65).  ``tiles``: Tile list with bands in local
    x coordinates (== global columns on one rank)."""
    T = len(tiles)
    arrs = [np.array([getattr(t, f) for t in tiles], np.int64)
            for f in ("r0", "r1", "band_lo", "band_hi")]
    need = C.c_int64()
    args = [n_rows, T, *[a.ctypes.data_as(N.lp) for a in arrs], diag_shift, plane,
            int(ghost_lo), int(ghost_hi), iterations]
    N.check(_lib().tw_task_dag_edges(*args, None, 0, C.byref(need)))
    buf = C.create_string_buffer(int(need.value))
    N.check(_lib().tw_task_dag_edges(*args, buf, need.value, C.byref(need)))
    return [tuple(l.split()) for l in buf.value.decode().splitlines() if l]


def rhs_xorshift(rt: Runtime, n: int, seed: int = 7, first: int = 0, out=None):
    """b of acceptance.cpp:48-58 (xorshift64), generated on the device."""
    out = out if out is not None else rt.alloc(n)
    N.check(_lib().tw_rhs_xorshift(rt.h, seed, first, n, C.c_void_p(_ptr(out)), None))
    return out


def rhs_splitmix(rt: Runtime, n: int, seed: int = 7, first: int = 0, out=None):
    """b of scenario.cpp:46-55 / 91-95 (SplitMix64), generated on the device."""
    out = out if out is not None else rt.alloc(n)
    N.check(_lib().tw_rhs_splitmix(rt.h, seed, first, n, C.c_void_p(_ptr(out)), None))
    return out


# ----------------------------------------------------------------------- CG

class CgBackend:
    """CgBackend (cg.hpp:24-28) plus the real device: only ``cuda`` runs here."""
    cuda = "cuda"


@dataclass
class CgOptions:
    """CgOptions (cg.hpp:37-45) for the CUDA backend."""
    tiles: int = 16
    backend: str = CgBackend.cuda
    stream_pool_capacity: int = 4
    iteration_marks: bool = True
    tol: float = 0.0
    use_graph: bool = False
    persistent: bool = False  # tasks variant: one persistent kernel runs the whole DAG
    auto_dispatch: bool = False  # TW_DISPATCH_AUTO: chain / persistent / streams, the measured winner
    chain: bool = False  # TW_DISPATCH_CHAIN: tile kernels on one stream, programmatic launches
    # placement / tuning (no result bit changes, except the dispatcher's chunk
    # sizes, which set its chunk-order reduction tree): None = the library's choice
    x_update: str | None = None   # "k2" | "k3" | "k3_pairs": where x += alpha p runs
    l2_keep: bool | None = None   # staged K1: x runs with an L2 evict_last hint
    dag_spmv_slices: int = 0
    dag_vec_rows: int = 0

    def to_c(self, variant: int) -> N.CgOptionsC:
        if self.backend != CgBackend.cuda:
            raise ConfigError(f"backend {self.backend!r} is not available on the B200 build")
        o = N.CgOptionsC()
        o.variant = variant
        o.tiles = int(self.tiles)
        o.stream_pool_capacity = int(self.stream_pool_capacity)
        o.use_graph = 1 if self.use_graph else 0
        o.iteration_marks = 1 if self.iteration_marks else 0
        o.tol = float(self.tol)
        if self.persistent + self.auto_dispatch + self.chain > 1:
            raise ConfigError("persistent, auto_dispatch and chain are exclusive")
        o.dispatch = (N.TW_DISPATCH_PERSISTENT if self.persistent else
                      N.TW_DISPATCH_AUTO if self.auto_dispatch else
                      N.TW_DISPATCH_CHAIN if self.chain else N.TW_DISPATCH_STREAMS)
        o.x_update = {None: N.TW_XUPD_AUTO, "k2": N.TW_XUPD_K2, "k3": N.TW_XUPD_K3,
                      "k3_pairs": N.TW_XUPD_K3_PAIRS}[self.x_update]
        o.l2_keep = (N.TW_L2KEEP_AUTO if self.l2_keep is None else
                     N.TW_L2KEEP_ON if self.l2_keep else N.TW_L2KEEP_OFF)
        o.dag_spmv_slices = int(self.dag_spmv_slices)
        o.dag_vec_rows = int(self.dag_vec_rows)
        return o


@dataclass
class CgResult:
    """CgResult (cg.hpp:12-17)."""
    residual_history: np.ndarray
    x: np.ndarray
    iterations: int = 0
    converged: bool = False
    iteration_marks: np.ndarray = field(default_factory=lambda: np.zeros(0))


class CgSolver:
    """Persistent solve state (CgRun, cg.cpp:24-48) for repeated runs."""

    def __init__(self, rt: Runtime, A: EllMatrix, max_iterations: int,
                 opt: CgOptions | None = None, variant: int = N.TW_CG_TASKS):
        self.rt, self.A, self.opt = rt, A, opt or CgOptions()
        self.max_iterations = max_iterations
        h = C.c_void_p()
        copt = self.opt.to_c(variant)
        N.check(_lib().tw_cg_create(rt.h, A.h, C.byref(copt), max_iterations, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            N.check(_lib().tw_cg_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_rhs(self, b) -> None:
        if isinstance(b, np.ndarray):
            b = np.ascontiguousarray(b, np.float64)
            if len(b) != self.A.n:
                raise ContractViolation("rhs length differs from the owned rows")
            N.check(_lib().tw_cg_set_rhs(self.h, b.ctypes.data_as(C.c_void_p), 0))
        else:
            N.check(_lib().tw_cg_set_rhs(self.h, C.c_void_p(_ptr(b)), 1))

    def iterate(self, k: int) -> None:
        N.check(_lib().tw_cg_iterate(self.h, k))

    def wait(self) -> None:
        N.check(_lib().tw_cg_wait(self.h))

    def history(self, count: int) -> np.ndarray:
        out = np.zeros(count, np.float64)
        N.check(_lib().tw_cg_history(self.h, out.ctypes.data_as(N.dp), count))
        return out

    def solution(self) -> np.ndarray:
        out = np.zeros(self.A.n, np.float64)
        N.check(_lib().tw_cg_solution(self.h, out.ctypes.data_as(N.dp)))
        return out

    def marks(self, count: int) -> np.ndarray:
        out = np.zeros(count, np.float64)
        N.check(_lib().tw_cg_iteration_marks(self.h, out.ctypes.data_as(N.dp), count))
        return out

    def iteration_times(self, count: int) -> np.ndarray:
        """Device-timed seconds per iteration (needs iteration_marks)."""
        out = np.zeros(count, np.float64)
        N.check(_lib().tw_cg_iteration_times(self.h, out.ctypes.data_as(N.dp), count))
        return out

    def iterations_done(self) -> int:
        d = C.c_int()
        N.check(_lib().tw_cg_iterations_done(self.h, C.byref(d)))
        return d.value

    def vectors(self):
        ps = [C.c_void_p() for _ in range(4)]
        N.check(_lib().tw_cg_vectors(self.h, *[C.byref(p) for p in ps]))
        return [int(p.value or 0) for p in ps]

    def task_edges(self) -> list[tuple[str, str]]:
        need = C.c_int64()
        N.check(_lib().tw_cg_task_edges(self.h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(int(need.value))
        N.check(_lib().tw_cg_task_edges(self.h, buf, need.value, C.byref(need)))
        return [tuple(l.split()) for l in buf.value.decode().splitlines() if l]

    def enable_kernel_timing(self, on: bool = True) -> None:
        N.check(_lib().tw_cg_enable_kernel_timing(self.h, 1 if on else 0))

    def kernel_times(self) -> tuple[float, float, float, int]:
        """(K1 ms, K2 ms, K3 ms, timed iterations) summed since enable."""
        a, b, c, k = C.c_double(), C.c_double(), C.c_double(), C.c_int()
        N.check(_lib().tw_cg_kernel_times(self.h, C.byref(a), C.byref(b), C.byref(c), C.byref(k)))
        return a.value, b.value, c.value, k.value

    PEER_BLOB_BYTES = 256

    def peer_export(self) -> bytes:
        """This rank's CUDA-IPC blob for the NVLink peer transport."""
        buf = C.create_string_buffer(self.PEER_BLOB_BYTES)
        N.check(_lib().tw_cg_peer_export(self.h, buf))
        return buf.raw

    def peer_connect(self, blobs: list) -> None:
        """blobs: every rank's peer_export() in rank order (allgathered by
        the caller); switches the iteration to the peer transport."""
        if any(len(b) != self.PEER_BLOB_BYTES for b in blobs):
            raise ContractViolation("peer blobs must be PEER_BLOB_BYTES long")
        N.check(_lib().tw_cg_peer_connect(self.h, b"".join(blobs)))

    def peer_ping_send(self) -> None:
        N.check(_lib().tw_cg_peer_ping_send(self.h))

    def peer_ping_check(self, timeout_ms: int = 2000) -> bool:
        ok = C.c_int()
        N.check(_lib().tw_cg_peer_ping_check(self.h, timeout_ms, C.byref(ok)))
        return bool(ok.value)

    def enable_peer_transport(self) -> None:
        """Collective over torch.distributed: export, allgather, connect."""
        import torch.distributed as dist
        blobs = [None] * dist.get_world_size()
        dist.all_gather_object(blobs, self.peer_export())
        self.peer_connect(blobs)

    def launches_per_iteration(self) -> tuple[int, int]:
        k, c = C.c_int(), C.c_int()
        N.check(_lib().tw_cg_launches_per_iteration(self.h, C.byref(k), C.byref(c)))
        return k.value, c.value

    def mode(self) -> dict:
        """What this solver executes (tw_cg_mode): K1 form, x-run L2 policy,
        x-update placement, dispatch, transport, launches per iteration."""
        m = N.CgMode()
        N.check(_lib().tw_cg_mode(self.h, C.byref(m)))
        d = {k: getattr(m, k) for k, _ in N.CgMode._fields_}
        d["k1_kernel"] = N.TW_K1_NAMES[m.k1_form]
        return d


class EmulatedRankGroup:
    """P z-slab ranks on ONE device, driven together (tw_cg_group_*): the
    multi-GPU algorithm with loopback copies in place of the NCCL transport,
    for the monolithic variant (also over the peer transport) and the
    block-task DAG (variant TW_CG_TASKS, options.tiles tiles per rank, the
    halo task and rank-ordered alpha / beta_res).  Test infrastructure for
    the multi-rank path on a single B200."""

    def __init__(self, nx: int, ny: int, nz: int, nranks: int, max_iterations: int,
                 device: int = 0, transport: str = "loopback", x_staged: bool = True,
                 options: CgOptions | None = None, variant: int = N.TW_CG_MONOLITHIC):
        if transport not in ("loopback", "peer"):
            raise ValueError(f"unknown transport {transport!r}")
        self.P = nranks
        self.transport = transport
        self.rts, self.mats, self.solvers = [], [], []
        opt = options or CgOptions(iteration_marks=False)
        for r in range(nranks):
            rt = Runtime(device)
            rt.init_emulated_rank(r, nranks)
            zb, ze = slab_partition(nz, r, nranks)
            A = gen_stencil_matrix(nx, ny, nz, rt=rt, z_begin=zb, z_end=ze)
            if not x_staged:
                A.set_x_staged(False)
            self.rts.append(rt)
            self.mats.append(A)
            self.solvers.append(CgSolver(rt, A, max_iterations, opt, variant=variant))
        self._arr = (C.c_void_p * nranks)(*[s.h.value for s in self.solvers])
        if transport == "peer":
            N.check(_lib().tw_cg_group_enable_peer(self._arr, nranks))

    def set_rhs(self, b: np.ndarray) -> None:
        """b: the GLOBAL right-hand side; each rank takes its rows."""
        b = np.ascontiguousarray(b, np.float64)
        parts, keep = [], []
        for A in self.mats:
            off = int(A.info.row_offset)
            piece = np.ascontiguousarray(b[off:off + A.n])
            keep.append(piece)
            parts.append(piece.ctypes.data)
        ptrs = (C.c_void_p * self.P)(*parts)
        N.check(_lib().tw_cg_group_set_rhs(self._arr, self.P, ptrs, 0))

    def iterate(self, k: int) -> None:
        N.check(_lib().tw_cg_group_iterate(self._arr, self.P, k))

    def peer_check(self, timeout_ms: int = 2000) -> bool:
        """Transport check of the peer group: every rank pings, then every
        rank checks (no kernel waits on one not yet launched)."""
        for s in self.solvers:
            s.peer_ping_send()
        return all(s.peer_ping_check(timeout_ms) for s in self.solvers)

    def iterate_concurrent(self, k: int, jitter: bool = False) -> None:
        """Peer transport only: all ranks as one cooperative kernel, really
        waiting on one another's flags (tw_cg_group_iterate_concurrent)."""
        N.check(_lib().tw_cg_group_iterate_concurrent(self._arr, self.P, k, 1 if jitter else 0))

    def history(self, count: int) -> list:
        return [s.history(count) for s in self.solvers]

    def solution(self) -> np.ndarray:
        return np.concatenate([s.solution() for s in self.solvers])

    def close(self):
        for s in self.solvers:
            s.close()
        self.solvers = []


def _solve(rt: Runtime, A: EllMatrix, b, iterations: int, opt: CgOptions | None,
           variant: int) -> CgResult:
    opt = opt or CgOptions()
    s = CgSolver(rt, A, iterations, opt, variant)
    try:
        s.set_rhs(b)
        s.iterate(iterations)
        hist = s.history(iterations)
        x = s.solution()
        marks = s.marks(iterations) if opt.iteration_marks else np.zeros(0)
    finally:
        s.close()
    conv = bool(opt.tol > 0 and iterations > 0 and hist[-1] < opt.tol)
    return CgResult(hist, x, iterations, conv, marks)


def cg_solve(rt: Runtime, A: EllMatrix, b: np.ndarray, iterations: int,
             opt: CgOptions | None = None, variant: int = N.TW_CG_MONOLITHIC,
             x_out: np.ndarray | None = None) -> CgResult:
    """One solve through the single C-ABI entry a reference binding calls
    (tw_cg_solve): host b in, host history and x out."""
    opt = opt or CgOptions(iteration_marks=False)
    bh = np.ascontiguousarray(b, np.float64)
    if bh.shape != (A.n,):
        raise ContractViolation("rhs length differs from the matrix rows")
    hist = np.empty(max(iterations, 1), np.float64)
    x = x_out if x_out is not None else np.empty(A.n, np.float64)
    conv = C.c_int(0)
    o = opt.to_c(variant)
    N.check(_lib().tw_cg_solve(rt.h, A.h, bh.ctypes.data_as(C.c_void_p), iterations, C.byref(o),
                               hist.ctypes.data_as(N.dp), x.ctypes.data_as(N.dp), C.byref(conv)))
    return CgResult(hist[:iterations], x, iterations, bool(conv.value))


def cg_monolithic(rt: Runtime, A: EllMatrix, b, iterations: int,
                  opt: CgOptions | None = None) -> CgResult:
    """cg_monolithic (cg.cpp:397-436): one stream, tiles forced to 1."""
    return _solve(rt, A, b, iterations, opt, N.TW_CG_MONOLITHIC)


def cg_tasks(rt: Runtime, A: EllMatrix, b, iterations: int,
             opt: CgOptions | None = None) -> CgResult:
    """cg_tasks (cg.cpp:438-447): the block-task DAG on pooled streams."""
    return _solve(rt, A, b, iterations, opt, N.TW_CG_TASKS)
