"""TEST INFRASTRUCTURE ONLY -- the CPU checker for the HPCCG hot path.

Two checkers live here, both loaded through ctypes:

* ``Oracle`` wraps ``_build/liboracle.so``, the plain-C restatement in
  ``hpccg_oracle.c`` (each function cites the reference file:line it follows).
* ``Reference`` wraps ``_ref/libtwref.so``, the reference's own C++ sources
  (``/root/reference/proj/src``) compiled by ``oracle/Makefile``, reached
  through ``ref_capi.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only to check or to time the CPU baseline.  The product package
``paper_2602_21897_b200`` never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtwref.so")

_i64 = C.c_int64
_dp = C.POINTER(C.c_double)
_lp = C.POINTER(C.c_int64)


def _d(a):
    return a.ctypes.data_as(_dp)


def _l(a):
    return a.ctypes.data_as(_lp)


def build(ref: bool | None = None) -> None:
    """Run oracle/Makefile (the reference target only when its sources exist)."""
    target = ["all"] if ref is None else (["oracle", "ref"] if ref else ["oracle"])
    subprocess.run(["make", "-s", "-C", HERE, *target], check=True)


class OracleError(RuntimeError):
    pass


@dataclass
class Csr:
    n: int
    row_ptr: np.ndarray  # int64[n+1]
    col_idx: np.ndarray  # int64[nnz]
    values: np.ndarray   # float64[nnz]

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])


class Oracle:
    """ctypes face of hpccg_oracle.c."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.orc_stencil_nnz.restype = _i64
        L.orc_stencil_nnz.argtypes = [_i64, _i64, _i64]
        L.orc_stencil_check.argtypes = [_i64, _i64, _i64]
        L.orc_gen_stencil_csr.argtypes = [_i64, _i64, _i64, _lp, _lp, _dp]
        L.orc_gen_stencil_csr_rows.argtypes = [_i64] * 5 + [_lp, _lp, _dp]
        L.orc_cg_stencil_mt.argtypes = [_i64, _i64, _i64, _dp, C.c_int, C.c_int, C.c_int, _dp,
                                        _dp, _dp]
        L.orc_stencil_row_len.restype = _i64
        L.orc_stencil_row_len.argtypes = [_i64] * 6
        L.orc_csr_validate.argtypes = [_i64, _lp, _i64, _lp]
        L.orc_spmv_range.argtypes = [_lp, _lp, _dp, _dp, _dp, _i64, _i64]
        L.orc_dot_range.restype = C.c_double
        L.orc_dot_range.argtypes = [_dp, _dp, _i64, _i64]
        L.orc_waxpby_range.argtypes = [C.c_double, _dp, C.c_double, _dp, _dp, _i64, _i64]
        L.orc_make_tile_plan.argtypes = [_i64, _lp, _lp, C.c_int, _lp, _lp, _lp, _lp]
        L.orc_cg.argtypes = [_i64, _lp, _lp, _dp, _dp, C.c_int, C.c_double, C.c_int, _dp, _dp,
                             _dp, C.POINTER(C.c_int)]
        L.orc_stencil_spmv_range.argtypes = [_i64, _i64, _i64, _dp, _dp, _i64, _i64]
        L.orc_cg_stencil.argtypes = [_i64, _i64, _i64, _dp, C.c_int, C.c_int, _dp, _dp, _dp]
        L.orc_rhs_xorshift.argtypes = [_i64, C.c_uint64, _dp]
        L.orc_rhs_splitmix.argtypes = [_i64, C.c_uint64, _dp]

    # generate_matrix (csr.cpp:29-59)
    def stencil(self, nx: int, ny: int, nz: int) -> Csr:
        if self.lib.orc_stencil_check(nx, ny, nz) != 0:
            raise OracleError("stencil dims must be at least 1 / overflow")
        n = nx * ny * nz
        nnz = self.lib.orc_stencil_nnz(nx, ny, nz)
        rp = np.empty(n + 1, np.int64)
        ci = np.empty(nnz, np.int64)
        va = np.empty(nnz, np.float64)
        self.lib.orc_gen_stencil_csr(nx, ny, nz, _l(rp), _l(ci), _d(va))
        return Csr(n, rp, ci, va)

    def stencil_rows(self, nx: int, ny: int, nz: int, r0: int, r1: int) -> Csr:
        """Rows [r0, r1) of the full stencil matrix (row_ptr relative to r0)."""
        if self.lib.orc_stencil_check(nx, ny, nz) != 0 or not 0 <= r0 <= r1 <= nx * ny * nz:
            raise OracleError("stencil dims / row range")
        rp = np.empty(r1 - r0 + 1, np.int64)
        cap = 27 * (r1 - r0)
        ci = np.empty(cap, np.int64)
        va = np.empty(cap, np.float64)
        self.lib.orc_gen_stencil_csr_rows(nx, ny, nz, r0, r1, _l(rp), _l(ci), _d(va))
        k = int(rp[-1])
        return Csr(r1 - r0, rp, ci[:k], va[:k])

    def stencil_nnz(self, nx, ny, nz) -> int:
        return int(self.lib.orc_stencil_nnz(nx, ny, nz))

    def validate(self, m: Csr) -> bool:
        return self.lib.orc_csr_validate(m.n, _l(m.row_ptr), len(m.col_idx), _l(m.col_idx)) == 0

    # HPC_sparsemv / ddot / waxpby (kernels.cpp:5-26)
    def spmv(self, m: Csr, x: np.ndarray, r0: int = 0, r1: int | None = None,
             y: np.ndarray | None = None) -> np.ndarray:
        r1 = m.n if r1 is None else r1
        y = np.zeros(m.n, np.float64) if y is None else y
        self.lib.orc_spmv_range(_l(m.row_ptr), _l(m.col_idx), _d(m.values), _d(x), _d(y), r0, r1)
        return y

    def stencil_spmv(self, nx, ny, nz, x, r0=0, r1=None):
        n = nx * ny * nz
        r1 = n if r1 is None else r1
        y = np.zeros(n, np.float64)
        self.lib.orc_stencil_spmv_range(nx, ny, nz, _d(x), _d(y), r0, r1)
        return y

    def dot(self, a, b, i0=0, i1=None) -> float:
        i1 = len(a) if i1 is None else i1
        return float(self.lib.orc_dot_range(_d(a), _d(b), i0, i1))

    def waxpby(self, alpha, x, beta, y, w=None, i0=0, i1=None):
        i1 = len(x) if i1 is None else i1
        w = np.zeros_like(x) if w is None else w
        self.lib.orc_waxpby_range(alpha, _d(x), beta, _d(y), _d(w), i0, i1)
        return w

    # make_tile_plan (cg.cpp:348-370)
    def tile_plan(self, m: Csr, tiles: int):
        out = [np.empty(tiles, np.int64) for _ in range(4)]
        if self.lib.orc_make_tile_plan(m.n, _l(m.row_ptr), _l(m.col_idx), tiles,
                                       *[_l(a) for a in out]) != 0:
            raise OracleError("tile plan needs 1 <= tiles <= n")
        return out

    # cg_reference (cg.cpp:372-395); tiles>1 = cg_tasks' tile-order reduction
    def cg(self, m: Csr, b: np.ndarray, iterations: int, tol: float = 0.0, tiles: int = 1):
        hist = np.zeros(max(iterations, 1), np.float64)
        x = np.zeros(m.n, np.float64)
        work = np.zeros(3 * m.n, np.float64)
        conv = C.c_int(0)
        if self.lib.orc_cg(m.n, _l(m.row_ptr), _l(m.col_idx), _d(m.values), _d(b), iterations,
                           tol, tiles, _d(hist), _d(x), _d(work), C.byref(conv)) != 0:
            raise OracleError("cg: bad tile count")
        return hist[:iterations], x, bool(conv.value)

    def cg_stencil(self, nx, ny, nz, b, iterations, tiles=1):
        n = nx * ny * nz
        hist = np.zeros(max(iterations, 1), np.float64)
        x = np.zeros(n, np.float64)
        work = np.zeros(3 * n, np.float64)
        if self.lib.orc_cg_stencil(nx, ny, nz, _d(b), iterations, tiles, _d(hist), _d(x),
                                   _d(work)) != 0:
            raise OracleError("cg_stencil: bad dims / tiles")
        return hist[:iterations], x

    def cg_stencil_mt(self, nx, ny, nz, b, iterations, tiles=1, threads=None):
        """cg_stencil with the row-parallel phases threaded (bit-identical)."""
        n = nx * ny * nz
        threads = threads or min(os.cpu_count() or 1, 64)
        hist = np.zeros(max(iterations, 1), np.float64)
        x = np.empty(n, np.float64)
        work = np.empty(3 * n, np.float64)
        if self.lib.orc_cg_stencil_mt(nx, ny, nz, _d(b), iterations, tiles, threads, _d(hist),
                                      _d(x), _d(work)) != 0:
            raise OracleError("cg_stencil_mt: bad dims / tiles / threads")
        return hist[:iterations], x

    # right-hand sides (acceptance.cpp:48-58, scenario.cpp:46-55)
    def rhs_xorshift(self, n: int, seed: int = 7) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.lib.orc_rhs_xorshift(n, seed, _d(out))
        return out

    def rhs_splitmix(self, n: int, seed: int = 7) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.lib.orc_rhs_splitmix(n, seed, _d(out))
        return out


class Reference:
    """ctypes face of the reference's own sources (oracle/_ref/libtwref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise OracleError(f"{path} missing: build it with `make -C oracle ref` where "
                              "/root/reference is mounted")
        L = self.lib = C.CDLL(path)
        vpp = C.POINTER(C.c_void_p)
        L.twref_last_error.restype = C.c_char_p
        L.twref_matrix_stencil.argtypes = [_i64, _i64, _i64, vpp]
        L.twref_matrix_from_csr.argtypes = [_i64, _lp, _lp, _dp, vpp]
        L.twref_matrix_free.argtypes = [C.c_void_p]
        L.twref_matrix_n.restype = _i64
        L.twref_matrix_n.argtypes = [C.c_void_p]
        L.twref_matrix_nnz.restype = _i64
        L.twref_matrix_nnz.argtypes = [C.c_void_p]
        L.twref_matrix_export.argtypes = [C.c_void_p, _lp, _lp, _dp]
        L.twref_matrix_dump.restype = _i64
        L.twref_matrix_dump.argtypes = [C.c_void_p, C.c_char_p, _i64]
        L.twref_matrix_load.argtypes = [C.c_char_p, vpp]
        L.twref_spmv_range.argtypes = [C.c_void_p, _dp, _dp, _i64, _i64]
        L.twref_dot_range.restype = C.c_double
        L.twref_dot_range.argtypes = [_dp, _dp, _i64, _i64]
        L.twref_waxpby_range.argtypes = [C.c_double, _dp, C.c_double, _dp, _dp, _i64, _i64]
        L.twref_tile_plan.argtypes = [C.c_void_p, C.c_int, _lp, _lp, _lp, _lp]
        L.twref_cg_reference.argtypes = [C.c_void_p, _dp, C.c_int, C.c_double, _dp, _dp,
                                         C.POINTER(C.c_int)]
        L.twref_cg_tasks.argtypes = [C.c_void_p, _dp, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.c_int, C.c_int, _dp, _dp, _dp, _dp]
        L.twref_cg_task_edges.restype = _i64
        L.twref_cg_task_edges.argtypes = [C.c_void_p, _dp, C.c_int, C.c_int, C.c_char_p, _i64]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(self.lib.twref_last_error().decode())

    class Matrix:
        def __init__(self, ref: "Reference", handle):
            self.ref, self.h = ref, handle

        def __del__(self):
            if getattr(self, "h", None):
                self.ref.lib.twref_matrix_free(self.h)
                self.h = None

        @property
        def n(self) -> int:
            return int(self.ref.lib.twref_matrix_n(self.h))

        @property
        def nnz(self) -> int:
            return int(self.ref.lib.twref_matrix_nnz(self.h))

        def export(self) -> Csr:
            n, nnz = self.n, self.nnz
            rp = np.empty(n + 1, np.int64)
            ci = np.empty(nnz, np.int64)
            va = np.empty(nnz, np.float64)
            self.ref.lib.twref_matrix_export(self.h, _l(rp), _l(ci), _d(va))
            return Csr(n, rp, ci, va)

        def dump(self) -> str:
            need = self.ref.lib.twref_matrix_dump(self.h, None, 0)
            buf = C.create_string_buffer(int(need))
            self.ref.lib.twref_matrix_dump(self.h, buf, need)
            return buf.value.decode()

    def stencil(self, nx, ny, nz) -> "Reference.Matrix":
        h = C.c_void_p()
        self._check(self.lib.twref_matrix_stencil(nx, ny, nz, C.byref(h)))
        return Reference.Matrix(self, h)

    def from_csr(self, m: Csr) -> "Reference.Matrix":
        h = C.c_void_p()
        self._check(self.lib.twref_matrix_from_csr(m.n, _l(m.row_ptr), _l(m.col_idx),
                                                   _d(m.values), C.byref(h)))
        return Reference.Matrix(self, h)

    def load(self, text: str) -> "Reference.Matrix":
        h = C.c_void_p()
        self._check(self.lib.twref_matrix_load(text.encode(), C.byref(h)))
        return Reference.Matrix(self, h)

    def spmv(self, M, x, r0=0, r1=None):
        r1 = M.n if r1 is None else r1
        y = np.zeros(M.n, np.float64)
        self.lib.twref_spmv_range(M.h, _d(x), _d(y), r0, r1)
        return y

    def dot(self, a, b, i0=0, i1=None):
        i1 = len(a) if i1 is None else i1
        return float(self.lib.twref_dot_range(_d(a), _d(b), i0, i1))

    def waxpby(self, alpha, x, beta, y, i0=0, i1=None):
        i1 = len(x) if i1 is None else i1
        w = np.zeros_like(x)
        self.lib.twref_waxpby_range(alpha, _d(x), beta, _d(y), _d(w), i0, i1)
        return w

    def tile_plan(self, M, tiles):
        out = [np.empty(tiles, np.int64) for _ in range(4)]
        self._check(self.lib.twref_tile_plan(M.h, tiles, *[_l(a) for a in out]))
        return out

    def cg_reference(self, M, b, iterations, tol=0.0):
        hist = np.zeros(max(iterations, 1), np.float64)
        x = np.zeros(M.n, np.float64)
        conv = C.c_int(0)
        self._check(self.lib.twref_cg_reference(M.h, _d(b), iterations, tol, _d(hist), _d(x),
                                                C.byref(conv)))
        return hist[:iterations], x, bool(conv.value)

    def cg_tasks(self, M, b, iterations, tiles=16, workers=4, real_threads=False,
                 monolithic=False, backend=0):
        """Returns (history, x, wall_seconds)."""
        h, x, secs, _ = self.cg_tasks_marks(M, b, iterations, tiles, workers, real_threads,
                                            monolithic, backend)
        return h, x, secs

    def cg_tasks_marks(self, M, b, iterations, tiles=16, workers=4, real_threads=False,
                       monolithic=False, backend=0):
        """Returns (history, x, wall_seconds, marks): marks[i] = time of the
        reference's cg_iter=i mark (substrate seconds since runtime start;
        real seconds with real_threads), as scenario.cpp:116-124 reads them."""
        hist = np.zeros(max(iterations, 1), np.float64)
        x = np.zeros(M.n, np.float64)
        marks = np.zeros(max(iterations, 1), np.float64)
        secs = C.c_double(0.0)
        self._check(self.lib.twref_cg_tasks(M.h, _d(b), iterations, 0 if monolithic else 1,
                                            tiles, workers, 1 if real_threads else 0, backend,
                                            _d(hist), _d(x), C.byref(secs), _d(marks)))
        return hist[:iterations], x, secs.value, marks[:iterations]

    def cg_task_edges(self, M, b, iterations, tiles):
        need = self.lib.twref_cg_task_edges(M.h, _d(b), iterations, tiles, None, 0)
        if need < 0:
            raise OracleError(self.lib.twref_last_error().decode())
        buf = C.create_string_buffer(int(need))
        self.lib.twref_cg_task_edges(M.h, _d(b), iterations, tiles, buf, need)
        return [tuple(l.split()) for l in buf.value.decode().splitlines() if l]


def reference_available() -> bool:
    return os.path.exists(REF_SO)
