/*
 * hpccg_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's HPCCG conjugate-gradient hot path
 * (taskweave, /root/reference/proj).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this file's
 * shared object, and only as the checker.  The product path
 * (paper_2602_21897_b200/csrc, libtw_hpccg.so) never links or calls it.
 *
 * Parity pin: every function is checked against the reference itself built
 * from its own sources (oracle/_ref/libtwref.so, see oracle/Makefile) and
 * against the committed golden vectors in tests/golden/ (tests/test_oracle.py).
 *
 * Floating point: compiled with -O2 -ffp-contract=off so a*b+c is two
 * roundings, exactly as the reference's default x86-64 build (no -march, so
 * no FMA: SURVEY.md section 7 "Bitwise SpMV/waxpby need no-FMA arithmetic").
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stddef.h>

#define ORC_OK 0
#define ORC_ERR_CONFIG 1

/* ---------------------------------------------------------------------- */
/* generate_matrix: proj/src/csr.cpp:29-59                                 */
/* ---------------------------------------------------------------------- */

/* Number of in-bounds neighbours along one axis for coordinate c in [0,d). */
static int64_t axis_span(int64_t c, int64_t d) {
    int64_t lo = c > 0 ? c - 1 : c;
    int64_t hi = c + 1 < d ? c + 1 : c;
    return hi - lo + 1;
}

/* nnz of the 27-point stencil on nx*ny*nz: product of per-axis sums
 * (3d-2 for d>=2, 1 for d==1).  Same count gen_stencil_matrix pushes. */
int64_t orc_stencil_nnz(int64_t nx, int64_t ny, int64_t nz) {
    int64_t sx = nx == 1 ? 1 : 3 * nx - 2;
    int64_t sy = ny == 1 ? 1 : 3 * ny - 2;
    int64_t sz = nz == 1 ? 1 : 3 * nz - 2;
    return sx * sy * sz;
}

/* Validation rules of csr.cpp:30-34: dims >= 1 and 27*cells*8 fits int64. */
int orc_stencil_check(int64_t nx, int64_t ny, int64_t nz) {
    if (nx < 1 || ny < 1 || nz < 1)
        return ORC_ERR_CONFIG;
    __int128 cells = (__int128)nx * ny * nz;
    if (cells * 27 > (__int128)(INT64_MAX / 8))
        return ORC_ERR_CONFIG;
    return ORC_OK;
}

/* Rows z-major, row = (z*ny + y)*nx + x (csr.cpp:43-45); per row the
 * neighbours in (dz,dy,dx) lexicographic order, which is ascending column
 * order (csr.cpp:46-53); 27.0 on the diagonal, -1.0 elsewhere (csr.cpp:54).
 * Rows [r0, r1) of the full matrix; row_ptr is relative (row_ptr[0] = 0,
 * r1 - r0 + 1 entries), so a grid whose CSR does not fit host memory is
 * checked a z-slab at a time.  Caller sizes col_idx/values. */
int orc_gen_stencil_csr_rows(int64_t nx, int64_t ny, int64_t nz, int64_t r0, int64_t r1,
                             int64_t* row_ptr, int64_t* col_idx, double* values) {
    if (orc_stencil_check(nx, ny, nz) != ORC_OK)
        return ORC_ERR_CONFIG;
    if (r0 < 0 || r1 < r0 || r1 > nx * ny * nz)
        return ORC_ERR_CONFIG;
    int64_t k = 0;
    row_ptr[0] = 0;
    for (int64_t row = r0; row < r1; ++row) {
        const int64_t x = row % nx, y = (row / nx) % ny, z = row / (nx * ny);
        for (int64_t cz = z - 1; cz <= z + 1; ++cz) {
            if (cz < 0 || cz >= nz) continue;
            for (int64_t cy = y - 1; cy <= y + 1; ++cy) {
                if (cy < 0 || cy >= ny) continue;
                int64_t line = (cz * ny + cy) * nx;
                for (int64_t cx = x - 1; cx <= x + 1; ++cx) {
                    if (cx < 0 || cx >= nx) continue;
                    col_idx[k] = line + cx;
                    values[k] = (cx == x && cy == y && cz == z) ? 27.0 : -1.0;
                    ++k;
                }
            }
        }
        row_ptr[row - r0 + 1] = k;
    }
    return ORC_OK;
}

/* The whole matrix (gen_stencil_matrix, csr.cpp:29-59). */
int orc_gen_stencil_csr(int64_t nx, int64_t ny, int64_t nz, int64_t* row_ptr,
                        int64_t* col_idx, double* values) {
    if (orc_stencil_check(nx, ny, nz) != ORC_OK)
        return ORC_ERR_CONFIG;
    return orc_gen_stencil_csr_rows(nx, ny, nz, 0, nx * ny * nz, row_ptr, col_idx, values);
}

/* Row length of the stencil at (x,y,z), used by structure checks. */
int64_t orc_stencil_row_len(int64_t nx, int64_t ny, int64_t nz, int64_t x, int64_t y,
                            int64_t z) {
    return axis_span(x, nx) * axis_span(y, ny) * axis_span(z, nz);
}

/* CsrMatrix::validate, csr.cpp:13-27.  Returns 0 when valid. */
int orc_csr_validate(int64_t n, const int64_t* row_ptr, int64_t nnz_stored,
                     const int64_t* col_idx) {
    if (n < 0) return ORC_ERR_CONFIG;
    if (row_ptr[0] != 0) return ORC_ERR_CONFIG;
    for (int64_t i = 0; i < n; ++i)
        if (row_ptr[i] > row_ptr[i + 1]) return ORC_ERR_CONFIG;
    if (nnz_stored != row_ptr[n]) return ORC_ERR_CONFIG;
    for (int64_t k = 0; k < nnz_stored; ++k)
        if (col_idx[k] < 0 || col_idx[k] >= n) return ORC_ERR_CONFIG;
    return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* HPC_sparsemv / ddot / waxpby: proj/src/kernels.cpp:5-26                 */
/* ---------------------------------------------------------------------- */

/* y[i] = sum_k values[k]*x[col[k]], accumulator from 0.0, k ascending,
 * multiply then add (kernels.cpp:5-13). */
void orc_spmv_range(const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                    const double* x, double* y, int64_t r0, int64_t r1) {
    for (int64_t i = r0; i < r1; ++i) {
        double sum = 0.0;
        int64_t k1 = row_ptr[i + 1];
        for (int64_t k = row_ptr[i]; k < k1; ++k) {
            double prod = values[k] * x[col_idx[k]];
            sum = sum + prod;
        }
        y[i] = sum;
    }
}

/* Sequential left-to-right sum of a[i]*b[i] (kernels.cpp:15-20). */
double orc_dot_range(const double* a, const double* b, int64_t i0, int64_t i1) {
    double s = 0.0;
    for (int64_t i = i0; i < i1; ++i) {
        double prod = a[i] * b[i];
        s = s + prod;
    }
    return s;
}

/* w = alpha*x + beta*y, three roundings, w may alias x or y (kernels.cpp:22-26). */
void orc_waxpby_range(double alpha, const double* x, double beta, const double* y, double* w,
                      int64_t i0, int64_t i1) {
    for (int64_t i = i0; i < i1; ++i) {
        double ax = alpha * x[i];
        double by = beta * y[i];
        w[i] = ax + by;
    }
}

/* ---------------------------------------------------------------------- */
/* make_tile_plan: proj/src/cg.cpp:348-370                                 */
/* ---------------------------------------------------------------------- */

/* Equal contiguous row blocks r0 = n*t/T; band = min/max touched column,
 * collapsed to [r0,r0] for an empty tile.  Outputs four int64[T] arrays. */
int orc_make_tile_plan(int64_t n, const int64_t* row_ptr, const int64_t* col_idx, int tiles,
                       int64_t* r0, int64_t* r1, int64_t* band_lo, int64_t* band_hi) {
    if (tiles < 1 || (int64_t)tiles > n)
        return ORC_ERR_CONFIG;
    for (int t = 0; t < tiles; ++t) {
        int64_t a = n * t / tiles, b = n * (t + 1) / tiles;
        int64_t lo = n, hi = 0;
        for (int64_t k = row_ptr[a]; k < row_ptr[b]; ++k) {
            if (col_idx[k] < lo) lo = col_idx[k];
            if (col_idx[k] > hi) hi = col_idx[k];
        }
        if (row_ptr[a] == row_ptr[b]) { lo = a; hi = a; }
        r0[t] = a; r1[t] = b; band_lo[t] = lo; band_hi[t] = hi;
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* CG drivers: proj/src/cg.cpp:372-395 (cg_reference) and the tile-order   */
/* reduction of cg_tasks (cg.cpp:209-225, 290-311).                         */
/* ---------------------------------------------------------------------- */

/* Unpreconditioned CG with x0 = 0, r0 = p0 = b.  Per iteration: spmv, pAp,
 * alpha, x += alpha p, r -= alpha Ap, rr, beta, history = sqrt(rr),
 * p = r + beta p.  `tiles` = 1 reproduces cg_reference / cg_monolithic;
 * tiles > 1 reproduces cg_tasks' numerics exactly (per-tile partials summed
 * in tile order), which is schedule independent.  Work arrays: 4n doubles.
 * Returns converged flag semantics of cg.cpp:392-393 via *converged. */
int orc_cg(int64_t n, const int64_t* row_ptr, const int64_t* col_idx, const double* values,
           const double* b, int iterations, double tol, int tiles, double* history,
           double* x_out, double* work, int* converged) {
    if (tiles < 1 || (int64_t)tiles > n)
        return ORC_ERR_CONFIG;
    double* r = work;
    double* p = work + n;
    double* Ap = work + 2 * n;
    double* x = x_out;
    for (int64_t i = 0; i < n; ++i) {
        x[i] = 0.0;
        r[i] = b[i];
        p[i] = b[i];
        Ap[i] = 0.0;
    }
    double rtrans = orc_dot_range(r, r, 0, n);
    for (int it = 0; it < iterations; ++it) {
        orc_spmv_range(row_ptr, col_idx, values, p, Ap, 0, n);
        double pAp = 0.0;
        for (int t = 0; t < tiles; ++t)
            pAp += orc_dot_range(p, Ap, n * t / tiles, n * (t + 1) / tiles);
        double alpha = rtrans / pAp;
        orc_waxpby_range(1.0, x, alpha, p, x, 0, n);
        orc_waxpby_range(1.0, r, -alpha, Ap, r, 0, n);
        double rr = 0.0;
        for (int t = 0; t < tiles; ++t)
            rr += orc_dot_range(r, r, n * t / tiles, n * (t + 1) / tiles);
        double beta = rr / rtrans;
        rtrans = rr;
        history[it] = sqrt(rr);
        orc_waxpby_range(1.0, r, beta, p, p, 0, n);
    }
    if (converged)
        *converged = tol > 0 && iterations > 0 && history[iterations - 1] < tol;
    return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* Matrix-free restatement for grids whose CSR does not fit host memory    */
/* (SURVEY.md 8(c)): identical row order, neighbour order, constants and   */
/* rounding sequence as gen_stencil_matrix + spmv_range, so its Ap is      */
/* bit-identical to the CSR path (pinned by tests/test_oracle.py).          */
/* ---------------------------------------------------------------------- */

void orc_stencil_spmv_range(int64_t nx, int64_t ny, int64_t nz, const double* x, double* y,
                            int64_t r0, int64_t r1) {
    const int64_t plane = nx * ny;
    for (int64_t row = r0; row < r1; ++row) {
        int64_t z = row / plane;
        int64_t rem = row - z * plane;
        int64_t yy = rem / nx;
        int64_t xx = rem - yy * nx;
        double sum = 0.0;
        for (int64_t cz = z - 1; cz <= z + 1; ++cz) {
            if (cz < 0 || cz >= nz) continue;
            for (int64_t cy = yy - 1; cy <= yy + 1; ++cy) {
                if (cy < 0 || cy >= ny) continue;
                const double* line = x + (cz * ny + cy) * nx;
                for (int64_t cx = xx - 1; cx <= xx + 1; ++cx) {
                    if (cx < 0 || cx >= nx) continue;
                    double v = (cx == xx && cy == yy && cz == z) ? 27.0 : -1.0;
                    double prod = v * line[cx];
                    sum = sum + prod;
                }
            }
        }
        y[row] = sum;
    }
}

/* cg_reference over the matrix-free operator; work = 4n doubles. */
int orc_cg_stencil(int64_t nx, int64_t ny, int64_t nz, const double* b, int iterations,
                   int tiles, double* history, double* x_out, double* work) {
    if (orc_stencil_check(nx, ny, nz) != ORC_OK)
        return ORC_ERR_CONFIG;
    const int64_t n = nx * ny * nz;
    if (tiles < 1 || (int64_t)tiles > n)
        return ORC_ERR_CONFIG;
    double* r = work;
    double* p = work + n;
    double* Ap = work + 2 * n;
    double* x = x_out;
    for (int64_t i = 0; i < n; ++i) {
        x[i] = 0.0; r[i] = b[i]; p[i] = b[i]; Ap[i] = 0.0;
    }
    double rtrans = orc_dot_range(r, r, 0, n);
    for (int it = 0; it < iterations; ++it) {
        orc_stencil_spmv_range(nx, ny, nz, p, Ap, 0, n);
        double pAp = 0.0;
        for (int t = 0; t < tiles; ++t)
            pAp += orc_dot_range(p, Ap, n * t / tiles, n * (t + 1) / tiles);
        double alpha = rtrans / pAp;
        orc_waxpby_range(1.0, x, alpha, p, x, 0, n);
        orc_waxpby_range(1.0, r, -alpha, Ap, r, 0, n);
        double rr = 0.0;
        for (int t = 0; t < tiles; ++t)
            rr += orc_dot_range(r, r, n * t / tiles, n * (t + 1) / tiles);
        double beta = rr / rtrans;
        rtrans = rr;
        history[it] = sqrt(rr);
        orc_waxpby_range(1.0, r, beta, p, p, 0, n);
    }
    return ORC_OK;
}

/* The same CG with the row-parallel phases on `threads` host threads, for
 * the sizes the GPU headline runs (256^3, 512^3).  SpMV rows and waxpby
 * elements are independent, so splitting them changes no bit; every dot
 * stays a sequential left-to-right sum per tile, tiles summed in order, so
 * the result is bit-identical to orc_cg_stencil for any thread count
 * (pinned by tests/test_oracle.py). */
typedef struct {
    int64_t nx, ny, nz, n, i0, i1;
    int phase; /* 0: Ap = A p; 1: x += alpha p, r -= alpha Ap; 2: p = r + beta p */
    double alpha, beta;
    double *x, *r, *p, *Ap;
} orc_job;

static void* orc_job_run(void* arg) {
    orc_job* j = (orc_job*)arg;
    if (j->phase == 0) {
        orc_stencil_spmv_range(j->nx, j->ny, j->nz, j->p, j->Ap, j->i0, j->i1);
    } else if (j->phase == 1) {
        orc_waxpby_range(1.0, j->x, j->alpha, j->p, j->x, j->i0, j->i1);
        orc_waxpby_range(1.0, j->r, -j->alpha, j->Ap, j->r, j->i0, j->i1);
    } else {
        orc_waxpby_range(1.0, j->r, j->beta, j->p, j->p, j->i0, j->i1);
    }
    return NULL;
}

#define ORC_MAX_THREADS 256

static int orc_parallel(orc_job* tmpl, int threads) {
    pthread_t th[ORC_MAX_THREADS];
    orc_job jobs[ORC_MAX_THREADS];
    int started = 0;
    for (int t = 0; t < threads; ++t) {
        jobs[t] = *tmpl;
        jobs[t].i0 = tmpl->n * t / threads;
        jobs[t].i1 = tmpl->n * (t + 1) / threads;
        if (t == threads - 1 || pthread_create(&th[t], NULL, orc_job_run, &jobs[t]) != 0) {
            orc_job_run(&jobs[t]);
        } else {
            ++started;
        }
    }
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
    return ORC_OK;
}

int orc_cg_stencil_mt(int64_t nx, int64_t ny, int64_t nz, const double* b, int iterations,
                      int tiles, int threads, double* history, double* x_out, double* work) {
    if (orc_stencil_check(nx, ny, nz) != ORC_OK)
        return ORC_ERR_CONFIG;
    const int64_t n = nx * ny * nz;
    if (tiles < 1 || (int64_t)tiles > n || threads < 1 || threads > ORC_MAX_THREADS)
        return ORC_ERR_CONFIG;
    if ((int64_t)threads > n) threads = (int)n;
    orc_job j = {nx, ny, nz, n, 0, n, 0, 0.0, 0.0, x_out, work, work + n, work + 2 * n};
    for (int64_t i = 0; i < n; ++i) {
        j.x[i] = 0.0; j.r[i] = b[i]; j.p[i] = b[i]; j.Ap[i] = 0.0;
    }
    double rtrans = orc_dot_range(j.r, j.r, 0, n);
    for (int it = 0; it < iterations; ++it) {
        j.phase = 0;
        orc_parallel(&j, threads);
        double pAp = 0.0;
        for (int t = 0; t < tiles; ++t)
            pAp += orc_dot_range(j.p, j.Ap, n * t / tiles, n * (t + 1) / tiles);
        j.alpha = rtrans / pAp;
        j.phase = 1;
        orc_parallel(&j, threads);
        double rr = 0.0;
        for (int t = 0; t < tiles; ++t)
            rr += orc_dot_range(j.r, j.r, n * t / tiles, n * (t + 1) / tiles);
        j.beta = rr / rtrans;
        rtrans = rr;
        history[it] = sqrt(rr);
        j.phase = 2;
        orc_parallel(&j, threads);
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* Right-hand sides                                                        */
/* ---------------------------------------------------------------------- */

/* xorshift64 (13, 7, 17), value 0.5 + (s mod 1000)/1000:
 * proj/tests/acceptance.cpp:48-58 and proj/tests/test_bench.cpp:26-36. */
void orc_rhs_xorshift(int64_t n, uint64_t seed, double* out) {
    uint64_t s = seed;
    for (int64_t i = 0; i < n; ++i) {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        out[i] = 0.5 + (double)(s % 1000u) / 1000.0;
    }
}

/* SplitMix64 uniform [0,1) doubles: proj/src/scenario.cpp:46-55, used for
 * b at scenario.cpp:91-95. */
void orc_rhs_splitmix(int64_t n, uint64_t seed, double* out) {
    uint64_t s = seed;
    for (int64_t i = 0; i < n; ++i) {
        s += 0x9e3779b97f4a7c15ull;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z ^= z >> 31;
        out[i] = (double)(z >> 11) * 0x1.0p-53;
    }
}
