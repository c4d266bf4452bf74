// TEST INFRASTRUCTURE ONLY -- extern "C" face of the reference's own CPU
// implementation, compiled together with the reference sources under
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libtwref.so.
// Used (a) to pin the C restatement in hpccg_oracle.c and to generate the
// golden vectors in tests/golden/, and (b) as bench.py's --impl reference /
// cpu_baseline arm.  Nothing in the product library links it.
//
// Every entry point maps one reference call:
//   twref_matrix_stencil  -> tw::bench::gen_stencil_matrix   (csr.cpp:29-59)
//   twref_spmv_range      -> tw::bench::spmv_range           (kernels.cpp:5-13)
//   twref_dot_range       -> tw::bench::dot_range            (kernels.cpp:15-20)
//   twref_waxpby_range    -> tw::bench::waxpby_range         (kernels.cpp:22-26)
//   twref_tile_plan       -> tw::bench::make_tile_plan       (cg.cpp:348-370)
//   twref_cg_reference    -> tw::bench::cg_reference         (cg.cpp:372-395)
//   twref_cg_tasks        -> tw::bench::cg_tasks / cg_monolithic (cg.cpp:397-447)
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "taskweave/cg.hpp"
#include "taskweave/csr.hpp"
#include "taskweave/kernels.hpp"
#include "taskweave/runtime.hpp"
#include "taskweave/types.hpp"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const tw::ConfigError& e) {
        return fail(e, 1);
    } catch (const tw::ContractViolation& e) {
        return fail(e, 2);
    } catch (const std::exception& e) {
        return fail(e, 3);
    }
}

tw::bench::CsrMatrix* as_mat(void* h) { return static_cast<tw::bench::CsrMatrix*>(h); }

void write_result(const tw::bench::CgResult& r, double* history, double* x) {
    if (history)
        std::copy(r.residual_history.begin(), r.residual_history.end(), history);
    if (x)
        std::copy(r.x.begin(), r.x.end(), x);
}

} // namespace

extern "C" {

const char* twref_last_error() { return g_err.c_str(); }

int twref_matrix_stencil(std::int64_t nx, std::int64_t ny, std::int64_t nz, void** out) {
    return guarded([&] {
        *out = new tw::bench::CsrMatrix(tw::bench::gen_stencil_matrix(nx, ny, nz));
    });
}

int twref_matrix_from_csr(std::int64_t n, const std::int64_t* row_ptr,
                          const std::int64_t* col_idx, const double* values, void** out) {
    return guarded([&] {
        auto* m = new tw::bench::CsrMatrix;
        m->n = n;
        m->row_ptr.assign(row_ptr, row_ptr + n + 1);
        std::int64_t nnz = row_ptr[n];
        m->col_idx.assign(col_idx, col_idx + nnz);
        m->values.assign(values, values + nnz);
        try {
            m->validate();
        } catch (...) {
            delete m;
            throw;
        }
        *out = m;
    });
}

void twref_matrix_free(void* h) { delete as_mat(h); }

std::int64_t twref_matrix_n(void* h) { return as_mat(h)->n; }
std::int64_t twref_matrix_nnz(void* h) { return as_mat(h)->nnz(); }

void twref_matrix_export(void* h, std::int64_t* row_ptr, std::int64_t* col_idx,
                         double* values) {
    auto* m = as_mat(h);
    std::copy(m->row_ptr.begin(), m->row_ptr.end(), row_ptr);
    std::copy(m->col_idx.begin(), m->col_idx.end(), col_idx);
    std::copy(m->values.begin(), m->values.end(), values);
}

// dump_csr (csr.cpp:61-74) into a caller buffer; returns the needed size.
std::int64_t twref_matrix_dump(void* h, char* buf, std::int64_t cap) {
    std::ostringstream os;
    tw::bench::dump_csr(*as_mat(h), os);
    std::string s = os.str();
    if (buf && cap > 0) {
        std::int64_t k = std::min<std::int64_t>(cap - 1, static_cast<std::int64_t>(s.size()));
        std::memcpy(buf, s.data(), static_cast<std::size_t>(k));
        buf[k] = '\0';
    }
    return static_cast<std::int64_t>(s.size()) + 1;
}

int twref_matrix_load(const char* text, void** out) {
    return guarded([&] {
        std::istringstream is(text);
        *out = new tw::bench::CsrMatrix(tw::bench::load_csr(is));
    });
}

void twref_spmv_range(void* h, const double* x, double* y, std::int64_t r0, std::int64_t r1) {
    tw::bench::spmv_range(*as_mat(h), x, y, r0, r1);
}

double twref_dot_range(const double* a, const double* b, std::int64_t i0, std::int64_t i1) {
    return tw::bench::dot_range(a, b, i0, i1);
}

void twref_waxpby_range(double alpha, const double* x, double beta, const double* y,
                        double* w, std::int64_t i0, std::int64_t i1) {
    tw::bench::waxpby_range(alpha, x, beta, y, w, i0, i1);
}

int twref_tile_plan(void* h, int tiles, std::int64_t* r0, std::int64_t* r1,
                    std::int64_t* band_lo, std::int64_t* band_hi) {
    return guarded([&] {
        auto plan = tw::bench::make_tile_plan(*as_mat(h), tiles);
        for (std::size_t t = 0; t < plan.size(); ++t) {
            r0[t] = plan[t].r0;
            r1[t] = plan[t].r1;
            band_lo[t] = plan[t].band_lo;
            band_hi[t] = plan[t].band_hi;
        }
    });
}

int twref_cg_reference(void* h, const double* b, int iterations, double tol, double* history,
                       double* x, int* converged) {
    return guarded([&] {
        auto* m = as_mat(h);
        std::vector<double> bv(b, b + m->n);
        auto r = tw::bench::cg_reference(*m, bv, iterations, tol);
        write_result(r, history, x);
        if (converged)
            *converged = r.converged ? 1 : 0;
    });
}

// The reference's task-based path.  variant 0 = cg_monolithic, 1 = cg_tasks.
// real_threads = 1 runs the threaded substrate with real_seconds_per_unit = 0
// (no synthetic busy-spin, substrate_threads.cpp:118-125), the only mode in
// which wall-clock is a CPU performance number.
// backend 0 = host, 1 = device_ta, 2 = device_blocking (simulated device).
// Returns wall seconds spent inside the solver call in *seconds.
// marks (nullable, `iterations` entries): the time of each cg_iter=i mark
// (cg.cpp:307-308, :427) in substrate seconds since the runtime started --
// the reference's own per-iteration timing (scenario.cpp:116-124).
int twref_cg_tasks(void* h, const double* b, int iterations, int variant, int tiles,
                   int workers, int real_threads, int backend, double* history, double* x,
                   double* seconds, double* marks) {
    return guarded([&] {
        auto* m = as_mat(h);
        std::vector<double> bv(b, b + m->n);
        tw::RuntimeConfig rc;
        rc.substrate.workers = static_cast<unsigned>(workers);
        if (real_threads) {
            rc.substrate.clock = tw::ClockMode::real_threads;
            rc.substrate.real_seconds_per_unit = 0.0;
        }
        if (backend != 0) {
            // the simulated arena must hold x|r|p|Ap|pa|rr (cg.cpp:92-97)
            std::size_t need = static_cast<std::size_t>(4 * m->n + 2 * tiles + 64) * 8;
            rc.device.arena_bytes = std::max<std::size_t>(rc.device.arena_bytes, need * 2);
        }
        tw::Runtime rt(rc);
        tw::bench::CgOptions opt;
        opt.tiles = tiles;
        opt.backend = backend == 0   ? tw::bench::CgBackend::host
                      : backend == 1 ? tw::bench::CgBackend::device_ta
                                     : tw::bench::CgBackend::device_blocking;
        auto t0 = std::chrono::steady_clock::now();
        tw::bench::CgResult r = variant == 0
                                    ? tw::bench::cg_monolithic(rt, *m, bv, iterations, opt)
                                    : tw::bench::cg_tasks(rt, *m, bv, iterations, opt);
        auto t1 = std::chrono::steady_clock::now();
        if (seconds)
            *seconds = std::chrono::duration<double>(t1 - t0).count();
        if (marks) {
            std::fill(marks, marks + iterations, 0.0);
            for (const tw::LogRecord& rec : rt.log().sorted())
                if (rec.transition == tw::Transition::mark && rec.note.rfind("cg_iter=", 0) == 0) {
                    const int i = std::stoi(rec.note.substr(sizeof("cg_iter=") - 1));
                    if (i >= 0 && i < iterations) marks[i] = rec.time;
                }
        }
        write_result(r, history, x);
    });
}

// Dependency edges the reference's depsys infers for cg_tasks (the block-task
// DAG of cg.cpp:166-334), as (pred_label, succ_label) lines "a b\n" in buf.
// Returns the needed size.  Virtual clock, host backend.
std::int64_t twref_cg_task_edges(void* h, const double* b, int iterations, int tiles,
                                 char* buf, std::int64_t cap) {
    std::string s;
    int rc_code = guarded([&] {
        auto* m = as_mat(h);
        std::vector<double> bv(b, b + m->n);
        tw::RuntimeConfig rc;
        rc.substrate.workers = 4;
        tw::Runtime rt(rc);
        tw::bench::CgOptions opt;
        opt.tiles = tiles;
        opt.iteration_marks = false;
        tw::bench::cg_tasks(rt, *m, bv, iterations, opt);
        std::ostringstream os;
        for (const auto& [a, c] : rt.deps().edges())
            os << rt.deps().label(a) << ' ' << rt.deps().label(c) << '\n';
        s = os.str();
    });
    if (rc_code != 0)
        return -1;
    if (buf && cap > 0) {
        std::int64_t k = std::min<std::int64_t>(cap - 1, static_cast<std::int64_t>(s.size()));
        std::memcpy(buf, s.data(), static_cast<std::size_t>(k));
        buf[k] = '\0';
    }
    return static_cast<std::int64_t>(s.size()) + 1;
}

} // extern "C"
