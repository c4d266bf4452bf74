// The reference-side binding of INTEGRATION.md section 2, as a maintainer
// would add it to proj/src/cg.cpp: a `cuda` CgBackend routed to the C ABI.
// tests/test_binding_cpu.py compiles it against the reference's own headers
// (/root/reference/proj/include) and links it against libtw_hpccg.so with
// --no-undefined, so every ABI call below resolves.  Not part of the product.
#include <vector>

#include "taskweave/cg.hpp"
#include "taskweave/csr.hpp"
#include "taskweave/types.hpp"
#include "tw_hpccg.h"

namespace tw::bench {
namespace {

struct TwCtx { // one device context per process (Runtime + sim::Device replacement)
    tw_ctx* h = nullptr;
    explicit TwCtx(unsigned pool) { check(tw_ctx_create(0, pool, &h)); }
    ~TwCtx() { tw_ctx_destroy(h); }
    static void check(int rc) {
        if (rc == TW_ERR_CONFIG) throw ConfigError(tw_last_error_string());
        if (rc != TW_OK) throw ContractViolation(tw_last_error_string());
    }
};

} // namespace

CgResult cg_cuda(const CsrMatrix& A, const std::vector<double>& b, int iterations,
                 const CgOptions& opt, int variant) {
    static TwCtx ctx(opt.stream_pool_capacity);
    tw_ell* ell = nullptr; // CsrMatrix -> device sliced ELL (validated like csr.cpp:13-27)
    TwCtx::check(tw_ell_from_csr(ctx.h, A.n, A.row_ptr.data(), A.col_idx.data(),
                                 A.values.data(), &ell));
    tw_cg_options o;
    tw_cg_options_default(&o);
    o.variant = variant; // TW_CG_MONOLITHIC | TW_CG_TASKS
    o.tiles = opt.tiles;
    o.stream_pool_capacity = opt.stream_pool_capacity;
    o.iteration_marks = opt.iteration_marks;
    o.tol = opt.tol;
    CgResult res;
    res.residual_history.resize(static_cast<size_t>(iterations));
    res.x.resize(static_cast<size_t>(A.n));
    int conv = 0;
    const int rc = tw_cg_solve(ctx.h, ell, b.data(), iterations, &o, res.residual_history.data(),
                               res.x.data(), &conv);
    tw_ell_destroy(ell);
    TwCtx::check(rc);
    res.iterations = iterations;
    res.converged = conv != 0;
    return res;
}

// spmv_body's device_ta case: one tile of the
// reference's own task DAG on a pooled stream, released by the poller.
void spmv_tile_cuda(tw_ctx* ctx, const tw_ell* ell, const double* p_dev, double* Ap_dev,
                    std::int64_t r0, std::int64_t r1, void (*release_dependents)(void*),
                    void* task) {
    void* s = nullptr;
    TwCtx::check(tw_stream_acquire(ctx, &s));
    TwCtx::check(tw_spmv_range(ell, p_dev, Ap_dev, r0, r1, s));
    void* ev = nullptr;
    TwCtx::check(tw_event_create(&ev));
    TwCtx::check(tw_event_record(ev, s));
    TwCtx::check(tw_event_bind_async(ctx, ev, release_dependents, task));
    TwCtx::check(tw_stream_release(ctx, s));
}

} // namespace tw::bench
