// Drop-in demonstration (test infrastructure): the reference's own CsrMatrix
// from its own gen_stencil_matrix goes through the binding of
// cg_cuda_binding.cpp into libtw_hpccg on the GPU, and the result is checked
// against the reference's own cg_reference -- the residual window rule of
// SURVEY.md 8(c) and 1e-10 on x.  Exit 0 and "binding ok" on success.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "taskweave/cg.hpp"
#include "taskweave/csr.hpp"
#include "tw_hpccg.h"

namespace tw::bench {
CgResult cg_cuda(const CsrMatrix& A, const std::vector<double>& b, int iterations,
                 const CgOptions& opt, int variant);
void cg_cuda_forget(const CsrMatrix& A);
std::uint64_t cg_cuda_cache_hits();
}

int main() {
    using namespace tw::bench;
    const CsrMatrix A = gen_stencil_matrix(32, 32, 32);
    // b = xorshift64 seed 7, 0.5 + (s % 1000) / 1000 (acceptance.cpp:48-58)
    std::vector<double> b(static_cast<size_t>(A.n));
    std::uint64_t s = 7;
    for (auto& v : b) {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        v = 0.5 + static_cast<double>(s % 1000) / 1000.0;
    }
    const int iters = 150;
    const CgResult want = cg_reference(A, b, iters);
    const double res0 = want.residual_history[0];
    int bad = 0;
    for (int variant : {TW_CG_MONOLITHIC, TW_CG_TASKS}) {
        CgOptions opt;
        opt.tiles = variant == TW_CG_MONOLITHIC ? 1 : 8;
        const CgResult got = cg_cuda(A, b, iters, opt, variant);
        for (int k = 0; k < iters; ++k) {
            const double w = want.residual_history[static_cast<size_t>(k)];
            const double g = got.residual_history[static_cast<size_t>(k)];
            const bool in_window = w >= 1e-15 * res0;
            const bool ok = in_window ? std::fabs(g - w) <= 1e-10 * std::fabs(w)
                                      : std::fabs(g - w) <= 1e-10 * res0;
            if (!ok) {
                std::printf("variant %d: residual %d differs: %.17g vs %.17g\n", variant, k, g, w);
                ++bad;
                break;
            }
        }
        for (size_t i = 0; i < got.x.size(); ++i)
            if (std::fabs(got.x[i] - want.x[i]) > 1e-10 * std::fabs(want.x[i])) {
                std::printf("variant %d: x[%zu] differs\n", variant, i);
                ++bad;
                break;
            }
    }
    // the device matrix was built once: the tasks solve reused it
    if (cg_cuda_cache_hits() != 1) {
        std::printf("ELL cache: %llu hits, want 1\n", (unsigned long long)cg_cuda_cache_hits());
        ++bad;
    }
    // a matrix changed in place is re-uploaded once forgotten
    CsrMatrix B = gen_stencil_matrix(8, 8, 8);
    std::vector<double> bb(static_cast<size_t>(B.n), 1.0);
    CgOptions o1;
    o1.tiles = 1;
    const CgResult r1 = cg_cuda(B, bb, 5, o1, TW_CG_MONOLITHIC);
    for (auto& v : B.values) v *= 2.0;
    cg_cuda_forget(B);
    const CgResult r2 = cg_cuda(B, bb, 5, o1, TW_CG_MONOLITHIC);
    if (!(std::fabs(2.0 * r2.x[0] - r1.x[0]) <= 1e-12 * std::fabs(r1.x[0]))) { // 2A: x halves
        std::printf("a forgotten matrix was not re-uploaded\n");
        ++bad;
    }
    if (bad) return 1;
    std::printf("binding ok: the reference's CsrMatrix through tw_cg_solve matches cg_reference "
                "(32^3, 150 iterations, monolithic and 8-tile tasks; device matrix cached)\n");
    return 0;
}
