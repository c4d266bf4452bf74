// Device helpers shared by the kernel translation units (tw_kernels.cu,
// tw_dag.cu): fixed-order reductions, the finalize step of the scalar
// state, mbarrier / TMA bulk-copy wrappers and the per-row SpMV bodies.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "tw_internal.h"

// Device-side checks of the checked build (make NVFLAGS_EXTRA=-DTW_CHECKS,
// scripts/gpu_checked.sh): the bounds compute-sanitizer would watch, as traps.
#ifdef TW_CHECKS
#define TW_DCHECK(c)                                                                       \
    do {                                                                                   \
        if (!(c)) {                                                                        \
            printf("tw_hpccg check failed: %s (%s:%d)\n", #c, __FILE__, __LINE__);        \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#else
#define TW_DCHECK(c) \
    do {             \
    } while (0)
#endif

namespace tw {
namespace dev {

constexpr int kThreads = 256;
#ifndef TW_TMA_WARPS
#define TW_TMA_WARPS 18
#endif
#ifndef TW_TMA_STAGES
#define TW_TMA_STAGES 1
#endif
constexpr int kTmaWarps = TW_TMA_WARPS;   // consumer warps per CTA (one CTA per SM)
constexpr int kTmaStages = TW_TMA_STAGES; // shared-memory stages per warp

// Grid for a grid-stride kernel of `work_threads` threads, at most `blocks`.
inline int clamp_blocks(int64_t work_threads, int blocks) {
    int64_t need = (work_threads + kThreads - 1) / kThreads;
    if (need < 1) need = 1;
    return static_cast<int>(need < blocks ? need : blocks);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide fixed-order sum; result valid in thread 0.
__device__ __forceinline__ double block_sum(double v, double* smem) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) smem[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0) {
        const int nw = blockDim.x >> 5;
        for (int w = 0; w < nw; ++w) t = __dadd_rn(t, smem[w]);
    }
    __syncthreads();
    return t;
}

// ------------------------------------ programmatic dependent launch (sm_90+)
// No-ops when the kernel was launched without the PDL attribute.
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Roles of a tile kernel in the tasks variant's programmatic chain (one
// stream, every tile kernel launched programmatically; tw_cg.cpp
// enqueue_tasks_chain), PdlRole in tw_internal.h.  A griddepcontrol.wait
// returns once every grid before it in the stream has completed (completion
// is in stream order: scripts/pdl_transitive.cu), so only a phase's first
// tile waits; it lets the next tile launch after its wait, so the later
// tiles start after the previous phase has completed and need no wait; the
// last tile lets the next phase's first tile launch only after its main loop
// (that tile's blocks then wait beside the phase's tail, not beside its bulk).
__device__ __forceinline__ void pdl_role_entry(int role) {
    if (role == PDL_DEFAULT || role == PDL_INNER) pdl_launch_dependents();
    if (role == PDL_DEFAULT || role == PDL_GATE || role == PDL_GATE_LAST) pdl_wait();
    if (role == PDL_GATE) pdl_launch_dependents();
}
#ifndef TW_CHAIN_EARLY_NEXT
#define TW_CHAIN_EARLY_NEXT 1 // 0: the last tile triggers only by completing (A/B)
#endif
__device__ __forceinline__ void pdl_role_exit(int role) {
    if (TW_CHAIN_EARLY_NEXT && (role == PDL_LAST || role == PDL_GATE_LAST)) pdl_launch_dependents();
}

// ------------------------------------------------ peer transport primitives

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Wrap-around ticket with acquire-release semantics at GPU scope.
__device__ __forceinline__ unsigned atom_inc_acq_rel(unsigned* p, unsigned wrap) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.inc.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(wrap)
                 : "memory");
    return old;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Flag stamp of the current iteration (+ahead): solve epoch << 32 | iter + 1.
__device__ __forceinline__ unsigned long long stamp_of(const CgScalars* sc, int ahead) {
    return (static_cast<unsigned long long>(sc->epoch) << 32) |
           static_cast<unsigned long long>(sc->iter + 1 + ahead);
}

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

#ifndef TW_PEER_TIMEOUT_NS
#define TW_PEER_TIMEOUT_NS 20000000000ull // 20 s: a peer that never publishes
#endif

// Block-wide: thread 0 acquire-spins until every flag carries `want`; the
// barrier extends the acquire to the block.  Call from uniform control flow.
// A flag that stays stale for TW_PEER_TIMEOUT_NS traps (the context reports
// an error to every later call) instead of hanging the GPU.
// One thread acquire-waits until every flag reaches `want`; a flag that has
// not after TW_PEER_TIMEOUT_NS traps (a dead peer ends the kernel with an
// error instead of hanging the GPU).
static __device__ __noinline__ void thread_wait_flags(const unsigned long long* flags, int count,
                                                      unsigned long long want) {
    unsigned long long t0 = 0;
    for (int i = 0; i < count; ++i) {
        unsigned spins = 0;
        while (ld_acquire_sys(flags + i) < want) {
            __nanosleep(32);
            if ((++spins & 4095u) == 0) {
                const unsigned long long t = global_ns();
                if (!t0) t0 = t;
                else if (t - t0 > TW_PEER_TIMEOUT_NS) {
                    printf("tw_hpccg: peer flag %d never reached stamp %llx (has %llx)\n", i, want,
                           ld_acquire_sys(flags + i));
                    __trap();
                }
            }
        }
    }
}

static __device__ __forceinline__ void block_wait_flags(const unsigned long long* flags, int count,
                                                        unsigned long long want) {
    if (threadIdx.x == 0) thread_wait_flags(flags, count, want);
    __syncthreads();
}

__device__ __forceinline__ void finalize(const Fin& fin, double total) {
    switch (fin.mode) {
    case FIN_STORE:
        *fin.out = total;
        break;
    case FIN_ALPHA:
        fin.sc->pAp = total;
        fin.sc->alpha_prev = fin.sc->alpha;
        fin.sc->alpha = __ddiv_rn(fin.sc->rtrans, total);
        break;
    case FIN_BETA: {
        CgScalars* sc = fin.sc;
        sc->rr = total;
        sc->beta = __ddiv_rn(total, sc->rtrans);
        sc->rtrans = total;
        if (sc->iter < sc->history_cap) fin.history[sc->iter] = __dsqrt_rn(total);
        sc->iter = sc->iter + 1;
        break;
    }
    case FIN_RTRANS:
        fin.sc->rtrans = total;
        fin.sc->iter = 0;
        break;
    case FIN_TILES: {
        *fin.out = total;
        __threadfence(); // the partial before the ticket
        const unsigned t = atomicInc(fin.tticket, static_cast<unsigned>(fin.ntiles - 1));
        if (t != static_cast<unsigned>(fin.ntiles - 1)) break; // wraps to 0: reset for the next use
        __threadfence();
        double s = 0.0;
        for (int i = 0; i < fin.ntiles; ++i) s = __dadd_rn(s, __ldcg(fin.tparts + i));
        CgScalars* sc = fin.sc;
        if (fin.then == FIN_ALPHA) {
            sc->pAp = s;
            sc->alpha_prev = sc->alpha;
            sc->alpha = __ddiv_rn(sc->rtrans, s);
        } else {
            sc->rr = s;
            sc->beta = __ddiv_rn(s, sc->rtrans);
            sc->rtrans = s;
            if (sc->iter < sc->history_cap) fin.history[sc->iter] = __dsqrt_rn(s);
            sc->iter = sc->iter + 1;
        }
        break;
    }
    case FIN_PUBLISH_A:
    case FIN_PUBLISH_B: {
        if (fin.out) *fin.out = total;
        const double v = fin.pre ? __dadd_rn(__dadd_rn(0.0, *fin.pre), total) : total;
        const PeerLinks* L = fin.links;
        const bool a = fin.mode == FIN_PUBLISH_A;
        const int me = L->rank, P = L->nranks;
        TW_DCHECK(P >= 1 && P <= kMaxRanks && me >= 0 && me < P);
        // one thread stores the values, then the flags with release
        // semantics: each st.release.sys orders this thread's earlier value
        // stores before the flag (no separate system fence needed)
        for (int q = 0; q < P; ++q) (a ? L->win[q]->recv_a : L->win[q]->recv_b)[me] = v;
        const unsigned long long st = stamp_of(fin.sc, 0);
        for (int q = 0; q < P; ++q) st_release_sys((a ? L->win[q]->flag_a : L->win[q]->flag_b) + me, st);
        break;
    }
    default:
        break;
    }
}

// The blocks a body runs on: the launch grid, or one rank's share of the
// grid of the concurrent rank-group kernel (bid in [0, nblk)).
struct GridPos {
    int bid, nblk;
};

__device__ __forceinline__ GridPos launch_grid() {
    return GridPos{static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x)};
}

// Grid-wide fixed-order reduction finished by the last block to arrive.
__device__ __forceinline__ void grid_reduce_finalize(double v, RedScratch rs, const Fin& fin,
                                                     GridPos g = launch_grid()) {
    __shared__ double smem[32];
    __shared__ bool last;
    double b = block_sum(v, smem);
    if (threadIdx.x == 0) {
        rs.block_part[g.bid] = b;
        __threadfence();
        unsigned t = atomicInc(rs.ticket, static_cast<unsigned>(g.nblk - 1));
        last = (t == static_cast<unsigned>(g.nblk - 1));
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double acc = 0.0;
    for (int i = threadIdx.x; i < g.nblk; i += blockDim.x)
        acc = __dadd_rn(acc, __ldcg(rs.block_part + i));
    double total = block_sum(acc, smem);
    if (threadIdx.x == 0) finalize(fin, total);
}

// Two fixed-order reductions in one pass (K1's interior and boundary p.Ap
// partials): each is the tree grid_reduce_finalize would build on its own.
// The last block stores the first total to *fin.pre and finalizes the
// second with fin (FIN_PUBLISH_A reads *fin.pre back).
__device__ __forceinline__ void grid_reduce2_finalize(double va, double vb, RedScratch rs,
                                                      const Fin& fin, GridPos g = launch_grid()) {
    __shared__ double smem[32];
    __shared__ bool last;
    const double ba = block_sum(va, smem);
    const double bb = block_sum(vb, smem);
    if (threadIdx.x == 0) {
        rs.block_part[2 * g.bid] = ba;
        rs.block_part[2 * g.bid + 1] = bb;
        __threadfence();
        const unsigned t = atomicInc(rs.ticket, static_cast<unsigned>(g.nblk - 1));
        last = (t == static_cast<unsigned>(g.nblk - 1));
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double acc_a = 0.0, acc_b = 0.0;
    for (int i = threadIdx.x; i < g.nblk; i += blockDim.x) {
        acc_a = __dadd_rn(acc_a, __ldcg(rs.block_part + 2 * i));
        acc_b = __dadd_rn(acc_b, __ldcg(rs.block_part + 2 * i + 1));
    }
    const double ta = block_sum(acc_a, smem);
    const double tb = block_sum(acc_b, smem);
    if (threadIdx.x == 0) {
        *const_cast<double*>(fin.pre) = ta;
        finalize(fin, tb);
    }
}

__device__ __forceinline__ double sum_parts(const double* parts, int count) {
    double t = 0.0;
    for (int i = 0; i < count; ++i) t = __dadd_rn(t, __ldcg(parts + i));
    return t;
}

// ----------------------------------------------- K1 with TMA-staged matrix

// The matrix stream (12 B per nonzero, 95% of K1's bytes) is moved by the
// Tensor Memory Accelerator: every warp owns a ring of S shared-memory
// stages and keeps S slice blocks (values + columns, contiguous in HBM) in
// flight with cp.async.bulk, completing on a per-stage mbarrier.  The warp
// computes slice k from shared memory while slices k+1..k+S-1 stream in, so
// DRAM sees deep memory-level parallelism regardless of the gather latency
// of x (which stays on the L1/L2 path with __ldg).  The matrix copies carry
// an L2 evict-first policy so the p planes being gathered stay L2-resident.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// Cache hints of the produced vectors (same-box A/Bs in
// profiles/r02_ab_k2k3_sweep.md): K1 stores Ap with L2 evict_last, so K2
// finds more of it in L2 (256^3: K2 68 -> 62 us, iteration -4.3 us); K3
// stores p with evict_last for the next K1 (128^3 -0.6 %, neutral at 256^3);
// K2's r keeps the default policy (evict_last there: neutral).
#ifndef TW_K3_P_KEEP
#define TW_K3_P_KEEP 1
#endif
#ifndef TW_K1_AP_KEEP
#define TW_K1_AP_KEEP 1
#endif
__device__ __forceinline__ void st_evict_last(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st2_evict_last(double* p, double2 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y),
                 "l"(pol)
                 : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// The same without a cache-policy hint (vectors that are read again soon).
__device__ __forceinline__ void bulk_g2s_plain(void* dst, const void* src, uint32_t bytes,
                                               uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// One row of a width-W slice block resident in shared memory: columns first,
// then every gather issued before any use, then the reference's ordered sum.
// Gather of x (G):
//   kGatherNC (1): the read-only path, x constant for the whole kernel;
//   kGatherCA (0): a coherent L1-cached load (the DAG dispatcher, where p is
//                  rewritten inside the same kernel between dependent tasks);
//   kGatherCG (2): L2 only, bypassing L1 -- ghost planes written by another
//                  GPU while this kernel runs: an L1 line that also holds the
//                  edge of an owned plane may have been cached before the
//                  ghost flag was acquired.
constexpr int kGatherCA = 0, kGatherNC = 1, kGatherCG = 2;
template <int G>
__device__ __forceinline__ double gather(const double* x, int c) {
    if (G == kGatherNC) return __ldg(x + c);
    if (G == kGatherCG) return __ldcg(x + c);
    return __ldca(x + c); // ld.global.ca: L1-cached, coherent after the acquire + L1 invalidate
}

template <int W, int NC = kGatherNC>
__device__ __forceinline__ double smem_row_fixed(const double* vb, const int32_t* cb,
                                                 const double* x, int lane) {
    int c[W];
#pragma unroll
    for (int q = 0; q < W / 4; ++q) {
        int4 t = reinterpret_cast<const int4*>(cb + 128 * q)[lane];
        c[4 * q] = t.x;
        c[4 * q + 1] = t.y;
        c[4 * q + 2] = t.z;
        c[4 * q + 3] = t.w;
    }
    constexpr int F = W & ~3;
    if (W - F >= 2) {
        int2 t = reinterpret_cast<const int2*>(cb + 32 * F)[lane];
        c[F] = t.x;
        c[F + 1] = t.y;
    }
    if ((W - F) & 1) c[W - 1] = cb[32 * (W - 1) + lane];
    double xv[W];
#pragma unroll
    for (int k = 0; k < W; ++k) xv[k] = gather<NC>(x, max(c[k], 0)); // branch-free: padding loads x[0], masked below
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < W / 2; ++j) {
        double2 v = reinterpret_cast<const double2*>(vb + 64 * j)[lane];
        if (c[2 * j] >= 0) acc = __dadd_rn(acc, __dmul_rn(v.x, xv[2 * j]));
        if (c[2 * j + 1] >= 0) acc = __dadd_rn(acc, __dmul_rn(v.y, xv[2 * j + 1]));
    }
    if (W & 1)
        if (c[W - 1] >= 0) acc = __dadd_rn(acc, __dmul_rn(vb[32 * (W - 1) + lane], xv[W - 1]));
    return acc;
}

template <int NC = kGatherNC>
__device__ __forceinline__ double smem_row_generic(const double* vb, const int32_t* cb,
                                                   const double* x, int lane, int w) {
    double acc = 0.0;
    for (int k = 0; k < w; ++k) {
        const int c = cb[ell_col_pos(k, lane, w)];
        if (c < 0) break;
        acc = __dadd_rn(acc, __dmul_rn(vb[ell_val_pos(k, lane, w)], gather<NC>(x, c)));
    }
    return acc;
}

// One row of an x-staged slice: 16-bit columns index the slice's 9 staged
// runs of x in shared memory, so the 27 operands are shared-memory reads of
// data that arrived with the slice's own TMA transaction (no global gathers
// waiting on L1 / L2).  Same per-row order and roundings as smem_row_fixed.
template <int W>
__device__ __forceinline__ double staged_row_fixed(const double* vb, const uint16_t* cb,
                                                   const double* xs, int lane) {
    uint32_t c[W];
#pragma unroll
    for (int q = 0; q < W / 8; ++q) {
        const uint4 t = reinterpret_cast<const uint4*>(cb + 256 * q)[lane];
        const uint32_t w4[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            c[8 * q + 2 * h] = w4[h] & 0xFFFFu;
            c[8 * q + 2 * h + 1] = w4[h] >> 16;
        }
    }
    constexpr int F8 = W & ~7;
    constexpr int R = W - F8;
    constexpr int F4 = R >= 4 ? F8 + 4 : F8;
    if (R >= 4) {
        const uint2 t = reinterpret_cast<const uint2*>(cb + 32 * F8)[lane];
        c[F8] = t.x & 0xFFFFu;
        c[F8 + 1] = t.x >> 16;
        c[F8 + 2] = t.y & 0xFFFFu;
        c[F8 + 3] = t.y >> 16;
    }
    constexpr int R2 = W - F4;
    if (R2 >= 2) {
        const uint32_t t = reinterpret_cast<const uint32_t*>(cb + 32 * F4)[lane];
        c[F4] = t & 0xFFFFu;
        c[F4 + 1] = t >> 16;
    }
    if (R2 & 1) c[W - 1] = cb[32 * (W - 1) + lane];
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < W / 2; ++j) {
        const double2 v = reinterpret_cast<const double2*>(vb + 64 * j)[lane];
        if (c[2 * j] != kStagePad) acc = __dadd_rn(acc, __dmul_rn(v.x, xs[c[2 * j]]));
        if (c[2 * j + 1] != kStagePad) acc = __dadd_rn(acc, __dmul_rn(v.y, xs[c[2 * j + 1]]));
    }
    if (W & 1)
        if (c[W - 1] != kStagePad) acc = __dadd_rn(acc, __dmul_rn(vb[32 * (W - 1) + lane], xs[c[W - 1]]));
    return acc;
}

__device__ __forceinline__ double staged_row_generic(const double* vb, const uint16_t* cb,
                                                     const double* xs, int lane, int w) {
    double acc = 0.0;
    for (int k = 0; k < w; ++k) {
        const uint32_t c = cb[ell_c16_pos(k, lane, w)];
        if (c == kStagePad) break; // padding only ever trails a row
        acc = __dadd_rn(acc, __dmul_rn(vb[ell_val_pos(k, lane, w)], xs[c]));
    }
    return acc;
}

} // namespace dev
} // namespace tw
