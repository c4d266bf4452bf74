// sm_100a kernels of the HPCCG hot path (the matrix builders, K0, live in
// tw_ell_build.cu).
//
//   K1  SpMV fused with p.Ap                        (spmv_range + dot_range, kernels.cpp:5-20)
//   K2  x += a p ; r -= a Ap ; r.r                  (2x waxpby_range + dot_range, kernels.cpp:15-26)
//   K3  p = r + b p                                 (waxpby_range, kernels.cpp:22-26)
//   K4  dot / waxpby standalone, scalar combines
//
// Everything here is HBM-bound f64 streaming (0.16 flop/byte, far below the
// FP64 ridge), so the design levers are: 128-bit coalesced loads of the
// matrix with evict-first (__ldcs) so the gathered vector stays in L1/L2,
// grids sized to SMs x resident blocks with warps of a block walking
// neighbouring slices (shared x-lines hit L1), and fused reductions that
// finish in the last block (no extra launch, no host round trip).
//
// Arithmetic parity: this file is compiled with --fmad=false and uses
// __dmul_rn/__dadd_rn explicitly, so every product and sum rounds exactly as
// the reference's x86-64 build (no FMA).  Dot products are
// fixed-order trees: deterministic run to run, within reassociation error of
// the reference's sequential sums (SURVEY.md 8(c) tolerance rule).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <utility>

#include "tw_device.cuh"
#include "tw_internal.h"

namespace tw {

namespace {

#ifdef TW_TIMELINE
// Probe builds only (scripts/timeline.py): one record per CTA of the
// annotated kernels -- tag | SM | block, the first row of its range, and
// thread 0's globaltimer at entry and exit.  Not in the product library.
constexpr unsigned kTlCap = 1u << 20;
__device__ unsigned long long tw_tl_buf[kTlCap][4];
__device__ unsigned tw_tl_n;
struct TlScope {
    unsigned long long t0, i0;
    int tag;
    __device__ TlScope(int t, int64_t first) : t0(0), i0(static_cast<unsigned long long>(first)), tag(t) {
        if (threadIdx.x == 0) t0 = dev::global_ns();
    }
    __device__ ~TlScope() {
        if (threadIdx.x != 0) return;
        const unsigned long long t1 = dev::global_ns();
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        const unsigned k = atomicAdd(&tw_tl_n, 1u);
        if (k >= kTlCap) return;
        tw_tl_buf[k][0] = static_cast<unsigned long long>(tag) | (static_cast<unsigned long long>(sm) << 8) |
                          (static_cast<unsigned long long>(blockIdx.x) << 16);
        tw_tl_buf[k][1] = i0;
        tw_tl_buf[k][2] = t0;
        tw_tl_buf[k][3] = t1;
    }
};
#define TW_TL(tag, first) TlScope tw_tl_scope_((tag), (first))
#else
#define TW_TL(tag, first)
#endif

using namespace dev;


// ------------------------------------------------------------------ K1 SpMV

// One row of a width-W slice: all matrix loads issued up front as 128-bit
// evict-first loads, then the gathers, then the reference's left-to-right
// sum (acc from 0.0, multiply then add).
template <int W, int NC = kGatherNC>
__device__ __forceinline__ double slice_row_fixed(const double* __restrict__ vb,
                                                  const int32_t* __restrict__ cb,
                                                  const double* __restrict__ x, int lane) {
    double v[W];
    int c[W];
#pragma unroll
    for (int j = 0; j < W / 2; ++j) {
        double2 t = __ldcs(reinterpret_cast<const double2*>(vb + 64 * j) + lane);
        v[2 * j] = t.x;
        v[2 * j + 1] = t.y;
    }
    if (W & 1) v[W - 1] = __ldcs(vb + 32 * (W - 1) + lane);
#pragma unroll
    for (int q = 0; q < W / 4; ++q) {
        int4 t = __ldcs(reinterpret_cast<const int4*>(cb + 128 * q) + lane);
        c[4 * q] = t.x;
        c[4 * q + 1] = t.y;
        c[4 * q + 2] = t.z;
        c[4 * q + 3] = t.w;
    }
    constexpr int F = W & ~3;
    if (W - F >= 2) {
        int2 t = __ldcs(reinterpret_cast<const int2*>(cb + 32 * F) + lane);
        c[F] = t.x;
        c[F + 1] = t.y;
    }
    if ((W - F) & 1) c[W - 1] = __ldcs(cb + 32 * (W - 1) + lane);
    double xv[W];
#pragma unroll
    for (int k = 0; k < W; ++k) xv[k] = gather<NC>(x, max(c[k], 0)); // branch-free: padding loads x[0], masked below
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < W; ++k)
        if (c[k] >= 0) acc = __dadd_rn(acc, __dmul_rn(v[k], xv[k]));
    return acc;
}

template <int NC = kGatherNC>
__device__ __forceinline__ double slice_row_generic(const double* __restrict__ vb,
                                                    const int32_t* __restrict__ cb,
                                                    const double* __restrict__ x, int lane,
                                                    int w) {
    double acc = 0.0;
    for (int k = 0; k < w; ++k) {
        int c = __ldcs(cb + ell_col_pos(k, lane, w));
        if (c < 0) break; // padding only ever trails a row
        double v = __ldcs(vb + ell_val_pos(k, lane, w));
        acc = __dadd_rn(acc, __dmul_rn(v, gather<NC>(x, c)));
    }
    return acc;
}

// Register-path K1 body on the blocks of `g`.  NC: x is constant for the
// whole kernel (read-only path); the concurrent rank-group kernel, which
// rewrites p between its phases, gathers through the coherent L1 path.
template <bool DOT, int NC = kGatherNC>
__device__ __forceinline__ void spmv_rows(GridPos g, const EllView& A, const double* __restrict__ x,
                                          double* __restrict__ y, RowRange ra, RowRange rb,
                                          RedScratch rs, const Fin& fin,
                                          const unsigned long long* wait_flags, int nwait) {
    if (nwait) block_wait_flags(wait_flags, nwait, stamp_of(fin.sc, 0));
    const int lane = threadIdx.x & 31;
    const int64_t warp_g = (static_cast<int64_t>(g.bid) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(g.nblk) * blockDim.x) >> 5;
    // The slices covering range a, then those covering range b, as one index space.
    const int64_t sa0 = ra.r0 >> 5, sa1 = ra.r1 > ra.r0 ? (ra.r1 + 31) >> 5 : sa0;
    const int64_t sb0 = rb.r0 >> 5, sb1 = rb.r1 > rb.r0 ? (rb.r1 + 31) >> 5 : sb0;
    const int64_t na = sa1 - sa0, ntot = na + (sb1 - sb0);
    double part = 0.0;
    for (int64_t i = warp_g; i < ntot; i += nwarps) {
        const bool in_a = i < na;
        const int64_t s = in_a ? sa0 + i : sb0 + (i - na);
        const int64_t off = __ldg(A.slice_off + s);
        const int w = static_cast<int>((__ldg(A.slice_off + s + 1) - off) >> 5);
        const double* vb = A.vals + off;
        const int32_t* cb = A.cols + off;
        double acc;
        switch (w) {
        case 27: acc = slice_row_fixed<27, NC>(vb, cb, x, lane); break;
        case 18: acc = slice_row_fixed<18, NC>(vb, cb, x, lane); break;
        case 12: acc = slice_row_fixed<12, NC>(vb, cb, x, lane); break;
        case 8: acc = slice_row_fixed<8, NC>(vb, cb, x, lane); break;
        default: acc = slice_row_generic<NC>(vb, cb, x, lane, w); break;
        }
        const int64_t row = (s << 5) + lane;
        const RowRange r = in_a ? ra : rb;
        if (row >= r.r0 && row < r.r1) {
            y[row] = acc;
            if (DOT) part = __dadd_rn(part, __dmul_rn(gather<NC>(x, row + A.diag_shift), acc));
        }
    }
    if (DOT) grid_reduce_finalize(part, rs, fin, g);
}

template <bool DOT>
__global__ void __launch_bounds__(kThreads)
spmv_kernel(EllView A, const double* __restrict__ x, double* __restrict__ y, RowRange ra,
            RowRange rb, RedScratch rs, Fin fin, const unsigned long long* wait_flags, int nwait) {
    spmv_rows<DOT>(launch_grid(), A, x, y, ra, rb, rs, fin, wait_flags, nwait);
}


template <bool DOT>
__global__ void __launch_bounds__(kTmaWarps * 32, 1)
spmv_tma_kernel(EllView A, const double* __restrict__ x, double* __restrict__ y, RowRange ra,
                RowRange rb, int stage_bytes, int val_bytes, RedScratch rs, Fin fin,
                const unsigned long long* wait_flags, int nwait) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bars[kTmaWarps][kTmaStages];
    __shared__ int stage_w[kTmaWarps][kTmaStages];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* ring = smem + static_cast<size_t>(warp) * kTmaStages * stage_bytes;
    const int64_t warp_g = static_cast<int64_t>(blockIdx.x) * kTmaWarps + warp;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kTmaWarps;
    const int64_t sa0 = ra.r0 >> 5, sa1 = ra.r1 > ra.r0 ? (ra.r1 + 31) >> 5 : sa0;
    const int64_t sb0 = rb.r0 >> 5, sb1 = rb.r1 > rb.r0 ? (rb.r1 + 31) >> 5 : sb0;
    const int64_t na = sa1 - sa0, ntot = na + (sb1 - sb0);
    const int64_t mine = warp_g < ntot ? (ntot - warp_g + nwarps - 1) / nwarps : 0;
    auto slice_of = [&](int64_t k) {
        const int64_t i = warp_g + k * nwarps;
        return i < na ? sa0 + i : sb0 + (i - na);
    };
    pdl_launch_dependents(); // programmatic launch: the next kernel may queue up now
    if (lane == 0)
        for (int s = 0; s < kTmaStages; ++s) mbar_init(&bars[warp][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const uint64_t pol = l2_evict_first_policy();
    auto issue = [&](int64_t k, int st) {
        const int64_t s = slice_of(k);
        const int64_t off = A.slice_off[s], end = A.slice_off[s + 1];
        const uint32_t ents = static_cast<uint32_t>(end - off);
        TW_DCHECK(s >= 0 && s < A.n_slices && ents <= 32u * static_cast<uint32_t>(A.max_width));
        stage_w[warp][st] = static_cast<int>(ents >> 5);
        unsigned char* dst = ring + static_cast<size_t>(st) * stage_bytes;
        mbar_expect_tx(&bars[warp][st], ents * 12u); // ents == 0 (all rows empty): completes at once
        if (ents) {
            bulk_g2s(dst, A.vals + off, ents * 8u, &bars[warp][st], pol);
            bulk_g2s(dst + val_bytes, A.cols + off, ents * 4u, &bars[warp][st], pol);
        }
    };
    if (lane == 0)
        for (int st = 0; st < kTmaStages && st < mine; ++st) issue(st, st);
    __syncwarp();
    // The matrix does not depend on the previous kernel, so its first slice
    // streams in before the wait for that kernel's p (and scalars).
    pdl_wait();
    // peer transport: the matrix is already streaming in; the gathers of p
    // wait until the neighbours' ghost planes have landed
    if (nwait) block_wait_flags(wait_flags, nwait, stamp_of(fin.sc, 0));
    double part = 0.0;
    for (int64_t k = 0; k < mine; ++k) {
        const int st = static_cast<int>(k % kTmaStages);
        mbar_wait(&bars[warp][st], static_cast<uint32_t>((k / kTmaStages) & 1));
        const int w = stage_w[warp][st];
        const double* vb = reinterpret_cast<const double*>(ring + static_cast<size_t>(st) * stage_bytes);
        const int32_t* cb = reinterpret_cast<const int32_t*>(ring + static_cast<size_t>(st) * stage_bytes + val_bytes);
        double acc;
        switch (w) {
        case 27: acc = smem_row_fixed<27>(vb, cb, x, lane); break;
        case 18: acc = smem_row_fixed<18>(vb, cb, x, lane); break;
        case 12: acc = smem_row_fixed<12>(vb, cb, x, lane); break;
        case 8: acc = smem_row_fixed<8>(vb, cb, x, lane); break;
        default: acc = smem_row_generic<true>(vb, cb, x, lane, w); break;
        }
        const int64_t s = slice_of(k);
        const int64_t row = (s << 5) + lane;
        const RowRange rr = (warp_g + k * nwarps) < na ? ra : rb;
        if (row >= rr.r0 && row < rr.r1) {
            y[row] = acc;
            if (DOT) part = __dadd_rn(part, __dmul_rn(__ldg(x + row + A.diag_shift), acc));
        }
        __syncwarp();
        if (lane == 0 && k + kTmaStages < mine) {
            // generic-proxy reads of this stage are done; hand it back to TMA
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(k + kTmaStages, st);
        }
        __syncwarp();
    }
    if (DOT) grid_reduce_finalize(part, rs, fin);
}

// K1 of the peer transport in ONE launch: the interior rows, then -- after
// this warp's acquire of the ghost-plane flags -- the two boundary ranges.
// Each index space is walked exactly as the separate interior / boundary
// launches walk it (same grid, same slice-to-warp map) and the two p.Ap
// partials reduce separately, so pm[0] / pm[1] are bit-identical to the
// two-launch path (and to the NCCL transport).  The last block stores
// pm[0] and publishes (0 + pm[0]) + pm[1] (FIN_PUBLISH_A).
__global__ void __launch_bounds__(kTmaWarps * 32, 1)
spmv_tma_split_kernel(EllView A, const double* __restrict__ x, double* __restrict__ y,
                      RowRange ri, RowRange rb0, RowRange rb1, int stage_bytes, int val_bytes,
                      RedScratch rs, Fin fin, const unsigned long long* wait_flags, int nwait) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bars[kTmaWarps];
    __shared__ int stage_w[kTmaWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* stage = smem + static_cast<size_t>(warp) * stage_bytes;
    const int64_t warp_g = static_cast<int64_t>(blockIdx.x) * kTmaWarps + warp;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kTmaWarps;
    auto first = [](RowRange q) { return q.r0 >> 5; };
    auto count = [](RowRange q) { return q.r1 > q.r0 ? ((q.r1 + 31) >> 5) - (q.r0 >> 5) : int64_t(0); };
    const int64_t ni = count(ri), nb0 = count(rb0), nb = nb0 + count(rb1);
    const int64_t mine_i = warp_g < ni ? (ni - warp_g + nwarps - 1) / nwarps : 0;
    const int64_t mine_b = warp_g < nb ? (nb - warp_g + nwarps - 1) / nwarps : 0;
    // the k-th slice of this warp: interior ones first, then boundary ones
    auto slice_of = [&](int64_t k) {
        if (k < mine_i) return first(ri) + warp_g + k * nwarps;
        const int64_t i = warp_g + (k - mine_i) * nwarps;
        return i < nb0 ? first(rb0) + i : first(rb1) + (i - nb0);
    };
    auto range_of = [&](int64_t k) {
        if (k < mine_i) return ri;
        return warp_g + (k - mine_i) * nwarps < nb0 ? rb0 : rb1;
    };
    pdl_launch_dependents();
    if (lane == 0) mbar_init(&bars[warp], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const uint64_t pol = l2_evict_first_policy();
    auto issue = [&](int64_t k) {
        const int64_t s = slice_of(k);
        const int64_t off = A.slice_off[s];
        const uint32_t ents = static_cast<uint32_t>(A.slice_off[s + 1] - off);
        TW_DCHECK(s >= 0 && s < A.n_slices && ents <= 32u * static_cast<uint32_t>(A.max_width));
        stage_w[warp] = static_cast<int>(ents >> 5);
        mbar_expect_tx(&bars[warp], ents * 12u);
        if (ents) {
            bulk_g2s(stage, A.vals + off, ents * 8u, &bars[warp], pol);
            bulk_g2s(stage + val_bytes, A.cols + off, ents * 4u, &bars[warp], pol);
        }
    };
    const int64_t mine = mine_i + mine_b;
    if (lane == 0 && mine > 0) issue(0);
    __syncwarp();
    pdl_wait(); // p and the scalars come from the previous kernel
    const unsigned long long want = nwait ? stamp_of(fin.sc, 0) : 0ull;
    double part_i = 0.0, part_b = 0.0;
    const double* vb = reinterpret_cast<const double*>(stage);
    const int32_t* cb = reinterpret_cast<const int32_t*>(stage + val_bytes);
    for (int64_t k = 0; k < mine; ++k) {
        if (k == mine_i && nwait) { // first boundary slice: the ghost planes must have landed
            if (lane == 0) thread_wait_flags(wait_flags, nwait, want);
            __syncwarp();
        }
        mbar_wait(&bars[warp], static_cast<uint32_t>(k & 1));
        const int w = stage_w[warp];
        double acc;
        if (k < mine_i) {
            switch (w) {
            case 27: acc = smem_row_fixed<27>(vb, cb, x, lane); break;
            case 18: acc = smem_row_fixed<18>(vb, cb, x, lane); break;
            case 12: acc = smem_row_fixed<12>(vb, cb, x, lane); break;
            case 8: acc = smem_row_fixed<8>(vb, cb, x, lane); break;
            default: acc = smem_row_generic<kGatherNC>(vb, cb, x, lane, w); break;
            }
        } else { // boundary rows gather ghost planes that landed during this kernel
            switch (w) {
            case 27: acc = smem_row_fixed<27, kGatherCG>(vb, cb, x, lane); break;
            case 18: acc = smem_row_fixed<18, kGatherCG>(vb, cb, x, lane); break;
            case 12: acc = smem_row_fixed<12, kGatherCG>(vb, cb, x, lane); break;
            case 8: acc = smem_row_fixed<8, kGatherCG>(vb, cb, x, lane); break;
            default: acc = smem_row_generic<kGatherCG>(vb, cb, x, lane, w); break;
            }
        }
        const int64_t row = (slice_of(k) << 5) + lane;
        const RowRange rr = range_of(k);
        if (row >= rr.r0 && row < rr.r1) {
            y[row] = acc;
            const double d = __dmul_rn(__ldcg(x + row + A.diag_shift), acc);
#ifdef TW_BREAK_SPLIT // negative control of the bit-identity test only: one partial
            part_i = __dadd_rn(part_i, d);
#else
            if (k < mine_i) part_i = __dadd_rn(part_i, d);
            else part_b = __dadd_rn(part_b, d);
#endif
        }
        __syncwarp();
        if (lane == 0 && k + 1 < mine) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(k + 1);
        }
        __syncwarp();
    }
    grid_reduce2_finalize(part_i, part_b, rs, fin);
}

// ------------------------------------------------------ K1, x staged in smem
// (row bodies staged_row_fixed / staged_row_generic: tw_device.cuh)

// Up to three row ranges walked as one index space of slices (range k's
// slices follow range k-1's), the order launch_spmv walks its two in.
struct SliceSpace {
    RowRange q[3];
    int64_t c0, c1, n; // slices of q[0], of q[0] ++ q[1], of all three
    __device__ static int64_t count(RowRange r) {
        return r.r1 > r.r0 ? ((r.r1 + 31) >> 5) - (r.r0 >> 5) : int64_t(0);
    }
    __device__ SliceSpace(RowRange a, RowRange b, RowRange c) : q{a, b, c} {
        c0 = count(a);
        c1 = c0 + count(b);
        n = c1 + count(c);
    }
    __device__ int which(int64_t i) const { return i < c0 ? 0 : i < c1 ? 1 : 2; }
    __device__ int64_t slice(int64_t i, int w) const {
        return (q[w].r0 >> 5) + i - (w == 0 ? 0 : w == 1 ? c0 : c1);
    }
};

// K1 on an x-staged matrix: per warp one stage holding the slice's values,
// 16-bit columns and 9 x runs, one mbarrier transaction.  The warp's slices
// are those of space A (split only: the interior rows) and then of space B;
// B's x runs wait for the warp's acquire of the ghost-plane flags when there
// are any, and with SPLIT the two spaces keep separate p.Ap partials, so the
// results are bit-identical to one launch per space (the NCCL transport).
// NW warps per block over the blocks of g; `phase` counts the waits already
// done on the warp's barrier (a kernel that calls the body repeatedly keeps
// it); PDL: the programmatic-launch wait sits between the first slice's
// matrix block and its x runs.
template <bool SPLIT, int NW, bool PDL, bool KEEP = false>
__device__ __forceinline__ void staged_spmv_body(
    GridPos g, const EllView& A, const double* __restrict__ x, double* __restrict__ y, RowRange ra,
    RowRange rb0, RowRange rb1, int stage_bytes, int val_bytes, int c16_bytes, RedScratch rs,
    const Fin& fin, const unsigned long long* wait_flags, int nwait, unsigned char* smem,
    uint64_t* bars, int* stage_ws, uint32_t& phase, int role = PDL_DEFAULT) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* stage = smem + static_cast<size_t>(warp) * stage_bytes;
    uint64_t* bar = bars + warp;
    int* stage_w = stage_ws + warp;
    const double* vb = reinterpret_cast<const double*>(stage);
    const uint16_t* cb = reinterpret_cast<const uint16_t*>(stage + val_bytes);
    double* xs = reinterpret_cast<double*>(stage + val_bytes + c16_bytes);
    const int64_t warp_g = static_cast<int64_t>(g.bid) * NW + warp;
    const int64_t nwarps = static_cast<int64_t>(g.nblk) * NW;
    // a tile of the tasks variant may start and end inside a slice: rows
    // outside the ranges are neither written nor dotted
    const RowRange none{0, 0};
    const SliceSpace sa(SPLIT ? ra : none, none, none);
    const SliceSpace sb(SPLIT ? rb0 : ra, SPLIT ? rb1 : rb0, SPLIT ? none : rb1);
    auto mine_of = [&](int64_t n) { return warp_g < n ? (n - warp_g + nwarps - 1) / nwarps : int64_t(0); };
    const int64_t mine_a = mine_of(sa.n), mine = mine_a + mine_of(sb.n);
    // one range (the single-domain CG, a tile): slice k of the warp directly
    const bool one = !SPLIT && rb0.r1 <= rb0.r0 && rb1.r1 <= rb1.r0;
    auto locate = [&](int64_t k, RowRange& rr) {
        if (one) {
            rr = ra;
            return (ra.r0 >> 5) + warp_g + k * nwarps;
        }
        const SliceSpace& sp = k < mine_a ? sa : sb;
        const int64_t i = warp_g + (k < mine_a ? k : k - mine_a) * nwarps;
        const int w = sp.which(i);
        rr = sp.q[w];
        return sp.slice(i, w);
    };
    const uint64_t pol = l2_evict_first_policy();
    const uint64_t xpol = KEEP ? l2_evict_last_policy() : 0;
    const uint64_t appol = TW_K1_AP_KEEP ? l2_evict_last_policy() : 0;
    constexpr uint32_t kRunBytes = kStageRunLen * 8;
    const unsigned long long want = nwait ? stamp_of(fin.sc, 0) : 0ull;
    // lane 0: the slice block (values + 16-bit columns) and then its 9 x runs,
    // all on one mbarrier transaction
    auto issue_block = [&](int64_t s) {
        const int64_t off = A.slice_off[s];
        const uint32_t ents = static_cast<uint32_t>(A.slice_off[s + 1] - off);
        TW_DCHECK(s >= 0 && s < A.n_slices && ents <= 32u * static_cast<uint32_t>(A.max_width));
        *stage_w = static_cast<int>(ents >> 5);
        mbar_expect_tx(bar, ents * 10u + kStageRuns * kRunBytes);
        if (ents) {
            bulk_g2s(stage, A.vals + off, ents * 8u, bar, pol);
            bulk_g2s(stage + val_bytes, A.cols16 + off, ents * 2u, bar, pol);
        }
    };
    auto issue_x = [&](int64_t k, int64_t s) { // default L2 policy: neighbouring slices share runs
        if (k == mine_a && nwait) {
            // first slice of space B: the neighbours' ghost planes must have
            // landed; then order the async-proxy (TMA) reads after the acquire
            thread_wait_flags(wait_flags, nwait, want);
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        int64_t starts[kStageRuns];
        run_starts(A, s, starts);
#pragma unroll
        for (int r = 0; r < kStageRuns; ++r) {
            const int64_t st = starts[r];
            // x carries 2 doubles of slack before index 0 and kStageRunLen after x_len
            TW_DCHECK(st >= -2 && st <= A.x_len);
            if (KEEP) // small x: keep its lines in L2 (evict_last) for the other runs
                bulk_g2s(xs + r * kStageRunLen, x + st, kRunBytes, bar, xpol);
            else
                bulk_g2s_plain(xs + r * kStageRunLen, x + st, kRunBytes, bar);
        }
    };
    // the matrix does not depend on the previous kernel: the first block
    // streams in before the wait for it; x (that kernel's p) only after
    RowRange rr;
    int64_t s = mine > 0 ? locate(0, rr) : 0;
    if (lane == 0 && mine > 0) issue_block(s);
    __syncwarp();
    if (PDL) {
        if (role == PDL_DEFAULT || role == PDL_GATE || role == PDL_GATE_LAST) pdl_wait();
        if (role == PDL_GATE) pdl_launch_dependents();
    }
    if (lane == 0 && mine > 0) issue_x(0, s);
    __syncwarp();
    double part_a = 0.0, part_b = 0.0;
    for (int64_t k = 0; k < mine; ++k) {
        mbar_wait(bar, phase & 1u);
        ++phase;
        const int w = *stage_w;
        double acc;
        switch (w) {
        case 27: acc = staged_row_fixed<27>(vb, cb, xs, lane); break;
        case 18: acc = staged_row_fixed<18>(vb, cb, xs, lane); break;
        case 12: acc = staged_row_fixed<12>(vb, cb, xs, lane); break;
        case 8: acc = staged_row_fixed<8>(vb, cb, xs, lane); break;
        default: acc = staged_row_generic(vb, cb, xs, lane, w); break;
        }
        const int64_t row = (s << 5) + lane;
        if (row >= rr.r0 && row < rr.r1) {
            if (TW_K1_AP_KEEP) st_evict_last(y + row, acc, appol);
            else y[row] = acc;
            const double d = __dmul_rn(xs[4 * kStageRunLen + 2 + lane], acc); // p[row] * (Ap)[row]
            if (SPLIT && k < mine_a) part_a = __dadd_rn(part_a, d);
            else part_b = __dadd_rn(part_b, d);
        }
        __syncwarp();
        if (k + 1 < mine) {
            s = locate(k + 1, rr);
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue_block(s);
                issue_x(k + 1, s);
            }
        }
        __syncwarp();
    }
    if (PDL) pdl_role_exit(role);
    if (SPLIT) grid_reduce2_finalize(part_a, part_b, rs, fin, g);
    else grid_reduce_finalize(part_b, rs, fin, g);
}

template <bool SPLIT, bool KEEP>
__global__ void __launch_bounds__(kTmaWarps * 32, 1)
spmv_tma_staged_kernel(EllView A, const double* __restrict__ x, double* __restrict__ y,
                       RowRange ra, RowRange rb0, RowRange rb1, int stage_bytes, int val_bytes,
                       int c16_bytes, RedScratch rs, Fin fin, const unsigned long long* wait_flags,
                       int nwait, int role) {
    TW_TL(1, ra.r1 > ra.r0 ? ra.r0 : rb0.r0);
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bars[kTmaWarps];
    __shared__ int stage_w[kTmaWarps];
    if (role == PDL_DEFAULT || role == PDL_INNER) pdl_launch_dependents();
    if ((threadIdx.x & 31) == 0) mbar_init(&bars[threadIdx.x >> 5], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t phase = 0;
    staged_spmv_body<SPLIT, kTmaWarps, true, KEEP>(launch_grid(), A, x, y, ra, rb0, rb1, stage_bytes,
                                             val_bytes, c16_bytes, rs, fin, wait_flags, nwait, smem,
                                             bars, stage_w, phase, role);
}

// --------------------------------------------------------- K2 / K3 / K4 streams

#ifndef TW_PAIRS_UNROLL
#define TW_PAIRS_UNROLL 1
#endif
constexpr int kPairsUnroll = TW_PAIRS_UNROLL;
// Pair-vectorised loop over [i0, i1): pairs (2j, 2j+1) fully inside use
// 128-bit accesses, the (at most two) ragged ends go scalar.
// Sweep direction of the vector passes (L2 reuse across kernel boundaries,
// 126 MB of L2 against 134 MB vectors at 256^3): K2 walks up and stores r
// with the default L2 policy (TW_K2_KEEP_R), K3 walks DOWN (TW_K3_REV), so
// it starts on the r lines K2 wrote last, still in L2, and ends on the low
// p lines the next K1 reads first.  Measured at 256^3: K3 112.6 -> 108.3 us,
// the iteration 865 -> 859.6 us; K2 walking down instead (reusing K1's Ap)
// gave 862 (profiles/r02_ab_k2k3_sweep.md).  K3 has no reduction, so its
// direction changes no bit; TW_K2_REV (a different fixed r.r tree) stays off.
#ifndef TW_K2_REV
#define TW_K2_REV 0
#endif
#ifndef TW_K2_KEEP_R
#define TW_K2_KEEP_R 1
#endif
#ifndef TW_K3_REV
#define TW_K3_REV 1
#endif
template <bool REV = false, typename F>
__device__ __forceinline__ void for_pairs(GridPos g, int64_t i0, int64_t i1, F&& f) {
    const int64_t j0 = i0 >> 1, j1 = (i1 + 1) >> 1;
    const int64_t stride = static_cast<int64_t>(g.nblk) * blockDim.x;
#pragma unroll kPairsUnroll
    for (int64_t t = j0 + static_cast<int64_t>(g.bid) * blockDim.x + threadIdx.x; t < j1;
         t += stride) {
        const int64_t j = REV ? j0 + j1 - 1 - t : t;
        const int64_t e = 2 * j;
        f(e, e >= i0, e + 1 < i1);
    }
}

// WX = false: K2 updates r only and the x update (x += alpha p_old) moves
// into K3, which reads p_old anyway -- 8 n bytes less per iteration, same
// roundings (x feeds nothing inside the iteration); with alpha from rank
// partials block 0 leaves it in sc->alpha for K3.
template <bool WX>
__device__ __forceinline__ void update_xr_rows(GridPos g, int64_t i0, int64_t i1,
                                               double* __restrict__ x, const double* __restrict__ p,
                                               double* __restrict__ r, const double* __restrict__ Ap,
                                               CgScalars* sc, ScalarSrc asrc, RedScratch rs,
                                               const Fin& fin, int role = PDL_DEFAULT) {
    pdl_role_entry(role); // Ap and alpha come from K1
    double alpha;
    if (asrc.flags) block_wait_flags(asrc.flags, asrc.count, stamp_of(sc, 0));
    if (asrc.count > 0)
        alpha = __ddiv_rn(sc->rtrans, sum_parts(asrc.parts, asrc.count));
    else
        alpha = sc ? sc->alpha : __ldcg(asrc.parts); // standalone op: alpha from a device scalar
    const double nalpha = -alpha; // waxpby(1, r, -alpha, Ap, r) (cg.cpp:383)
    if (!WX && asrc.count > 0 && g.bid == 0 && threadIdx.x == 0) {
        sc->alpha_prev = sc->alpha; // the previous iteration's (paired x updates in K3)
        sc->alpha = alpha;
    }
    double part = 0.0;
    for_pairs<TW_K2_REV != 0>(g, i0, i1, [&](int64_t e, bool lo, bool hi) {
        if (!WX) {
            if (lo && hi) {
                double2 rv = __ldcs(reinterpret_cast<const double2*>(r + e));
                const double2 av = __ldcs(reinterpret_cast<const double2*>(Ap + e));
                rv.x = __dadd_rn(rv.x, __dmul_rn(nalpha, av.x));
                rv.y = __dadd_rn(rv.y, __dmul_rn(nalpha, av.y));
                if (TW_K2_KEEP_R == 2) st2_evict_last(r + e, rv, l2_evict_last_policy());
                else if (TW_K2_KEEP_R) *reinterpret_cast<double2*>(r + e) = rv;
                else __stcs(reinterpret_cast<double2*>(r + e), rv);
                part = __dadd_rn(part, __dmul_rn(rv.x, rv.x));
                part = __dadd_rn(part, __dmul_rn(rv.y, rv.y));
            } else {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (!(h == 0 ? lo : hi)) continue;
                    const int64_t i = e + h;
                    const double rv = __dadd_rn(r[i], __dmul_rn(nalpha, Ap[i]));
                    r[i] = rv;
                    part = __dadd_rn(part, __dmul_rn(rv, rv));
                }
            }
        } else if (lo && hi) {
            double2 xv = __ldcs(reinterpret_cast<const double2*>(x + e));
            double2 pv = __ldcs(reinterpret_cast<const double2*>(p + e));
            double2 rv = __ldcs(reinterpret_cast<const double2*>(r + e));
            double2 av = __ldcs(reinterpret_cast<const double2*>(Ap + e));
            xv.x = __dadd_rn(xv.x, __dmul_rn(alpha, pv.x));
            xv.y = __dadd_rn(xv.y, __dmul_rn(alpha, pv.y));
            rv.x = __dadd_rn(rv.x, __dmul_rn(nalpha, av.x));
            rv.y = __dadd_rn(rv.y, __dmul_rn(nalpha, av.y));
            __stcs(reinterpret_cast<double2*>(x + e), xv);
            __stcs(reinterpret_cast<double2*>(r + e), rv);
            part = __dadd_rn(part, __dmul_rn(rv.x, rv.x));
            part = __dadd_rn(part, __dmul_rn(rv.y, rv.y));
        } else {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (!(h == 0 ? lo : hi)) continue;
                const int64_t i = e + h;
                x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
                double rv = __dadd_rn(r[i], __dmul_rn(nalpha, Ap[i]));
                r[i] = rv;
                part = __dadd_rn(part, __dmul_rn(rv, rv));
            }
        }
    });
    pdl_role_exit(role);
    grid_reduce_finalize(part, rs, fin, g);
}

template <bool WX>
__global__ void __launch_bounds__(kThreads)
update_xr_kernel(int64_t i0, int64_t i1, double* __restrict__ x, const double* __restrict__ p,
                 double* __restrict__ r, const double* __restrict__ Ap, CgScalars* sc,
                 ScalarSrc asrc, RedScratch rs, Fin fin, int role) {
    TW_TL(2, i0);
    update_xr_rows<WX>(launch_grid(), i0, i1, x, p, r, Ap, sc, asrc, rs, fin, role);
}

// K3's streaming loop over [a0, b0): p = r + beta psrc, two pairs per
// thread and step.  U: compiler unroll of that loop on top (measured: 4 for
// the lean kernel, 2 in the peer instantiation, where 3+ costs registers).
#ifndef TW_K3PX_UNROLL
#define TW_K3PX_UNROLL 4 // the peer K3 with the x update (124 registers; 2.3 % faster than 2)
#endif
#ifndef TW_K3X_UNROLL
#define TW_K3X_UNROLL 4 // lean K3 with the x update (126 registers; 1.5 % faster than 2)
#endif
// The K3s of an x-update pair run best at the highest occupancy (no extra
// unroll; 60 / 72 registers): 256^3, K3 averaged over the pair 118.0 us
// with unroll 4 / 2, 98.3 with 1 / 1 (profiles/r02_ab_k2k3_sweep.md)
#ifndef TW_K3_UNROLL
#define TW_K3_UNROLL 1 // lean K3 without the x update
#endif
#ifndef TW_K3XX_UNROLL
#define TW_K3XX_UNROLL 1 // K3 with the paired x update
#endif
#ifndef TW_K3PXX_UNROLL
#define TW_K3PXX_UNROLL 1 // the peer K3 with the paired x update
#endif
// XU: the x update riding on K3's read of p_old --
//   0: none;
//   1: x += alpha p_old (the x update moved out of K2);
//   2: the second iteration of a pair: x = (x + alpha0 p0) + alpha p_old,
//      p0 / alpha0 = the previous iteration's p and alpha, whose update the
//      first iteration of the pair deferred (the same two roundings in the
//      same order as two single updates; x is read and written once per pair).
template <int U, int XU>
__device__ __forceinline__ void p_stream(int64_t a0, int64_t b0, int64_t tid, int64_t stride,
                                         const double* __restrict__ r,
                                         const double* __restrict__ psrc, double* __restrict__ p,
                                         double beta, double* __restrict__ x, double alpha,
                                         const double* p0 = nullptr, // may alias p (pair: p_k+2 over p_k)
                                         double alpha0 = 0.0) {
    constexpr bool WX = XU != 0;
    const int64_t a = (a0 + 1) & ~int64_t(1), b = b0 & ~int64_t(1);
    const uint64_t ppol = TW_K3_P_KEEP ? l2_evict_last_policy() : 0;
    auto pair = [&](int64_t e, double2 rv, double2 pv, double2 xv, double2 ov) {
        if (XU == 2) {
            xv.x = __dadd_rn(xv.x, __dmul_rn(alpha0, ov.x));
            xv.y = __dadd_rn(xv.y, __dmul_rn(alpha0, ov.y));
        }
        if (WX) {
            xv.x = __dadd_rn(xv.x, __dmul_rn(alpha, pv.x));
            xv.y = __dadd_rn(xv.y, __dmul_rn(alpha, pv.y));
            __stcs(reinterpret_cast<double2*>(x + e), xv);
        }
        pv.x = __dadd_rn(rv.x, __dmul_rn(beta, pv.x));
        pv.y = __dadd_rn(rv.y, __dmul_rn(beta, pv.y));
        if (TW_K3_P_KEEP) st2_evict_last(p + e, pv, ppol);
        else *reinterpret_cast<double2*>(p + e) = pv;
    };
    const int64_t J0 = a >> 1, J1 = b >> 1;
#pragma unroll U
    for (int64_t j = J0 + tid; j < J1; j += 2 * stride) {
        const bool two = j + stride < J1;
        const int64_t e0 = 2 * (TW_K3_REV ? J0 + J1 - 1 - j : j);
        const int64_t e1 = 2 * (TW_K3_REV ? J0 + J1 - 1 - (j + stride) : j + stride);
        const double2 r0 = __ldcs(reinterpret_cast<const double2*>(r + e0));
        const double2 q0 = __ldcs(reinterpret_cast<const double2*>(psrc + e0));
        double2 r1 = make_double2(0.0, 0.0), q1 = r1, x0 = r1, x1 = r1, o0 = r1, o1 = r1;
        if (WX) x0 = __ldcs(reinterpret_cast<const double2*>(x + e0));
        if (XU == 2) o0 = __ldcs(reinterpret_cast<const double2*>(p0 + e0));
        if (two) {
            r1 = __ldcs(reinterpret_cast<const double2*>(r + e1));
            q1 = __ldcs(reinterpret_cast<const double2*>(psrc + e1));
            if (WX) x1 = __ldcs(reinterpret_cast<const double2*>(x + e1));
            if (XU == 2) o1 = __ldcs(reinterpret_cast<const double2*>(p0 + e1));
        }
        pair(e0, r0, q0, x0, o0);
        if (two) pair(e1, r1, q1, x1, o1);
    }
    if (tid == 0) {
        auto one = [&](int64_t i) {
            if (XU == 2) x[i] = __dadd_rn(x[i], __dmul_rn(alpha0, p0[i]));
            if (WX) x[i] = __dadd_rn(x[i], __dmul_rn(alpha, psrc[i]));
            p[i] = __dadd_rn(r[i], __dmul_rn(beta, psrc[i]));
        };
        if ((a0 & 1) && a0 < b0) one(a0);
        if (b < b0 && b >= a0 && b >= a) one(b);
    }
}

// PEER: the peer-transport instantiation (flag wait, fused halo stores);
// the plain one stays lean so the grid keeps its full occupancy.
// XU: the x update riding on this K3 (p_stream): 0 none, 1 x += alpha p_old,
// 2 the second K3 of an x-update pair (p0 = the previous iteration's p,
// alpha0 = its alpha, kept in sc->alpha_prev by K1's alpha finalisation).
template <bool PEER, int XU>
__device__ __forceinline__ void update_p_rows(GridPos g, int64_t i0, int64_t i1,
                                              const double* __restrict__ r, double* __restrict__ p,
                                              CgScalars* sc, ScalarSrc bsrc, RedScratch rs,
                                              double* history, const PeerLinks* links_,
                                              const double* __restrict__ psrc,
                                              double* __restrict__ x, const double* p0,
                                              int role = PDL_DEFAULT) {
    // psrc: p_old, == p in place (each element is read, then written, by the
    // same thread, so the restrict-qualified aliasing is never observable);
    // p0 may alias p the same way (the pair writes p_k+2 over p_k)
    constexpr bool WX = XU != 0;
    const PeerLinks* links = PEER ? links_ : nullptr;
    pdl_role_entry(role); // r and beta come from K2
    double beta, rr = 0.0;
    const double alpha = WX ? sc->alpha : 0.0; // this iteration's (K1 / K2 left it there)
    const double alpha0 = XU == 2 ? sc->alpha_prev : 0.0;
    unsigned long long next = 0; // flag stamp of the next iteration (peer ghost flags)
    if (PEER && bsrc.flags) block_wait_flags(bsrc.flags, bsrc.count, stamp_of(sc, 0));
    if (bsrc.count > 0) {
        // beta from the rank partials; then the iteration's commit (beta_res,
        // cg.cpp:290-311) by the LAST block to have read the scalars: every
        // block takes an acq_rel ticket right after its reads, so the commit
        // needs no end-of-kernel ticket (which would wait for the p stores)
        rr = sum_parts(bsrc.parts, bsrc.count);
        const int it = sc->iter;
        beta = __ddiv_rn(rr, sc->rtrans);
        next = (static_cast<unsigned long long>(sc->epoch) << 32) |
               static_cast<unsigned long long>(it + 2);
        __syncthreads(); // the whole block has read sc
        if (threadIdx.x == 0) {
            const unsigned t = atom_inc_acq_rel(rs.ticket, static_cast<unsigned>(g.nblk - 1));
            if (t == static_cast<unsigned>(g.nblk - 1)) {
                sc->rr = rr;
                sc->beta = beta;
                sc->rtrans = rr;
                if (it < sc->history_cap) history[it] = __dsqrt_rn(rr);
                sc->iter = it + 1;
            }
        }
    } else {
        beta = sc ? sc->beta : __ldcg(bsrc.parts); // standalone op: beta from a device scalar
    }
    const int64_t tid = static_cast<int64_t>(g.bid) * blockDim.x + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(g.nblk) * blockDim.x;
    // Full pairs of [a0, b0) with 128-bit accesses, two pairs per thread and
    // step (both pairs' loads issued before either store: twice the bytes in
    // flight of a one-pair loop); the at most two ragged ends go scalar.
    constexpr int U = XU == 2 ? (PEER ? TW_K3PXX_UNROLL : TW_K3XX_UNROLL)
                              : PEER ? (WX ? TW_K3PX_UNROLL : 2) : (WX ? TW_K3X_UNROLL : TW_K3_UNROLL);
    auto stream = [&](int64_t a0, int64_t b0) {
        p_stream<U, XU>(a0, b0, tid, stride, r, psrc, p, beta, x, alpha, p0, alpha0);
    };
    if (!links) {
        stream(i0, i1);
        pdl_role_exit(role);
        return;
    }
    // Fused halo (peer transport): the first / last owned plane of p also
    // goes straight into the neighbours' ghost planes over NVLink.  The bulk
    // streams through the lean loop; the two edge planes are a scalar pass
    // of the first kEdgeBlocks blocks only, which alone fence at system
    // scope and take a ticket -- the last of them raises the neighbours'
    // ghost flags for the next iteration.
    constexpr int kEdgeBlocks = 64;
    const int64_t plane = links->plane;
    double* lo_dst = links->ghost_lo_dst;
    double* hi_dst = links->ghost_hi_dst;
    // an edge plane without a neighbour streams with the bulk
    const int64_t lo_end = lo_dst ? (i0 + plane < i1 ? i0 + plane : i1) : i0;
    const int64_t hi_beg = hi_dst ? (i1 - plane > lo_end ? i1 - plane : lo_end) : i1;
    // the edge planes FIRST, so their system-scope fence waits only for the
    // edge stores (after the bulk it waited for the block's share of the
    // bulk too: 20 us of a 100 us K3 on a 1-rank communicator), and the
    // neighbours' flags rise a whole K3 earlier
    const int ne = g.nblk < kEdgeBlocks ? g.nblk : kEdgeBlocks;
    const int64_t nlo = lo_end - i0, nedge = nlo + (i1 - hi_beg);
    if (g.bid < ne && nedge > 0) {
        const int64_t etid = static_cast<int64_t>(g.bid) * blockDim.x + threadIdx.x;
        const int64_t estride = static_cast<int64_t>(ne) * blockDim.x;
#pragma unroll 1
        for (int64_t k = etid; k < nedge; k += estride) {
            const int64_t i = k < nlo ? i0 + k : hi_beg + (k - nlo);
            TW_DCHECK(i >= i0 && i < i1);
            if (XU == 2) x[i] = __dadd_rn(x[i], __dmul_rn(alpha0, p0[i]));
            if (WX) x[i] = __dadd_rn(x[i], __dmul_rn(alpha, psrc[i]));
            const double v = __dadd_rn(r[i], __dmul_rn(beta, psrc[i]));
            p[i] = v;
            if (lo_dst && i - i0 < plane) lo_dst[i - i0] = v;
            if (hi_dst && i >= i1 - plane) hi_dst[i - (i1 - plane)] = v;
        }
        __syncthreads(); // the block's ghost stores are issued
        if (threadIdx.x == 0) {
            __threadfence_system(); // ... and have landed in the neighbours' memory
            const unsigned t = atomicInc(rs.ticket + 1, static_cast<unsigned>(ne - 1));
            if (t == static_cast<unsigned>(ne - 1)) {
                __threadfence_system();
                if (links->ghost_lo_flag) st_release_sys(links->ghost_lo_flag, next);
                if (links->ghost_hi_flag) st_release_sys(links->ghost_hi_flag, next);
            }
        }
    }
    stream(lo_end, hi_beg);
    pdl_role_exit(role);
}

template <bool PEER, int XU>
__global__ void __launch_bounds__(kThreads)
update_p_kernel(int64_t i0, int64_t i1, const double* __restrict__ r, double* __restrict__ p,
                CgScalars* sc, ScalarSrc bsrc, RedScratch rs, double* history,
                const PeerLinks* links, const double* __restrict__ psrc, double* __restrict__ x,
                const double* p0, int role) {
    TW_TL(3, i0);
    update_p_rows<PEER, XU>(launch_grid(), i0, i1, r, p, sc, bsrc, rs, history, links, psrc, x, p0,
                            role);
}

// ------------------------------------------- concurrent rank group (1 GPU)

// Barrier of one rank's blocks inside the rank-group kernel: stands in for
// the kernel boundaries between that rank's launches.  Generation counting;
// the gpu-scope acquire + fence also drops stale L1 lines before the next
// phase gathers p.
__device__ __forceinline__ void group_barrier(unsigned* bar, int nblk) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned gen = ld_acquire_gpu(bar + 1);
        __threadfence();
        if (atomicAdd(bar, 1u) == static_cast<unsigned>(nblk - 1)) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            const unsigned long long t0 = global_ns();
            while (ld_acquire_gpu(bar + 1) == gen) {
                __nanosleep(32);
                if (global_ns() - t0 > TW_PEER_TIMEOUT_NS) {
                    printf("tw_hpccg: rank-group barrier timed out\n");
                    __trap();
                }
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// P ranks of the peer transport as ONE cooperative kernel: blocks
// [r B, (r+1) B) run rank r's iterations -- the same phase bodies, flag
// waits, publishes and fused halo stores as the per-rank launches, with a
// group barrier where those have a kernel boundary.  The ranks run truly
// concurrently and wait on one another's flags, which separate launches on
// one GPU must never do; co-residency of the whole grid (cooperative
// launch) makes the waits safe.  `jitter` delays rank-dependent blocks to
// vary the interleavings.
//
// On an x-staged slab K1 is the staged one-launch form (interior slices,
// then per warp: acquire of the ghost flags, proxy fence, TMA of the ghost
// runs) with kThreads / 32 warps per block and their stages in dynamic
// shared memory -- the pattern of the peer path's spmv_tma_staged_kernel<true>
// under real concurrency.
__global__ void __launch_bounds__(kThreads)
rank_group_kernel(const GroupRank* ranks, int B, int iterations, int jitter) {
    static_assert(kThreads == kGroupThreads, "host sizes the group's stages by kGroupThreads");
    constexpr int kW = kThreads / 32;
    extern __shared__ __align__(128) unsigned char gsmem[];
    __shared__ uint64_t gbars[kW];
    __shared__ int gstage_w[kW];
    const int rk = blockIdx.x / B;
    const GridPos g{static_cast<int>(blockIdx.x % B), B};
    const GroupRank& R = ranks[rk];
    const RowRange all{0, 0};
    const bool staged = R.A.cols16 != nullptr;
    if (staged && (threadIdx.x & 31) == 0) mbar_init(&gbars[threadIdx.x >> 5], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    uint32_t phase = 0;
    for (int it = 0; it < iterations; ++it) {
        if (jitter && threadIdx.x == 0 && g.bid == (it * 7 + rk * 3) % B)
            __nanosleep(static_cast<unsigned>(((it + 1) * (rk + 1) * 977) % 20000));
        if (staged) {
            staged_spmv_body<true, kW, false>(
                g, R.A, R.p_local, R.Ap, RowRange{R.int_r0, R.int_r1}, RowRange{0, R.int_r0},
                RowRange{R.int_r1, R.n}, R.stage_bytes, R.val_bytes, R.c16_bytes, R.rs,
                Fin{FIN_PUBLISH_A, R.pm + 1, R.sc, nullptr, R.links, R.pm}, R.ghost_flags,
                R.n_ghost, gsmem, gbars, gstage_w, phase);
            group_barrier(R.bar, B);
        } else {
            // K1 interior rows (no ghost plane), partial into pm[0]
            spmv_rows<true, kGatherCA>(g, R.A, R.p_local, R.Ap, RowRange{R.int_r0, R.int_r1}, all,
                                       R.rs, Fin{FIN_STORE, R.pm, nullptr, nullptr, nullptr, nullptr},
                                       nullptr, 0);
            group_barrier(R.bar, B);
            // K1 boundary rows after the ghost flags; publish (0 + pm[0]) + pm[1]
            spmv_rows<true, kGatherCG>(g, R.A, R.p_local, R.Ap, RowRange{0, R.int_r0},
                                       RowRange{R.int_r1, R.n}, R.rs,
                                       Fin{FIN_PUBLISH_A, R.pm + 1, R.sc, nullptr, R.links, R.pm},
                                       R.ghost_flags, R.n_ghost);
            group_barrier(R.bar, B);
        }
#ifdef TW_BREAK_PEER_WAIT // negative control of the concurrency test only
        update_xr_rows<false>(g, 0, R.n, R.x, R.p_owned, R.r, R.Ap, R.sc,
                              ScalarSrc{R.win->recv_a, R.P, nullptr}, R.rs,
#else
        update_xr_rows<false>(g, 0, R.n, R.x, R.p_owned, R.r, R.Ap, R.sc,
                              ScalarSrc{R.win->recv_a, R.P, R.win->flag_a}, R.rs,
#endif
                       Fin{FIN_PUBLISH_B, R.send_b, R.sc, nullptr, R.links, nullptr});
        group_barrier(R.bar, B);
        update_p_rows<true, 1>(g, 0, R.n, R.r, R.p_owned, R.sc,
                                  ScalarSrc{R.win->recv_b, R.P, R.win->flag_b}, R.rs, R.history,
                                  R.links, R.p_owned, R.x, nullptr);
        group_barrier(R.bar, B);
    }
}

__global__ void __launch_bounds__(kThreads)
dot_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t i0, int64_t i1,
           RedScratch rs, Fin fin) {
    double part = 0.0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = i0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < i1;
         i += stride)
        part = __dadd_rn(part, __dmul_rn(__ldg(a + i), __ldg(b + i)));
    grid_reduce_finalize(part, rs, fin);
}

__global__ void __launch_bounds__(kThreads)
waxpby_kernel(double alpha, const double* x, double beta, const double* y, double* w, int64_t i0,
              int64_t i1) {
    // x, y, w may alias (kernels.cpp:22-26): each element is read before it
    // is written by the same thread, so aliasing is safe.
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = i0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < i1;
         i += stride)
        w[i] = __dadd_rn(__dmul_rn(alpha, x[i]), __dmul_rn(beta, y[i]));
}

__global__ void combine_kernel(const double* parts, int count, Fin fin) {
    TW_TL(4, 0);
    if (threadIdx.x == 0) finalize(fin, sum_parts(parts, count));
}

__global__ void fill_kernel(double* p, int64_t n, double v) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += stride)
        p[i] = v;
}

// SplitMix64 (scenario.cpp:46-55) is counter based: element i uses state
// seed + (i+1)*gamma.
__global__ void rhs_splitmix_kernel(uint64_t seed, int64_t first, int64_t count, double* out) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += stride) {
        uint64_t z = seed + static_cast<uint64_t>(first + i + 1) * 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z ^= z >> 31;
        out[i] = __dmul_rn(static_cast<double>(z >> 11), 0x1.0p-53);
    }
}

// xorshift64 (acceptance.cpp:48-58) is sequential; the host jumps the state
// to every chunk start (GF(2) matrix powers) and each thread walks a chunk.
__global__ void rhs_xorshift_kernel(const uint64_t* states, int64_t chunk, int64_t count,
                                    int64_t skip, double* out) {
    const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t begin = c * chunk - skip; // output index of this chunk's first value
    if (begin >= count) return;
    uint64_t s = states[c];
    for (int64_t j = 0; j < chunk; ++j) {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        const int64_t i = begin + j;
        if (i >= count) break;
        if (i >= 0) out[i] = 0.5 + static_cast<double>(s % 1000u) / 1000.0;
    }
}

} // namespace

// ------------------------------------------------------------------ launchers

LaunchCfg query_launch_cfg(int sm_count) {
    int occ_spmv = 0, occ_stream = 0;
    TW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_spmv, spmv_kernel<true>, kThreads, 0));
    TW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_stream, update_xr_kernel<true>, kThreads, 0));
    LaunchCfg c;
    c.spmv_blocks = sm_count * (occ_spmv > 0 ? occ_spmv : 1);
    c.stream_blocks = sm_count * (occ_stream > 0 ? occ_stream : 1);
    c.threads = kThreads;
    c.tma_blocks = sm_count;
    return c;
}

static int tma_stage_bytes(int max_width, int* val_bytes) {
    const int vb = ((32 * max_width * 8) + 127) / 128 * 128;
    const int cb = ((32 * max_width * 4) + 127) / 128 * 128;
    *val_bytes = vb;
    return vb + cb;
}

int spmv_tma_warps() { return kTmaWarps; }

// Launch with programmatic dependent launch allowed (pdl): the kernel may
// start while its stream predecessor drains; its griddepcontrol.wait holds
// the dependent reads until that predecessor has completed and flushed.
template <typename... KArgs, typename... Args>
static void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t s, bool pdl, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = pdl ? attr : nullptr;
    cfg.numAttrs = pdl ? 1 : 0;
    TW_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

int spmv_tma_smem_bytes(int max_width) {
    int vb;
    return kTmaWarps * kTmaStages * tma_stage_bytes(max_width, &vb);
}

// The TMA-staged SpMV needs one slice block of the widest slice per warp in
// shared memory; returns false when that does not fit (then the register
// path runs).  The opt-in shared-memory size is a per-device attribute.
template <bool DOT>
static bool launch_spmv_tma(const EllView& A, const double* x, double* y, RowRange a, RowRange b,
                            RedScratch rs, Fin fin, cudaStream_t s, const unsigned long long* wait_flags,
                            int nwait, bool pdl = false) {
    if (A.max_width <= 0 || A.tma_blocks <= 0) return false;
    auto slices = [](RowRange q) { return q.r1 > q.r0 ? ((q.r1 + 31) >> 5) - (q.r0 >> 5) : 0; };
    const int64_t ns = slices(a) + slices(b);
    int vb;
    const int stage = tma_stage_bytes(A.max_width, &vb);
    const int smem = kTmaWarps * kTmaStages * stage;
    auto kern = spmv_tma_kernel<DOT>;
    constexpr int kMaxDev = 64;
    static std::mutex mu;
    static int attr_bytes[kMaxDev] = {};
    static int static_bytes = -1;
    int dev = 0;
    TW_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (static_bytes < 0) {
        cudaFuncAttributes fa;
        TW_CUDA(cudaFuncGetAttributes(&fa, kern));
        static_bytes = static_cast<int>(fa.sharedSizeBytes);
    }
    if (dev >= kMaxDev || smem + static_bytes > 227 * 1024) return false;
    if (attr_bytes[dev] < smem) {
        TW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr_bytes[dev] = smem;
    }
    const int64_t need = (ns + kTmaWarps - 1) / kTmaWarps;
    const int g = static_cast<int>(need < A.tma_blocks ? (need < 1 ? 1 : need) : A.tma_blocks);
    launch_k(kern, dim3(g), dim3(kTmaWarps * 32), smem, s, pdl, A, x, y, a, b, stage, vb, rs, fin,
             wait_flags, nwait);
    TW_CUDA(cudaGetLastError());
    return true;
}

void launch_spmv(const EllView& A, const double* x, double* y, RowRange a, RowRange b,
                 bool with_dot, RedScratch rs, Fin fin, int blocks, cudaStream_t s,
                 const unsigned long long* wait_flags, int nwait, bool pdl) {
    if (with_dot ? launch_spmv_tma<true>(A, x, y, a, b, rs, fin, s, wait_flags, nwait, pdl)
                 : launch_spmv_tma<false>(A, x, y, a, b, rs, fin, s, wait_flags, nwait, pdl))
        return;
    auto slices = [](RowRange q) { return q.r1 > q.r0 ? ((q.r1 + 31) >> 5) - (q.r0 >> 5) : 0; };
    const int g = clamp_blocks((slices(a) + slices(b)) * 32, blocks);
    if (with_dot)
        spmv_kernel<true><<<g, kThreads, 0, s>>>(A, x, y, a, b, rs, fin, wait_flags, nwait);
    else
        spmv_kernel<false><<<g, kThreads, 0, s>>>(A, x, y, a, b, rs, fin, wait_flags, nwait);
    TW_CUDA(cudaGetLastError());
}

int rank_group_blocks_per_rank(int nranks, int smem) {
    int occ = 0, dev = 0, sms = 0;
    TW_CUDA(cudaFuncSetAttribute(rank_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem));
    TW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rank_group_kernel, kThreads, smem));
    TW_CUDA(cudaGetDevice(&dev));
    TW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    return occ * sms / nranks;
}

void launch_rank_group(const GroupRank* ranks_dev, int nranks, int blocks_per_rank,
                       int iterations, int jitter, int smem, cudaStream_t s) {
    int B = blocks_per_rank, it = iterations;
    void* args[] = {&ranks_dev, &B, &it, &jitter};
    TW_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(rank_group_kernel),
                                        dim3(static_cast<unsigned>(nranks * B)), dim3(kThreads),
                                        args, static_cast<size_t>(smem), s));
}

bool launch_spmv_split(const EllView& A, const double* x, double* y, RowRange interior,
                       RowRange b0, RowRange b1, RedScratch rs, Fin fin, cudaStream_t s,
                       const unsigned long long* wait_flags, int nwait, bool pdl) {
    if (A.max_width <= 0 || A.tma_blocks <= 0) return false;
    int vb;
    const int stage = tma_stage_bytes(A.max_width, &vb);
    const int smem = kTmaWarps * stage;
    static std::mutex mu;
    static int attr_bytes[64] = {};
    static int static_bytes = -1;
    int dev = 0;
    TW_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(mu);
        if (static_bytes < 0) {
            cudaFuncAttributes fa;
            TW_CUDA(cudaFuncGetAttributes(&fa, spmv_tma_split_kernel));
            static_bytes = static_cast<int>(fa.sharedSizeBytes);
        }
        if (dev >= 64 || smem + static_bytes > 227 * 1024) return false;
        if (attr_bytes[dev] < smem) {
            TW_CUDA(cudaFuncSetAttribute(spmv_tma_split_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            attr_bytes[dev] = smem;
        }
    }
    // the grid the separate interior / boundary launches would use: both are
    // the full persistent grid whenever each range has >= one slice per warp
    // of it; smaller ranges would map differently, so they fall back
    auto slices = [](RowRange q) { return q.r1 > q.r0 ? ((q.r1 + 31) >> 5) - (q.r0 >> 5) : 0; };
    const int64_t full = static_cast<int64_t>(A.tma_blocks) * kTmaWarps;
    if (slices(interior) < full || slices(b0) + slices(b1) < full) return false;
    launch_k(spmv_tma_split_kernel, dim3(A.tma_blocks), dim3(kTmaWarps * 32), smem, s, pdl, A, x, y,
             interior, b0, b1, stage, vb, rs, fin, wait_flags, nwait);
    TW_CUDA(cudaGetLastError());
    return true;
}

int staged_stage_bytes(int max_width, int* val_bytes, int* c16_bytes) {
    *val_bytes = ((32 * max_width * 8) + 127) / 128 * 128;
    *c16_bytes = ((32 * max_width * 2) + 127) / 128 * 128;
    return *val_bytes + *c16_bytes + (kStageRuns * kStageRunLen * 8 + 127) / 128 * 128;
}

template <bool SPLIT, bool KEEP>
static bool staged_attr(int smem) {
    static std::mutex mu;
    static int attr_bytes[64] = {};
    static int static_bytes = -1;
    int dev = 0;
    TW_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (static_bytes < 0) {
        cudaFuncAttributes fa;
        TW_CUDA(cudaFuncGetAttributes(&fa, spmv_tma_staged_kernel<SPLIT, KEEP>));
        static_bytes = static_cast<int>(fa.sharedSizeBytes);
    }
    if (dev >= 64 || smem + static_bytes > 227 * 1024) return false;
    if (attr_bytes[dev] < smem) {
        TW_CUDA(cudaFuncSetAttribute(spmv_tma_staged_kernel<SPLIT, KEEP>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr_bytes[dev] = smem;
    }
    return true;
}

bool launch_spmv_staged(const EllView& A, const double* x, double* y, RowRange ra, RowRange rb0,
                        RowRange rb1, bool split, RedScratch rs, Fin fin, cudaStream_t s,
                        const unsigned long long* wait_flags, int nwait, bool pdl, int role) {
    if (!A.cols16 || A.max_width <= 0 || A.tma_blocks <= 0) return false;
    int vb, cb;
    const int stage = staged_stage_bytes(A.max_width, &vb, &cb);
    const int smem = kTmaWarps * stage;
    const bool keep = A.sx_keep != 0;
    const bool attr_ok = split ? (keep ? staged_attr<true, true>(smem) : staged_attr<true, false>(smem))
                               : (keep ? staged_attr<false, true>(smem) : staged_attr<false, false>(smem));
    if (!attr_ok) return false;
    auto slices = [](RowRange q) { return q.r1 > q.r0 ? ((q.r1 + 31) >> 5) - (q.r0 >> 5) : 0; };
    const int64_t full = static_cast<int64_t>(A.tma_blocks) * kTmaWarps;
    int g;
    if (split) {
        // the grid the separate launches would use: the full persistent grid
        // whenever each space has >= one slice per warp of it (else fall back)
        if (slices(ra) < full || slices(rb0) + slices(rb1) < full) return false;
        g = A.tma_blocks;
    } else {
        const int64_t ns = slices(ra) + slices(rb0) + slices(rb1);
        const int64_t need = (ns + kTmaWarps - 1) / kTmaWarps;
        g = static_cast<int>(need < A.tma_blocks ? (need < 1 ? 1 : need) : A.tma_blocks);
    }
    using K = decltype(&spmv_tma_staged_kernel<false, false>);
    const K kern = split ? (keep ? spmv_tma_staged_kernel<true, true> : spmv_tma_staged_kernel<true, false>)
                         : (keep ? spmv_tma_staged_kernel<false, true>
                                 : spmv_tma_staged_kernel<false, false>);
    launch_k(kern, dim3(g), dim3(kTmaWarps * 32), smem, s, pdl, A, x, y, ra, rb0, rb1, stage, vb, cb,
             rs, fin, wait_flags, nwait, role);
    return true;
}

int spmv_staged_smem_bytes(int max_width) {
    int vb, cb;
    return kTmaWarps * staged_stage_bytes(max_width, &vb, &cb);
}

void launch_update_xr(int64_t i0, int64_t i1, double* x, const double* p, double* r,
                      const double* Ap, CgScalars* sc, ScalarSrc asrc, RedScratch rs, Fin fin,
                      int blocks, cudaStream_t s, bool pdl, int role) {
    const int g = clamp_blocks((i1 - i0 + 1) / 2 + 1, blocks);
    if (x)
        launch_k(update_xr_kernel<true>, dim3(g), dim3(kThreads), 0, s, pdl, i0, i1, x, p, r, Ap, sc,
                 asrc, rs, fin, role);
    else
        launch_k(update_xr_kernel<false>, dim3(g), dim3(kThreads), 0, s, pdl, i0, i1, x, p, r, Ap,
                 sc, asrc, rs, fin, role);
    TW_CUDA(cudaGetLastError());
}

void launch_update_p(int64_t i0, int64_t i1, const double* r, double* p, CgScalars* sc,
                     ScalarSrc bsrc, RedScratch rs, double* history, int blocks,
                     cudaStream_t s, const PeerLinks* links, const double* psrc, bool pdl,
                     double* x, const double* p0, int role) {
    // grid: at most one resident wave of this instantiation (a partial
    // second wave of a grid-stride loop would double the tail)
    const bool peer = links != nullptr || bsrc.flags != nullptr;
    const int xu = x ? (p0 ? 2 : 1) : 0;
    if (p0 && !x) throw Error(TW_ERR_CONTRACT, "the pair's p0 comes with its x update");
    const int which = (peer ? 3 : 0) + xu;
    using K = decltype(&update_p_kernel<false, 0>);
    static const K kerns[6] = {update_p_kernel<false, 0>, update_p_kernel<false, 1>,
                               update_p_kernel<false, 2>, update_p_kernel<true, 0>,
                               update_p_kernel<true, 1>, update_p_kernel<true, 2>};
    // resident blocks per SM of each instantiation (thread-safe one-time init;
    // the grid multiplies by this device's SM count)
    auto occupancy = [](K k) {
        int o = 0;
        TW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, reinterpret_cast<const void*>(k),
                                                              kThreads, 0));
        return o > 0 ? o : 1;
    };
    static const int occ[6] = {occupancy(kerns[0]), occupancy(kerns[1]), occupancy(kerns[2]),
                               occupancy(kerns[3]), occupancy(kerns[4]), occupancy(kerns[5])};
    int dev = 0, sms = 0;
    TW_CUDA(cudaGetDevice(&dev));
    TW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int wave = occ[which] * sms;
    const int g = clamp_blocks((i1 - i0 + 1) / 2 + 1, blocks < wave ? blocks : wave);
    if (x && !sc) throw Error(TW_ERR_CONTRACT, "the fused x update needs the solver's scalars");
    launch_k(kerns[which], dim3(g), dim3(kThreads), 0, s, pdl, i0, i1, r, p, sc, bsrc, rs, history,
             links, psrc ? psrc : p, x, p0, role);
    TW_CUDA(cudaGetLastError());
}

void launch_dot(const double* a, const double* b, int64_t i0, int64_t i1, RedScratch rs, Fin fin,
                int blocks, cudaStream_t s) {
    const int g = clamp_blocks(i1 - i0, blocks);
    dot_kernel<<<g, kThreads, 0, s>>>(a, b, i0, i1, rs, fin);
    TW_CUDA(cudaGetLastError());
}

void launch_waxpby(double alpha, const double* x, double beta, const double* y, double* w,
                   int64_t i0, int64_t i1, int blocks, cudaStream_t s) {
    if (i1 <= i0) return;
    const int g = clamp_blocks(i1 - i0, blocks);
    waxpby_kernel<<<g, kThreads, 0, s>>>(alpha, x, beta, y, w, i0, i1);
    TW_CUDA(cudaGetLastError());
}

void launch_combine(const double* parts, int count, Fin fin, cudaStream_t s) {
    combine_kernel<<<1, 32, 0, s>>>(parts, count, fin);
    TW_CUDA(cudaGetLastError());
}

void launch_fill(double* p, int64_t n, double v, int blocks, cudaStream_t s) {
    if (n <= 0) return;
    fill_kernel<<<clamp_blocks(n, blocks), kThreads, 0, s>>>(p, n, v);
    TW_CUDA(cudaGetLastError());
}

void launch_rhs_splitmix(uint64_t seed, int64_t first, int64_t count, double* out, int blocks,
                         cudaStream_t s) {
    if (count <= 0) return;
    rhs_splitmix_kernel<<<clamp_blocks(count, blocks), kThreads, 0, s>>>(seed, first, count, out);
    TW_CUDA(cudaGetLastError());
}

void launch_rhs_xorshift(const uint64_t* chunk_states, int64_t chunk, int64_t count,
                         int64_t skip, double* out, int /*blocks*/, cudaStream_t s) {
    if (count <= 0) return;
    const int64_t nchunks = (count + skip + chunk - 1) / chunk;
    const int g = static_cast<int>((nchunks + kThreads - 1) / kThreads);
    rhs_xorshift_kernel<<<g, kThreads, 0, s>>>(chunk_states, chunk, count, skip, out);
    TW_CUDA(cudaGetLastError());
}

} // namespace tw

#ifdef TW_TIMELINE
extern "C" int tw_timeline_fetch(unsigned long long* host, int max_records) {
    unsigned n = 0;
    if (cudaMemcpyFromSymbol(&n, tw::tw_tl_n, sizeof(n)) != cudaSuccess) return -1;
    if (n > tw::kTlCap) n = tw::kTlCap;
    const unsigned m = static_cast<unsigned>(max_records) < n ? static_cast<unsigned>(max_records) : n;
    if (m && cudaMemcpyFromSymbol(host, tw::tw_tl_buf, static_cast<size_t>(m) * 32) != cudaSuccess)
        return -1;
    return static_cast<int>(n);
}
extern "C" int tw_timeline_reset() {
    const unsigned z = 0;
    return cudaMemcpyToSymbol(tw::tw_tl_n, &z, sizeof(z)) == cudaSuccess ? 0 : -1;
}
#endif
