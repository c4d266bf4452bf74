// Persistent device-side dispatcher for the cg_tasks block-task DAG
// (the paper's future work on fine task granularity,
// PAPER.md:715-729).
//
// One kernel executes K whole CG iterations of the DAG.  The host flattens
// the physical task graph (the same fused nodes and edges the stream/event
// executor uses, tw_cg.cpp) into a topologically ordered task table; every
// task is cut into chunks (slice ranges of an SpMV tile, row ranges of an
// update tile, one chunk for alpha / beta_res), and the chunks of all tasks
// form one ordered list.  Each CTA (one per SM, 18 warps, TMA stages as in
// the standalone SpMV) repeatedly:
//
//   1. takes the next chunk index from a global ticket,
//   2. waits until the chunk's task has no unfinished predecessor
//      (acquire-load of the task's dependency counter),
//   3. runs the chunk, writing a chunk partial for the tile-order dots,
//   4. counts the chunk done; the CTA finishing a task's last chunk sums the
//      chunk partials in chunk order (deterministic tile partial) and
//      release-decrements the counters of the task's successors.
//
// Chunks are handed out in topological order and every CTA is resident, so a
// CTA only ever waits on chunks taken earlier by running CTAs: no deadlock.
// Launch overhead per task disappears (a chunk costs one atomic), and tasks
// of consecutive iterations overlap wherever the DAG allows it.
//
// Coherence: p is rewritten inside the kernel (p_up) and read by later SpMV
// chunks, so gathers use coherent ld.global (not the read-only path); the
// acquire at chunk start plus a gpu-scope fence invalidates stale L1 lines.
// On an x-staged matrix the p runs come by TMA with the slice (as in the
// standalone K1), after a generic -> async proxy fence that orders them
// behind that acquire.  The matrix itself is read-only for the kernel.
#include <cuda_runtime.h>

#include <cstdint>

#include "tw_device.cuh"
#include "tw_internal.h"

namespace tw {

namespace {

using namespace dev;

#ifndef TW_DAG_WARPS
#define TW_DAG_WARPS 19
#endif
// Warps per dispatcher CTA: one CTA per SM with 18 compute warps (the
// standalone K1's warp count) and the scheduler warp, which takes the
// chunk-boundary bookkeeping (ticket, dependency acquire, completion
// atomics) off the compute warps.  All 18 share each chunk, so neighbouring
// slices' gathers share the SM's L1 (profiles/r01_dispatcher_summary.md).
constexpr int kDagWarps = TW_DAG_WARPS;
#ifndef TW_DAG_CTAS
#define TW_DAG_CTAS 1 // resident dispatcher CTAs per SM the register budget targets
#endif

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Named barriers of the slot ring (ids 1..4; 0 is __syncthreads).
__device__ __forceinline__ void bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

constexpr int kComputeWarps = kDagWarps - 1; // warp kDagWarps-1 schedules
#ifndef TW_DAG_VEC_UNROLL
#define TW_DAG_VEC_UNROLL 2
#endif
constexpr int kVecUnroll = TW_DAG_VEC_UNROLL; // pairs in flight per thread in update chunks
constexpr int kSlots = 2;

struct Slot {
    int c;     // chunk index, -1 = no more work
    int task;
    int ready; // the scheduler already observed (acquired) zero predecessors
    DagTask t;
};

// Stamp of the peer flags a task of iteration T.iter publishes / waits for.
__device__ __forceinline__ unsigned long long task_stamp(const DagRank& R, const DagTask& T) {
    return (static_cast<unsigned long long>(R.sc->epoch) << 32) |
           static_cast<unsigned long long>(R.iter0 + T.iter + 1);
}

// alpha / beta_res across ranks, in two halves so that no publication ever
// waits behind a wait (one thread each):
//  * publish: by the scheduler completing the rank's LAST SpMV (x/r) tile of
//    the iteration -- the tile partials summed in tile order into slot
//    `rank` of every rank's window, its flag raised with the stamp
//    (release, system scope); it waits on nothing;
//  * gather: by the alpha (beta_res) task, once every rank's flag in the own
//    window carries the stamp -- the partials summed in rank order, the sum
//    the NCCL executor forms from its allgather (tw_cg_dist.cpp).
// Every wait of the dispatcher is then on chunks with smaller tickets
// (earlier in the table's order), which every CTA runs in ticket order: the
// lowest-ticket waiting chunk always gets its producer.
__device__ __noinline__ void publish_partial(const DagRank& R, const DagTask& T, int ntiles,
                                             bool a) {
    const double* tp = a ? R.pa : R.rr;
    double v = 0.0;
    for (int t = 0; t < ntiles; ++t) v = __dadd_rn(v, __ldcg(tp + t));
    const PeerLinks* L = R.links;
    const int me = L->rank, P = L->nranks;
    const unsigned long long st = task_stamp(R, T);
    for (int q = 0; q < P; ++q) (a ? L->win[q]->recv_a : L->win[q]->recv_b)[me] = v;
    for (int q = 0; q < P; ++q) st_release_sys((a ? L->win[q]->flag_a : L->win[q]->flag_b) + me, st);
}

__device__ __noinline__ double gather_partials(const DagRank& R, const DagTask& T, bool a) {
    const int P = R.links->nranks;
    const unsigned long long st = task_stamp(R, T);
    thread_wait_flags(a ? R.win->flag_a : R.win->flag_b, P, st);
    double s = 0.0;
    for (int q = 0; q < P; ++q) s = __dadd_rn(s, __ldcg((a ? R.win->recv_a : R.win->recv_b) + q));
    return s;
}

// One chunk on the compute warps; returns this thread's dot partial.
// XP: the paired-x-update instantiation (buffer choice per task); the
// other one compiles the single-update chunks without that generality
// (which cost 3 us per iteration at 128^3 when it was a runtime choice)
template <bool XP>
__device__ __forceinline__ double run_chunk(const DagParams& P, const DagTask& T, int j, int warp,
                                            int lane, unsigned char* stage, uint64_t* bar,
                                            int* stage_w, uint32_t& phase, uint64_t pol) {
    TW_DCHECK(T.rank >= 0 && T.rank < P.nranks);
    const DagRank& R = P.rk[T.rank];
    const int ctid = warp * 32 + lane, cthreads = kComputeWarps * 32;
    double part = 0.0;
    switch (T.kind) {
    case DK_SPMV: {
#ifdef TW_DAG_PROBE_SKIP_SPMV // timing probe only (wrong results): SpMV chunks do nothing
        break;
#endif
        const int64_t s_first = T.r0 >> 5, s_end = (T.r1 + 31) >> 5;
        const int64_t s_lo = s_first + static_cast<int64_t>(j) * P.spmv_chunk_slices;
        int64_t s_hi = s_lo + P.spmv_chunk_slices;
        if (s_hi > s_end) s_hi = s_end;
        // p of this iteration: the pair buffer in the second of an x pair
        const bool p2 = XP && (T.flags & kDagReadP2) != 0;
        const double* pl = p2 ? R.p2_local : R.p_local;
        const double* po = p2 ? R.p2_owned : R.p_owned;
        TW_DCHECK(pl != nullptr);
        if (R.A.cols16) { // x-staged matrix: the slice's x runs ride its TMA transaction
            // a tile reading a ghost plane: the neighbour's halo task of this
            // iteration must have landed it (its flag carries the stamp)
            if (lane == 0 && (T.flags & (kDagGhostLo | kDagGhostHi))) {
                const unsigned long long st = task_stamp(R, T);
                if (T.flags & kDagGhostLo) thread_wait_flags(&R.win->flag_ghost_lo, 1, st);
                if (T.flags & kDagGhostHi) thread_wait_flags(&R.win->flag_ghost_hi, 1, st);
            }
            // p was written inside this kernel by other CTAs' generic stores
            // (made visible by the chunk's dependency acquire); order this
            // warp's async-proxy reads of it after that acquire
            if (lane == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
            const double* vb = reinterpret_cast<const double*>(stage);
            const uint16_t* cb = reinterpret_cast<const uint16_t*>(stage + P.val_bytes);
            double* xs = reinterpret_cast<double*>(stage + P.val_bytes + P.c16_bytes);
            constexpr uint32_t kRunBytes = kStageRunLen * 8;
            for (int64_t s = s_lo + warp; s < s_hi; s += kComputeWarps) {
                if (lane == 0) {
                    const int64_t off = R.A.slice_off[s];
                    const uint32_t ents = static_cast<uint32_t>(R.A.slice_off[s + 1] - off);
                    TW_DCHECK(ents <= 32u * static_cast<uint32_t>(P.max_width)); // fits the stage
                    *stage_w = static_cast<int>(ents >> 5);
                    mbar_expect_tx(bar, ents * 10u + kStageRuns * kRunBytes);
                    if (ents) {
                        bulk_g2s(stage, R.A.vals + off, ents * 8u, bar, pol);
                        bulk_g2s(stage + P.val_bytes, R.A.cols16 + off, ents * 2u, bar, pol);
                    }
                    int64_t starts[kStageRuns];
                    run_starts(R.A, s, starts);
#pragma unroll
                    for (int r = 0; r < kStageRuns; ++r) {
                        const int64_t st = starts[r];
                        TW_DCHECK(st >= -2 && st <= R.A.x_len);
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
                            " [%0], [%1], %2, [%3];" ::"r"(smem_u32(xs + r * kStageRunLen)),
                            "l"(pl + st), "r"(kRunBytes), "r"(smem_u32(bar))
                            : "memory");
                    }
                }
                __syncwarp();
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
                if (row >= T.r0 && row < T.r1) {
                    R.Ap[row] = acc;
                    part = __dadd_rn(part, __dmul_rn(xs[4 * kStageRunLen + 2 + lane], acc));
                }
                __syncwarp();
                if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            }
            break;
        }
        for (int64_t s = s_lo + warp; s < s_hi; s += kComputeWarps) {
            if (lane == 0) {
                const int64_t off = R.A.slice_off[s], end = R.A.slice_off[s + 1];
                const uint32_t ents = static_cast<uint32_t>(end - off);
                TW_DCHECK(ents <= 32u * static_cast<uint32_t>(P.max_width)); // fits the stage
                *stage_w = static_cast<int>(ents >> 5);
                mbar_expect_tx(bar, ents * 12u); // ents == 0 (all rows empty): completes at once
                if (ents) {
                    bulk_g2s(stage, R.A.vals + off, ents * 8u, bar, pol);
                    bulk_g2s(stage + P.val_bytes, R.A.cols + off, ents * 4u, bar, pol);
                }
            }
            __syncwarp();
            mbar_wait(bar, phase & 1u);
            ++phase;
            const int w = *stage_w;
            const double* vb = reinterpret_cast<const double*>(stage);
            const int32_t* cb = reinterpret_cast<const int32_t*>(stage + P.val_bytes);
            double acc;
            switch (w) {
            case 27: acc = smem_row_fixed<27, kGatherCA>(vb, cb, pl, lane); break;
            case 18: acc = smem_row_fixed<18, kGatherCA>(vb, cb, pl, lane); break;
            case 12: acc = smem_row_fixed<12, kGatherCA>(vb, cb, pl, lane); break;
            case 8: acc = smem_row_fixed<8, kGatherCA>(vb, cb, pl, lane); break;
            default: acc = smem_row_generic<kGatherCA>(vb, cb, pl, lane, w); break;
            }
            const int64_t row = (s << 5) + lane;
            if (row >= T.r0 && row < T.r1) {
                R.Ap[row] = acc;
                part = __dadd_rn(part, __dmul_rn(po[row], acc));
            }
            __syncwarp();
            if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        break;
    }
    case DK_HALO: {
        // this rank's first / last owned plane of p into the neighbours'
        // ghost planes (NVLink stores; the scheduler raises the flags); in
        // the second iteration of an x pair from and into the pair buffers
        const bool p2 = XP && (T.flags & kDagReadP2) != 0;
        const PeerLinks* L = p2 ? R.links2 : R.links;
        if (!L) break; // no neighbours
        const double* src = p2 ? R.p2_owned : R.p_owned;
        const int64_t pl = L->plane, n = R.A.n_rows;
        for (int64_t i = ctid; i < pl; i += cthreads) {
            if (L->ghost_lo_dst) L->ghost_lo_dst[i] = __ldcg(src + i);
            if (L->ghost_hi_dst) L->ghost_hi_dst[i] = __ldcg(src + n - pl + i);
        }
        break;
    }
    case DK_UPD:
    case DK_UPDP: {
#ifdef TW_DAG_PROBE_SKIP_UPD // timing probe only (wrong results): update chunks do nothing
        break;
#endif
        const bool upd = T.kind == DK_UPD;
        // paired x updates (p updates only): defer = p into the pair buffer,
        // x left alone; pair = x = (x + alpha_prev p0) + alpha p1 with p1 the
        // pair buffer and p0 = p_owned, p back into p_owned
        const bool xdef = XP && !upd && (T.flags & kDagXDefer) != 0;
        const bool xpair = XP && !upd && (T.flags & kDagXPair) != 0;
        // x_in_updp: x += alpha p_old rides on the p update's read of p_old
        // (alpha of this iteration is still in sc: the next alpha task waits
        // for every p update of this one)
        const bool xin = P.x_in_updp != 0 && !xdef;
        const double alpha = upd || xin ? R.sc->alpha : 0.0, nalpha = -alpha;
        const double alpha0 = xpair ? R.sc->alpha_prev : 0.0;
        const double beta = upd ? 0.0 : R.sc->beta;
        const double* pin = xpair ? R.p2_owned : R.p_owned;  // this iteration's p_old
        double* pout = xdef ? R.p2_owned : R.p_owned;       // the new p
        const int64_t a = T.r0 + static_cast<int64_t>(j) * P.vec_chunk_rows;
        int64_t b = a + P.vec_chunk_rows;
        if (b > T.r1) b = T.r1;
        // the pair's four operand streams take the x/r chunks' block size
        const int sb = upd || xpair ? P.upd_block_rows : P.updp_block_rows;
        TW_DCHECK(!(xdef || xpair) || (sb > 0 && P.x_in_updp));
        if (sb > 0) {
            // TMA path: each warp streams blocks of sb rows of its operands
            // (x, p, r, Ap or r, p) into its stage with bulk copies -- a whole
            // stage in flight per warp, no registers held -- and writes the
            // results back with 128-bit stores.  Rows [a2, b2) are the
            // 16-byte-aligned pairs; the ragged ends go scalar below.
            if (lane == 0) asm volatile("fence.proxy.async.global;" ::: "memory"); // see SpMV
            const int64_t a2 = (a + 1) & ~int64_t(1), b2 = b & ~int64_t(1);
            double* s0 = reinterpret_cast<double*>(stage);
            double* s1 = s0 + sb;
            double* s2 = s1 + sb;
            double* s3 = s2 + sb;
            for (int64_t q = a2 + static_cast<int64_t>(warp) * sb; q < b2;
                 q += static_cast<int64_t>(kComputeWarps) * sb) {
                const int rows = static_cast<int>((q + sb < b2 ? q + sb : b2) - q);
                const uint32_t bytes = static_cast<uint32_t>(rows) * 8u;
                if (lane == 0) {
                    mbar_expect_tx(bar, (upd ? (xin ? 2u : 4u) : xpair ? 4u : (xin ? 3u : 2u)) * bytes);
                    if (xpair) { // r, p1, p0, x
                        bulk_g2s_plain(s0, R.r + q, bytes, bar);
                        bulk_g2s_plain(s1, pin + q, bytes, bar);
                        bulk_g2s_plain(s2, R.p_owned + q, bytes, bar);
                        bulk_g2s_plain(s3, R.x + q, bytes, bar);
                    } else if (upd && xin) { // r, Ap
                        bulk_g2s_plain(s0, R.r + q, bytes, bar);
                        bulk_g2s_plain(s1, R.Ap + q, bytes, bar);
                    } else if (upd) {
                        bulk_g2s_plain(s0, R.x + q, bytes, bar);
                        bulk_g2s_plain(s1, R.p_owned + q, bytes, bar);
                        bulk_g2s_plain(s2, R.r + q, bytes, bar);
                        bulk_g2s_plain(s3, R.Ap + q, bytes, bar);
                    } else { // r, p (and x)
                        bulk_g2s_plain(s0, R.r + q, bytes, bar);
                        bulk_g2s_plain(s1, pin + q, bytes, bar);
                        if (xin) bulk_g2s_plain(s2, R.x + q, bytes, bar);
                    }
                }
                __syncwarp();
                mbar_wait(bar, phase & 1u);
                ++phase;
                for (int i = 2 * lane; i < rows; i += 64) {
                    if (xpair) {
                        const double2 rv = *reinterpret_cast<const double2*>(s0 + i);
                        double2 pv = *reinterpret_cast<const double2*>(s1 + i);
                        const double2 ov = *reinterpret_cast<const double2*>(s2 + i);
                        double2 xv = *reinterpret_cast<const double2*>(s3 + i);
                        xv.x = __dadd_rn(__dadd_rn(xv.x, __dmul_rn(alpha0, ov.x)), __dmul_rn(alpha, pv.x));
                        xv.y = __dadd_rn(__dadd_rn(xv.y, __dmul_rn(alpha0, ov.y)), __dmul_rn(alpha, pv.y));
                        *reinterpret_cast<double2*>(R.x + q + i) = xv;
                        pv.x = __dadd_rn(rv.x, __dmul_rn(beta, pv.x));
                        pv.y = __dadd_rn(rv.y, __dmul_rn(beta, pv.y));
                        *reinterpret_cast<double2*>(pout + q + i) = pv;
                    } else if (upd && xin) {
                        double2 rv = *reinterpret_cast<const double2*>(s0 + i);
                        const double2 av = *reinterpret_cast<const double2*>(s1 + i);
                        rv.x = __dadd_rn(rv.x, __dmul_rn(nalpha, av.x));
                        rv.y = __dadd_rn(rv.y, __dmul_rn(nalpha, av.y));
                        *reinterpret_cast<double2*>(R.r + q + i) = rv;
                        part = __dadd_rn(part, __dmul_rn(rv.x, rv.x));
                        part = __dadd_rn(part, __dmul_rn(rv.y, rv.y));
                    } else if (upd) {
                        double2 xv = *reinterpret_cast<const double2*>(s0 + i);
                        const double2 pv = *reinterpret_cast<const double2*>(s1 + i);
                        double2 rv = *reinterpret_cast<const double2*>(s2 + i);
                        const double2 av = *reinterpret_cast<const double2*>(s3 + i);
                        xv.x = __dadd_rn(xv.x, __dmul_rn(alpha, pv.x));
                        xv.y = __dadd_rn(xv.y, __dmul_rn(alpha, pv.y));
                        rv.x = __dadd_rn(rv.x, __dmul_rn(nalpha, av.x));
                        rv.y = __dadd_rn(rv.y, __dmul_rn(nalpha, av.y));
                        *reinterpret_cast<double2*>(R.x + q + i) = xv;
                        *reinterpret_cast<double2*>(R.r + q + i) = rv;
                        part = __dadd_rn(part, __dmul_rn(rv.x, rv.x));
                        part = __dadd_rn(part, __dmul_rn(rv.y, rv.y));
                    } else {
                        const double2 rv = *reinterpret_cast<const double2*>(s0 + i);
                        double2 pv = *reinterpret_cast<const double2*>(s1 + i);
                        if (xin) {
                            double2 xv = *reinterpret_cast<const double2*>(s2 + i);
                            xv.x = __dadd_rn(xv.x, __dmul_rn(alpha, pv.x));
                            xv.y = __dadd_rn(xv.y, __dmul_rn(alpha, pv.y));
                            *reinterpret_cast<double2*>(R.x + q + i) = xv;
                        }
                        pv.x = __dadd_rn(rv.x, __dmul_rn(beta, pv.x));
                        pv.y = __dadd_rn(rv.y, __dmul_rn(beta, pv.y));
                        *reinterpret_cast<double2*>(pout + q + i) = pv;
                    }
                }
                __syncwarp();
                if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            }
        } else {
        // pairs (2q, 2q+1) inside [a, b) with 128-bit accesses, ragged ends scalar
        const int64_t q0 = (a + 1) >> 1, q1 = b >> 1;
        // kVecUnroll pairs per thread and step, every load issued before the
        // first store: the few compute warps of a dispatcher CTA need that
        // many bytes in flight to stream at HBM rate.  The per-thread sum
        // still runs q, q + cthreads, q + 2 cthreads, ... as a one-pair loop.
        constexpr int U = kVecUnroll;
        for (int64_t q = q0 + ctid; q < q1; q += U * cthreads) {
            if (upd) {
                double2 xv[U], pv[U], rv[U], av[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t e = 2 * (q + static_cast<int64_t>(u) * cthreads);
                    if (e < 2 * q1) {
                        xv[u] = *reinterpret_cast<const double2*>(R.x + e);
                        pv[u] = *reinterpret_cast<const double2*>(R.p_owned + e);
                        rv[u] = *reinterpret_cast<const double2*>(R.r + e);
                        av[u] = *reinterpret_cast<const double2*>(R.Ap + e);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t e = 2 * (q + static_cast<int64_t>(u) * cthreads);
                    if (e < 2 * q1) {
                        xv[u].x = __dadd_rn(xv[u].x, __dmul_rn(alpha, pv[u].x));
                        xv[u].y = __dadd_rn(xv[u].y, __dmul_rn(alpha, pv[u].y));
                        rv[u].x = __dadd_rn(rv[u].x, __dmul_rn(nalpha, av[u].x));
                        rv[u].y = __dadd_rn(rv[u].y, __dmul_rn(nalpha, av[u].y));
                        *reinterpret_cast<double2*>(R.x + e) = xv[u];
                        *reinterpret_cast<double2*>(R.r + e) = rv[u];
                        part = __dadd_rn(part, __dmul_rn(rv[u].x, rv[u].x));
                        part = __dadd_rn(part, __dmul_rn(rv[u].y, rv[u].y));
                    }
                }
            } else {
                double2 rv[U], pv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t e = 2 * (q + static_cast<int64_t>(u) * cthreads);
                    if (e < 2 * q1) {
                        rv[u] = *reinterpret_cast<const double2*>(R.r + e);
                        pv[u] = *reinterpret_cast<const double2*>(R.p_owned + e);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t e = 2 * (q + static_cast<int64_t>(u) * cthreads);
                    if (e < 2 * q1) {
                        pv[u].x = __dadd_rn(rv[u].x, __dmul_rn(beta, pv[u].x));
                        pv[u].y = __dadd_rn(rv[u].y, __dmul_rn(beta, pv[u].y));
                        *reinterpret_cast<double2*>(R.p_owned + e) = pv[u];
                    }
                }
            }
        }
        } // register path
        const int64_t lo = (a & 1) ? a : -1;                               // odd start
        const int64_t hi = ((b & 1) && b - 1 >= a && b - 1 != lo) ? b - 1 : -1; // odd end
        const int64_t i = ctid == 0 ? lo : (ctid == 1 ? hi : -1);
        if (i >= 0) {
            if (upd) {
                if (!xin) R.x[i] = __dadd_rn(R.x[i], __dmul_rn(alpha, R.p_owned[i]));
                const double rv = __dadd_rn(R.r[i], __dmul_rn(nalpha, R.Ap[i]));
                R.r[i] = rv;
                part = __dadd_rn(part, __dmul_rn(rv, rv));
            } else {
                const double pv = pin[i];
                if (xpair) R.x[i] = __dadd_rn(R.x[i], __dmul_rn(alpha0, R.p_owned[i]));
                if (xin) R.x[i] = __dadd_rn(R.x[i], __dmul_rn(alpha, pv));
                pout[i] = __dadd_rn(R.r[i], __dmul_rn(beta, pv));
            }
        }
        break;
    }
    default:
        break;
    }
    return part;
}

// The scheduler warp's side of a chunk: alpha / beta_res bodies (one thread),
// then the chunk partial, completion count and, for a task's last chunk, the
// tile partial in chunk order and the release of the successors.
__device__ __forceinline__ void complete_chunk(const DagParams& P, const Slot& S,
                                               const double* wpart, int lane) {
    const DagTask& T = S.t;
    const DagRank& R = P.rk[T.rank];
    if (lane == 0) {
        if (T.kind == DK_ALPHA) { // alpha task: tile partials in tile order (cg.cpp:217-222)
            double pAp = 0.0;
            if (R.links) {
                pAp = gather_partials(R, T, true);
            } else {
                for (int t = 0; t < P.T; ++t) pAp = __dadd_rn(pAp, R.pa[t]);
            }
            R.sc->pAp = pAp;
            R.sc->alpha_prev = R.sc->alpha; // paired x updates
            R.sc->alpha = __ddiv_rn(R.sc->rtrans, pAp);
        } else if (T.kind == DK_BETA) { // beta_res task (cg.cpp:299-309)
            double rr = 0.0;
            if (R.links) {
                rr = gather_partials(R, T, false);
            } else {
                for (int t = 0; t < P.T; ++t) rr = __dadd_rn(rr, R.rr[t]);
            }
            CgScalars* sc = R.sc;
            sc->rr = rr;
            sc->beta = __ddiv_rn(rr, sc->rtrans);
            sc->rtrans = rr;
            if (sc->iter < sc->history_cap) {
                R.history[sc->iter] = __dsqrt_rn(rr);
                R.stamps[sc->iter + 1] = globaltimer();
            }
            sc->iter = sc->iter + 1;
        }
    }
    if (T.kind == DK_HALO && R.links && lane == 0) {
        // the compute warps' plane stores (ordered before the slot's EMPTY
        // barrier) land in the neighbours' memory, then their ghost flags rise
        __threadfence_system();
        const unsigned long long st = task_stamp(R, T);
        if (R.links->ghost_lo_flag) st_release_sys(R.links->ghost_lo_flag, st);
        if (R.links->ghost_hi_flag) st_release_sys(R.links->ghost_hi_flag, st);
    }
    const bool has_part = T.kind == DK_SPMV || T.kind == DK_UPD;
    unsigned last = 0;
    if (lane == 0) {
        if (has_part) {
            double s = 0.0;
            for (int w = 0; w < kComputeWarps; ++w) s = __dadd_rn(s, wpart[w]);
            P.chunk_part[S.c] = s;
        }
        __threadfence();
        const unsigned d = atomicAdd(P.chunk_done + S.task, 1u);
        last = d + 1 == static_cast<unsigned>(T.nchunks);
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    __threadfence();
    if (has_part) { // tile partial = chunk partials summed in chunk order
        double acc = 0.0;
        for (int i = lane; i < T.nchunks; i += 32) acc = __dadd_rn(acc, __ldcg(P.chunk_part + T.chunk0 + i));
        acc = warp_sum(acc);
        if (lane == 0) {
            (T.kind == DK_SPMV ? R.pa : R.rr)[T.tile] = acc;
            if (R.links) { // across ranks: the last tile of the phase publishes
                __threadfence();
                const bool sp = T.kind == DK_SPMV;
                const unsigned d = atomicInc(R.tctr + (sp ? 0 : 1), static_cast<unsigned>(P.T - 1));
                if (d == static_cast<unsigned>(P.T - 1)) { // wraps to 0: reset for the next iteration
                    __threadfence();
                    publish_partial(R, T, P.T, sp);
                }
            }
        }
    }
    __syncwarp();
    if (lane == 0) __threadfence();
    __syncwarp();
    for (int k = lane; k < T.nsucc; k += 32) atomicSub(P.remaining + P.succ[T.succ0 + k], 1);
}

// Takes the next chunk (scheduler warp).  Never blocks on dependencies: the
// scheduler must stay free to complete the chunk the compute warps are
// running, which the new chunk may depend on.  If the task is already
// runnable the acquire and the L1 invalidation happen here, off the critical
// path; otherwise the compute warps wait for it.
__device__ __forceinline__ void fill_slot(const DagParams& P, Slot* S, int lane) {
    if (lane == 0) {
        const int c = static_cast<int>(atomicAdd(P.ticket, 1u));
        if (c >= P.nchunks) {
            S->c = -1;
        } else {
            const int tk = P.chunk_task[c];
            TW_DCHECK(tk >= 0 && tk < P.ntasks);
            S->c = c;
            S->task = tk;
            S->t = P.tasks[tk];
            if (c == 0) *P.start_stamp = globaltimer();
            S->ready = ld_acquire(P.remaining + tk) <= 0;
            if (S->ready) __threadfence(); // gpu scope: drop stale L1 lines
        }
    }
    __syncwarp();
}

// Persistent dispatcher CTA: kComputeWarps compute warps + 1 scheduler warp
// over a 2-slot ring.  The scheduler fills slot b+1 (ticket, task record,
// dependency acquire) while the compute warps run slot b, and completes slot
// b (partials, counters, successor release) while they run slot b+1, so the
// per-chunk bookkeeping is off the critical path and chunks can be small.
template <bool XP>
__global__ void __launch_bounds__(kDagWarps * 32, TW_DAG_CTAS) dag_kernel(const __grid_constant__ DagParams P) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bars[kComputeWarps];
    __shared__ int stage_w[kComputeWarps];
    __shared__ Slot slots[kSlots];
    __shared__ double wpart[kSlots][kComputeWarps];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int kAll = kDagWarps * 32;
    if (warp < kComputeWarps && lane == 0) mbar_init(&bars[warp], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();

    if (warp == kComputeWarps) { // ---------------------------------- scheduler
        for (int b = 0; b < kSlots; ++b) {
            fill_slot(P, &slots[b], lane);
            bar_arrive(1 + b, kAll); // FULL[b]
        }
        for (int k = 0;; ++k) {
            const int b = k & 1;
            if (slots[b].c < 0) break; // compute warps saw the end marker too
            bar_sync(3 + b, kAll);     // EMPTY[b]: compute warps done with slot b
            complete_chunk(P, slots[b], wpart[b], lane);
            fill_slot(P, &slots[b], lane);
            bar_arrive(1 + b, kAll);
        }
        return;
    }
    // -------------------------------------------------------------- compute
    unsigned char* stage = smem + static_cast<size_t>(warp) * P.stage_bytes;
    const uint64_t pol = l2_evict_first_policy();
    uint32_t phase = 0;
    for (int k = 0;; ++k) {
        const int b = k & 1;
        bar_sync(1 + b, kAll); // FULL[b]
        const int c = slots[b].c;
        if (c < 0) break;
        if (!slots[b].ready) { // wait for the task's predecessors (compute warps only)
            if (tid == 0) {
                // bounded like every device wait of the library: a broken
                // task table (a counter that never reaches zero) reports and
                // traps instead of hanging the GPU
                unsigned spins = 0;
                unsigned long long t0 = 0;
                while (ld_acquire(P.remaining + slots[b].task) > 0) {
                    __nanosleep(32);
                    if ((++spins & 4095u) == 0) {
                        const unsigned long long t = global_ns();
                        if (!t0) {
                            t0 = t;
                        } else if (t - t0 > TW_PEER_TIMEOUT_NS) {
                            printf("tw_hpccg: dispatcher task %d still has %d predecessors\n",
                                   slots[b].task, ld_acquire(P.remaining + slots[b].task));
                            __trap();
                        }
                    }
                }
                __threadfence();
            }
            bar_sync(5, kComputeWarps * 32);
        }
        const DagTask T = slots[b].t;
        const double part = run_chunk<XP>(P, T, c - T.chunk0, warp, lane, stage, &bars[warp],
                                      &stage_w[warp], phase, pol);
        const double ws = warp_sum(part);
        if (lane == 0) wpart[b][warp] = ws;
        bar_arrive(3 + b, kAll); // EMPTY[b]
    }
}

} // namespace

int dag_smem_bytes(int max_width, bool staged, int* stage_bytes, int* val_bytes, int* c16_bytes) {
    const int vb = ((32 * max_width * 8) + 127) / 128 * 128;
    // x-staged: 16-bit columns and the 9 x runs; else 32-bit columns
    const int cb = ((32 * max_width * (staged ? 2 : 4)) + 127) / 128 * 128;
    const int xb = staged ? (kStageRuns * kStageRunLen * 8 + 127) / 128 * 128 : 0;
    *val_bytes = vb;
    *c16_bytes = cb;
    *stage_bytes = vb + cb + xb;
    return kComputeWarps * *stage_bytes; // the scheduler warp has no stage
}

int dag_threads() { return kDagWarps * 32; }

int dag_compute_warps() { return kComputeWarps; }

// Grid = every dispatcher CTA the device can hold at once (all CTAs must be
// co-resident: a CTA may wait on chunks other CTAs hold).
int dag_blocks(int max_width, bool staged, int sm_count) {
    int stage, vb, cb;
    const int smem = dag_smem_bytes(max_width, staged, &stage, &vb, &cb);
    TW_CUDA(cudaFuncSetAttribute(dag_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    TW_CUDA(cudaFuncSetAttribute(dag_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per_sm = 0;
    int per_sm_xp = 0; // both instantiations must fit the same grid
    TW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dag_kernel<false>, kDagWarps * 32, smem));
    TW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_xp, dag_kernel<true>, kDagWarps * 32, smem));
    per_sm = std::min(per_sm, per_sm_xp);
    if (per_sm < 1) config_error("dispatcher CTA does not fit on an SM");
    return per_sm * sm_count;
}

void launch_dag(const DagParams& P, int blocks, cudaStream_t s) {
    int stage, vb, cb;
    const int smem = dag_smem_bytes(P.max_width, P.rk[0].A.cols16 != nullptr, &stage, &vb, &cb);
    if (P.x_pairs)
        dag_kernel<true><<<blocks, kDagWarps * 32, smem, s>>>(P);
    else
        dag_kernel<false><<<blocks, kDagWarps * 32, smem, s>>>(P);
    TW_CUDA(cudaGetLastError());
}

} // namespace tw
