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
// Coherence: p is rewritten inside the kernel (p_up) and gathered by later
// SpMV chunks, so gathers use coherent ld.global (not the read-only path);
// the acquire at chunk start plus a gpu-scope fence invalidates stale L1
// lines.  The matrix stream stays on TMA (read-only for the kernel).
#include <cuda_runtime.h>

#include <cstdint>

#include "tw_device.cuh"
#include "tw_internal.h"

namespace tw {

namespace {

using namespace dev;

#ifndef TW_DAG_WARPS
#define TW_DAG_WARPS 9
#endif
// Warps per dispatcher CTA.  Several CTAs share an SM so the chunk-boundary
// bookkeeping of one (ticket, dependency acquire, completion atomics) runs
// while the others stream.
constexpr int kDagWarps = TW_DAG_WARPS;

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

__global__ void __launch_bounds__(kDagWarps * 32, 2) dag_kernel(DagParams P) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bars[kDagWarps];
    __shared__ int stage_w[kDagWarps];
    __shared__ int s_chunk;
    __shared__ int s_last;
    __shared__ double red[32];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    unsigned char* stage = smem + static_cast<size_t>(warp) * P.stage_bytes;
    if (lane == 0) mbar_init(&bars[warp], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const uint64_t pol = l2_evict_first_policy();
    uint32_t phase = 0; // completed TMA phases of this warp's stage

    for (;;) {
        if (tid == 0) s_chunk = static_cast<int>(atomicAdd(P.ticket, 1u));
        __syncthreads();
        const int c = s_chunk;
        if (c >= P.nchunks) break;
        const int tk = P.chunk_task[c];
        const DagTask T = P.tasks[tk];
        const int j = c - T.chunk0;
        if (tid == 0) {
            if (c == 0) *P.start_stamp = globaltimer();
            while (ld_acquire(P.remaining + tk) > 0) __nanosleep(64);
            __threadfence(); // gpu-scope: orders the acquire, drops stale L1 lines
        }
        __syncthreads();

        double part = 0.0;
        switch (T.kind) {
        case DK_SPMV: {
            const int64_t s_first = T.r0 >> 5, s_end = (T.r1 + 31) >> 5;
            const int64_t s_lo = s_first + static_cast<int64_t>(j) * P.spmv_chunk_slices;
            int64_t s_hi = s_lo + P.spmv_chunk_slices;
            if (s_hi > s_end) s_hi = s_end;
            for (int64_t s = s_lo + warp; s < s_hi; s += kDagWarps) {
                if (lane == 0) {
                    const int64_t off = P.A.slice_off[s], end = P.A.slice_off[s + 1];
                    const uint32_t ents = static_cast<uint32_t>(end - off);
                    stage_w[warp] = static_cast<int>(ents >> 5);
                    mbar_expect_tx(&bars[warp], ents * 12u);
                    bulk_g2s(stage, P.A.vals + off, ents * 8u, &bars[warp], pol);
                    bulk_g2s(stage + P.val_bytes, P.A.cols + off, ents * 4u, &bars[warp], pol);
                }
                __syncwarp();
                mbar_wait(&bars[warp], phase & 1u);
                ++phase;
                const int w = stage_w[warp];
                const double* vb = reinterpret_cast<const double*>(stage);
                const int32_t* cb = reinterpret_cast<const int32_t*>(stage + P.val_bytes);
                double acc;
                switch (w) {
                case 27: acc = smem_row_fixed<27, false>(vb, cb, P.p_local, lane); break;
                case 18: acc = smem_row_fixed<18, false>(vb, cb, P.p_local, lane); break;
                case 12: acc = smem_row_fixed<12, false>(vb, cb, P.p_local, lane); break;
                case 8: acc = smem_row_fixed<8, false>(vb, cb, P.p_local, lane); break;
                default: acc = smem_row_generic<false>(vb, cb, P.p_local, lane, w); break;
                }
                const int64_t row = (s << 5) + lane;
                if (row >= T.r0 && row < T.r1) {
                    P.Ap[row] = acc;
                    part = __dadd_rn(part, __dmul_rn(P.p_owned[row], acc));
                }
                __syncwarp();
                if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            }
            break;
        }
        case DK_UPD: {
            const double alpha = P.sc->alpha, nalpha = -alpha;
            const int64_t a = T.r0 + static_cast<int64_t>(j) * P.vec_chunk_rows;
            int64_t b = a + P.vec_chunk_rows;
            if (b > T.r1) b = T.r1;
            // pairs (2i, 2i+1) fully inside [a, b) use 128-bit accesses
            const int64_t q0 = (a + 1) >> 1, q1 = b >> 1;
            for (int64_t q = q0 + tid; q < q1; q += blockDim.x) {
                const int64_t e = 2 * q;
                double2 xv = *reinterpret_cast<const double2*>(P.x + e);
                const double2 pv = *reinterpret_cast<const double2*>(P.p_owned + e);
                double2 rv = *reinterpret_cast<const double2*>(P.r + e);
                const double2 av = *reinterpret_cast<const double2*>(P.Ap + e);
                xv.x = __dadd_rn(xv.x, __dmul_rn(alpha, pv.x));
                xv.y = __dadd_rn(xv.y, __dmul_rn(alpha, pv.y));
                rv.x = __dadd_rn(rv.x, __dmul_rn(nalpha, av.x));
                rv.y = __dadd_rn(rv.y, __dmul_rn(nalpha, av.y));
                *reinterpret_cast<double2*>(P.x + e) = xv;
                *reinterpret_cast<double2*>(P.r + e) = rv;
                part = __dadd_rn(part, __dmul_rn(rv.x, rv.x));
                part = __dadd_rn(part, __dmul_rn(rv.y, rv.y));
            }
            if (tid < 2) { // ragged ends
                const int64_t i = tid == 0 ? a : b - 1;
                const bool mine = tid == 0 ? (a & 1) != 0 : ((b & 1) != 0 && b - 1 >= a && !((a & 1) && b - 1 == a));
                if (mine && i < b) {
                    const double xv = __dadd_rn(P.x[i], __dmul_rn(alpha, P.p_owned[i]));
                    const double rv = __dadd_rn(P.r[i], __dmul_rn(nalpha, P.Ap[i]));
                    P.x[i] = xv;
                    P.r[i] = rv;
                    part = __dadd_rn(part, __dmul_rn(rv, rv));
                }
            }
            break;
        }
        case DK_UPDP: {
            const double beta = P.sc->beta;
            const int64_t a = T.r0 + static_cast<int64_t>(j) * P.vec_chunk_rows;
            int64_t b = a + P.vec_chunk_rows;
            if (b > T.r1) b = T.r1;
            const int64_t q0 = (a + 1) >> 1, q1 = b >> 1;
            for (int64_t q = q0 + tid; q < q1; q += blockDim.x) {
                const int64_t e = 2 * q;
                const double2 rv = *reinterpret_cast<const double2*>(P.r + e);
                double2 pv = *reinterpret_cast<const double2*>(P.p_owned + e);
                pv.x = __dadd_rn(rv.x, __dmul_rn(beta, pv.x));
                pv.y = __dadd_rn(rv.y, __dmul_rn(beta, pv.y));
                *reinterpret_cast<double2*>(P.p_owned + e) = pv;
            }
            if (tid < 2) {
                const int64_t i = tid == 0 ? a : b - 1;
                const bool mine = tid == 0 ? (a & 1) != 0 : ((b & 1) != 0 && b - 1 >= a && !((a & 1) && b - 1 == a));
                if (mine && i < b) P.p_owned[i] = __dadd_rn(P.r[i], __dmul_rn(beta, P.p_owned[i]));
            }
            break;
        }
        case DK_ALPHA:
            if (tid == 0) { // alpha task: tile partials in tile order (cg.cpp:217-222)
                double pAp = 0.0;
                for (int t = 0; t < P.T; ++t) pAp = __dadd_rn(pAp, P.pa[t]);
                P.sc->pAp = pAp;
                P.sc->alpha = __ddiv_rn(P.sc->rtrans, pAp);
            }
            break;
        case DK_BETA:
            if (tid == 0) { // beta_res task (cg.cpp:299-309)
                double rr = 0.0;
                for (int t = 0; t < P.T; ++t) rr = __dadd_rn(rr, P.rr[t]);
                CgScalars* sc = P.sc;
                sc->rr = rr;
                sc->beta = __ddiv_rn(rr, sc->rtrans);
                sc->rtrans = rr;
                if (sc->iter < sc->history_cap) {
                    P.history[sc->iter] = __dsqrt_rn(rr);
                    P.stamps[sc->iter + 1] = globaltimer();
                }
                sc->iter = sc->iter + 1;
            }
            break;
        default:
            break;
        }

        const bool has_part = T.kind == DK_SPMV || T.kind == DK_UPD;
        if (has_part) {
            const double bsum = block_sum(part, red);
            if (tid == 0) P.chunk_part[c] = bsum;
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            const unsigned d = atomicAdd(P.chunk_done + tk, 1u);
            s_last = d + 1 == static_cast<unsigned>(T.nchunks);
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            if (has_part) {
                // tile partial = chunk partials summed in chunk order
                double acc = 0.0;
                for (int i = tid; i < T.nchunks; i += blockDim.x)
                    acc = __dadd_rn(acc, __ldcg(P.chunk_part + T.chunk0 + i));
                const double tot = block_sum(acc, red);
                if (tid == 0) (T.kind == DK_SPMV ? P.pa : P.rr)[T.tile] = tot;
            }
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                for (int k = 0; k < T.nsucc; ++k) atomicSub(P.remaining + P.succ[T.succ0 + k], 1);
            }
        }
    }
}

} // namespace

int dag_smem_bytes(int max_width, int* stage_bytes, int* val_bytes) {
    const int vb = ((32 * max_width * 8) + 127) / 128 * 128;
    const int cb = ((32 * max_width * 4) + 127) / 128 * 128;
    *val_bytes = vb;
    *stage_bytes = vb + cb;
    return kDagWarps * (vb + cb);
}

int dag_threads() { return kDagWarps * 32; }

// Grid = every dispatcher CTA the device can hold at once (all CTAs must be
// co-resident: a CTA may wait on chunks other CTAs hold).
int dag_blocks(int max_width, int sm_count) {
    int stage, vb;
    const int smem = dag_smem_bytes(max_width, &stage, &vb);
    TW_CUDA(cudaFuncSetAttribute(dag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per_sm = 0;
    TW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dag_kernel, kDagWarps * 32, smem));
    if (per_sm < 1) config_error("dispatcher CTA does not fit on an SM");
    return per_sm * sm_count;
}

void launch_dag(const DagParams& P, int blocks, cudaStream_t s) {
    int stage, vb;
    const int smem = dag_smem_bytes(P.A.max_width, &stage, &vb);
    dag_kernel<<<blocks, kDagWarps * 32, smem, s>>>(P);
    TW_CUDA(cudaGetLastError());
}

} // namespace tw
