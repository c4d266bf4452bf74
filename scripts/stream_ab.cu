// K2 / K3 streaming A/B (tuning tool, not product code): the two vector
// passes of the CG iteration at the headline size, in several forms.
//   K2 shape: r -= a Ap; r.r partial        (reads r, Ap; writes r)      24 B/row
//   K3 shape: x += a p; p = r + b p         (reads r, p, x; writes p, x) 40 B/row
// Forms:
//   reg<U>      grid-stride 128-bit loads, U pairs in flight per thread (the product's form)
//   tma<S,CH>   persistent CTAs, an S-stage ring of CH-row chunks per operand
//               filled by cp.async.bulk (one elected thread), results stored
//               from registers with 128-bit streaming stores
//   tmas<S,CH>  the same with the results written back by cp.async.bulk
//               shared->global (bulk_group) from a staging buffer
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_ab scripts/stream_ab.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    printf("%s: %s (line %d)\n", #x, cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
                 "@!P1 bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void g2s(void* d, const void* s, uint32_t n, uint64_t* b, uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                 " [%0], [%1], %2, [%3], %4;" ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)), "l"(pol) : "memory");
}
__device__ __forceinline__ void s2g(void* d, const void* s, uint32_t n) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d), "r"(su32(s)), "r"(n) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void block_store_part(double v, double* out) {
    __shared__ double red[32];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        out[blockIdx.x] = t;
    }
}

// ---------------------------------------------------------------- register forms
template <int U>
__global__ void __launch_bounds__(256) k2_reg(int64_t n, double* __restrict__ r, const double* __restrict__ Ap,
                                              double na, double* parts) {
    const int64_t np = n / 2, stride = (int64_t)gridDim.x * blockDim.x;
    double part = 0;
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; j + (U - 1) * stride < np; j += U * stride) {
        double2 rv[U], av[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            rv[u] = __ldcs(reinterpret_cast<const double2*>(r) + j + u * stride);
            av[u] = __ldcs(reinterpret_cast<const double2*>(Ap) + j + u * stride);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            rv[u].x = __dadd_rn(rv[u].x, __dmul_rn(na, av[u].x));
            rv[u].y = __dadd_rn(rv[u].y, __dmul_rn(na, av[u].y));
            __stcs(reinterpret_cast<double2*>(r) + j + u * stride, rv[u]);
            part = __dadd_rn(part, __dmul_rn(rv[u].x, rv[u].x));
            part = __dadd_rn(part, __dmul_rn(rv[u].y, rv[u].y));
        }
    }
    for (; j < np; j += stride) {
        double2 rv = __ldcs(reinterpret_cast<const double2*>(r) + j);
        const double2 av = __ldcs(reinterpret_cast<const double2*>(Ap) + j);
        rv.x = __dadd_rn(rv.x, __dmul_rn(na, av.x));
        rv.y = __dadd_rn(rv.y, __dmul_rn(na, av.y));
        __stcs(reinterpret_cast<double2*>(r) + j, rv);
        part = __dadd_rn(part, __dmul_rn(rv.x, rv.x));
        part = __dadd_rn(part, __dmul_rn(rv.y, rv.y));
    }
    block_store_part(part, parts);
}

template <int U>
__global__ void __launch_bounds__(256) k3_reg(int64_t n, const double* __restrict__ r, double* __restrict__ p,
                                              double* __restrict__ x, double a, double b) {
    const int64_t np = n / 2, stride = (int64_t)gridDim.x * blockDim.x;
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; j + (U - 1) * stride < np; j += U * stride) {
        double2 rv[U], pv[U], xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            rv[u] = __ldcs(reinterpret_cast<const double2*>(r) + j + u * stride);
            pv[u] = __ldcs(reinterpret_cast<const double2*>(p) + j + u * stride);
            xv[u] = __ldcs(reinterpret_cast<const double2*>(x) + j + u * stride);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            xv[u].x = __dadd_rn(xv[u].x, __dmul_rn(a, pv[u].x));
            xv[u].y = __dadd_rn(xv[u].y, __dmul_rn(a, pv[u].y));
            pv[u].x = __dadd_rn(rv[u].x, __dmul_rn(b, pv[u].x));
            pv[u].y = __dadd_rn(rv[u].y, __dmul_rn(b, pv[u].y));
            __stcs(reinterpret_cast<double2*>(x) + j + u * stride, xv[u]);
            __stcs(reinterpret_cast<double2*>(p) + j + u * stride, pv[u]);
        }
    }
    for (; j < np; j += stride) {
        double2 rv = __ldcs(reinterpret_cast<const double2*>(r) + j);
        double2 pv = __ldcs(reinterpret_cast<const double2*>(p) + j);
        double2 xv = __ldcs(reinterpret_cast<const double2*>(x) + j);
        xv.x = __dadd_rn(xv.x, __dmul_rn(a, pv.x));
        xv.y = __dadd_rn(xv.y, __dmul_rn(a, pv.y));
        pv.x = __dadd_rn(rv.x, __dmul_rn(b, pv.x));
        pv.y = __dadd_rn(rv.y, __dmul_rn(b, pv.y));
        __stcs(reinterpret_cast<double2*>(x) + j, xv);
        __stcs(reinterpret_cast<double2*>(p) + j, pv);
    }
}

// ---------------------------------------------------------------- TMA forms
// NOPS operands per chunk (K2: r, Ap; K3: r, p, x), S stages of CH rows each.
// Chunk c of this CTA: global chunk blockIdx.x + c * gridDim.x.  STORE_BULK:
// results go through a staging buffer (NOUT operands) and cp.async.bulk s2g.
template <int KIND, int S, int CH, bool STORE_BULK>
__global__ void __launch_bounds__(512, 1) k_tma(int64_t n, double* __restrict__ r, double* __restrict__ q,
                                                double* __restrict__ x, double a, double b, double* parts) {
    constexpr int NOPS = KIND == 2 ? 2 : 3;
    constexpr int NOUT = KIND == 2 ? 1 : 2;
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ uint64_t bar[S];
    double* stage = reinterpret_cast<double*>(sm);                    // [S][NOPS][CH]
    double* outb = stage + (size_t)S * NOPS * CH;                      // [2][NOUT][CH]
    const int64_t nch = (n + CH - 1) / CH;
    const int64_t mine = blockIdx.x < nch ? (nch - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    if (threadIdx.x == 0) for (int s = 0; s < S; ++s) mb_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const uint64_t pol = pol_first();
    const double* src[3] = {r, q, x};
    auto issue = [&](int64_t k) {
        const int st = (int)(k % S);
        const int64_t c = blockIdx.x + k * gridDim.x;
        const int64_t r0 = c * CH, rows = ((int64_t)CH < n - r0 ? (int64_t)CH : n - r0);
        mb_expect(&bar[st], (uint32_t)(rows * 8 * NOPS));
        for (int o = 0; o < NOPS; ++o)
            g2s(stage + ((size_t)st * NOPS + o) * CH, src[o] + r0, (uint32_t)(rows * 8), &bar[st], pol);
    };
    if (threadIdx.x == 0)
        for (int k = 0; k < S - 1 && k < mine; ++k) issue(k);
    double part = 0;
    for (int64_t k = 0; k < mine; ++k) {
        if (threadIdx.x == 0 && k + S - 1 < mine) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); // stage read by the generic proxy
            issue(k + S - 1);
        }
        const int st = (int)(k % S);
        mb_wait(&bar[st], (uint32_t)((k / S) & 1));
        const int64_t c = blockIdx.x + k * gridDim.x;
        const int64_t r0 = c * CH;
        const int rows = (int)((int64_t)CH < n - r0 ? (int64_t)CH : n - r0);
        const double2* s0 = reinterpret_cast<const double2*>(stage + ((size_t)st * NOPS + 0) * CH);
        const double2* s1 = reinterpret_cast<const double2*>(stage + ((size_t)st * NOPS + 1) * CH);
        const double2* s2 = reinterpret_cast<const double2*>(stage + ((size_t)st * NOPS + 2) * CH);
        double2* o0 = reinterpret_cast<double2*>(outb + ((size_t)(k & 1) * NOUT + 0) * CH);
        double2* o1 = reinterpret_cast<double2*>(outb + ((size_t)(k & 1) * NOUT + 1) * CH);
        if (STORE_BULK && threadIdx.x == 0) bulk_wait_read<1>(); // staging buffer k&1 free again
        if (STORE_BULK) __syncthreads();
        for (int i = threadIdx.x; i < rows / 2; i += blockDim.x) {
            if (KIND == 2) {
                double2 rv = s0[i];
                const double2 av = s1[i];
                rv.x = __dadd_rn(rv.x, __dmul_rn(a, av.x));
                rv.y = __dadd_rn(rv.y, __dmul_rn(a, av.y));
                part = __dadd_rn(part, __dmul_rn(rv.x, rv.x));
                part = __dadd_rn(part, __dmul_rn(rv.y, rv.y));
                if (STORE_BULK) o0[i] = rv;
                else __stcs(reinterpret_cast<double2*>(r + r0) + i, rv);
            } else {
                const double2 rv = s0[i];
                double2 pv = s1[i], xv = s2[i];
                xv.x = __dadd_rn(xv.x, __dmul_rn(a, pv.x));
                xv.y = __dadd_rn(xv.y, __dmul_rn(a, pv.y));
                pv.x = __dadd_rn(rv.x, __dmul_rn(b, pv.x));
                pv.y = __dadd_rn(rv.y, __dmul_rn(b, pv.y));
                if (STORE_BULK) {
                    o0[i] = pv;
                    o1[i] = xv;
                } else {
                    __stcs(reinterpret_cast<double2*>(q + r0) + i, pv);
                    __stcs(reinterpret_cast<double2*>(x + r0) + i, xv);
                }
            }
        }
        __syncthreads(); // stage st fully consumed (and staging buffer written)
        if (STORE_BULK && threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (KIND == 2) {
                s2g(r + r0, o0, rows * 8);
            } else {
                s2g(q + r0, o0, rows * 8);
                s2g(x + r0, o1, rows * 8);
            }
            bulk_commit();
        }
    }
    if (STORE_BULK && threadIdx.x == 0) bulk_wait_all();
    if (KIND == 2) block_store_part(part, parts);
}

// K1-like producer: streams a large evict-first buffer (the matrix) and
// writes Ap ascending with default-policy stores, like K1's epilogue
__global__ void __launch_bounds__(256) k1_like(int64_t n, int64_t per_row, const double2* __restrict__ mat,
                                               double* __restrict__ Ap, double* out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double acc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 2; i += stride) {
        double2 a = make_double2(0, 0);
        for (int64_t k = 0; k < per_row; ++k) {
            const double2 v = __ldcs(mat + (i * per_row + k));
            a.x += v.x;
            a.y += v.y;
        }
        reinterpret_cast<double2*>(Ap)[i] = a;
        acc += a.x;
    }
    if (acc == 1234.5) *out = acc;
}

// K2 / K3 with a sweep direction (DESC: the grid walks from the top) and the
// store policy of the produced vector (KEEP: default stores, else evict-first)
template <bool DESC, bool KEEP>
__global__ void __launch_bounds__(256) k2_dir(int64_t n, double* __restrict__ r, const double* __restrict__ Ap,
                                              double na, double* parts) {
    const int64_t np = n / 2, stride = (int64_t)gridDim.x * blockDim.x;
    double part = 0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < np; t += stride) {
        const int64_t j = DESC ? np - 1 - t : t;
        double2 rv = __ldcs(reinterpret_cast<const double2*>(r) + j);
        const double2 av = __ldcs(reinterpret_cast<const double2*>(Ap) + j);
        rv.x = __dadd_rn(rv.x, __dmul_rn(na, av.x));
        rv.y = __dadd_rn(rv.y, __dmul_rn(na, av.y));
        if (KEEP) reinterpret_cast<double2*>(r)[j] = rv;
        else __stcs(reinterpret_cast<double2*>(r) + j, rv);
        part = __dadd_rn(part, __dmul_rn(rv.x, rv.x));
        part = __dadd_rn(part, __dmul_rn(rv.y, rv.y));
    }
    block_store_part(part, parts);
}

template <bool DESC, bool KEEP>
__global__ void __launch_bounds__(256) k3_dir(int64_t n, const double* __restrict__ r, double* __restrict__ p,
                                              double* __restrict__ x, double a, double b) {
    const int64_t np = n / 2, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < np; t += stride) {
        const int64_t j = DESC ? np - 1 - t : t;
        const double2 rv = __ldcs(reinterpret_cast<const double2*>(r) + j);
        double2 pv = __ldcs(reinterpret_cast<const double2*>(p) + j);
        double2 xv = __ldcs(reinterpret_cast<const double2*>(x) + j);
        xv.x = __dadd_rn(xv.x, __dmul_rn(a, pv.x));
        xv.y = __dadd_rn(xv.y, __dmul_rn(a, pv.y));
        pv.x = __dadd_rn(rv.x, __dmul_rn(b, pv.x));
        pv.y = __dadd_rn(rv.y, __dmul_rn(b, pv.y));
        __stcs(reinterpret_cast<double2*>(x) + j, xv);
        if (KEEP) reinterpret_cast<double2*>(p)[j] = pv;
        else __stcs(reinterpret_cast<double2*>(p) + j, pv);
    }
}

// ---------------------------------------------------------------- driver
template <typename L>
static float time_it(L&& launch, int reps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    std::vector<float> t;
    for (int i = 0; i < reps + 2; ++i) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (i >= 2) t.push_back(ms);
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : (int64_t)256 * 256 * 256;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *r, *q, *x, *parts, *flush;
    CK(cudaMalloc(&r, n * 8));
    CK(cudaMalloc(&q, n * 8));
    CK(cudaMalloc(&x, n * 8));
    CK(cudaMalloc(&parts, 1 << 20));
    const size_t fl = size_t(512) << 20;
    CK(cudaMalloc(&flush, fl));
    cudaMemset(r, 0, n * 8);
    cudaMemset(q, 0, n * 8);
    cudaMemset(x, 0, n * 8);
    const int reps = 15;
    auto fl_launch = [&] { cudaMemsetAsync(flush, 0, fl); };
    printf("n = %lld rows, %d SMs\n", (long long)n, sms);
    auto report = [&](const char* name, double bytes, auto&& launch) {
        // L2 flush before every timed launch: time flush+kernel minus flush
        const float tf = time_it(fl_launch, reps);
        const float tk = time_it([&] { fl_launch(); launch(); }, reps) - tf;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) { printf("%-28s error %s\n", name, cudaGetErrorString(e)); return; }
        printf("%-28s %8.2f us  %7.0f GB/s\n", name, tk * 1e3, bytes / (tk * 1e-3) / 1e9);
    };
    const double b2 = 24.0 * n, b3 = 40.0 * n;
    for (int bps : {4, 8}) {
        const int g = sms * bps;
        char nm[64];
        snprintf(nm, 64, "K2 reg U1 g=%d", g); report(nm, b2, [&] { k2_reg<1><<<g, 256>>>(n, r, q, -0.5, parts); });
        snprintf(nm, 64, "K2 reg U2 g=%d", g); report(nm, b2, [&] { k2_reg<2><<<g, 256>>>(n, r, q, -0.5, parts); });
        snprintf(nm, 64, "K2 reg U4 g=%d", g); report(nm, b2, [&] { k2_reg<4><<<g, 256>>>(n, r, q, -0.5, parts); });
        snprintf(nm, 64, "K3 reg U1 g=%d", g); report(nm, b3, [&] { k3_reg<1><<<g, 256>>>(n, r, q, x, 0.5, 0.25); });
        snprintf(nm, 64, "K3 reg U2 g=%d", g); report(nm, b3, [&] { k3_reg<2><<<g, 256>>>(n, r, q, x, 0.5, 0.25); });
        snprintf(nm, 64, "K3 reg U4 g=%d", g); report(nm, b3, [&] { k3_reg<4><<<g, 256>>>(n, r, q, x, 0.5, 0.25); });
    }
#define TMA(KIND, S, CH, SB, NAME, BYTES)                                                            \
    {                                                                                                \
        auto kern = k_tma<KIND, S, CH, SB>;                                                          \
        const int nops = KIND == 2 ? 2 : 3, nout = KIND == 2 ? 1 : 2;                                \
        const int smem = (S * nops + (SB ? 2 * nout : 0)) * CH * 8;                                  \
        if (smem <= 227 * 1024) {                                                                    \
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);           \
            for (int th : {256, 512}) {                                                              \
                char nm[64];                                                                         \
                snprintf(nm, 64, "%s S%d CH%d t%d", NAME, S, CH, th);                                \
                report(nm, BYTES, [&] { kern<<<sms, th, smem>>>(n, r, q, x, 0.5, 0.25, parts); });  \
            }                                                                                        \
        }                                                                                            \
    }
    TMA(2, 4, 2048, false, "K2 tma", b2)
    TMA(2, 6, 2048, false, "K2 tma", b2)
    TMA(2, 8, 1024, false, "K2 tma", b2)
    TMA(2, 3, 4096, false, "K2 tma", b2)
    TMA(2, 4, 2048, true, "K2 tmas", b2)
    TMA(2, 6, 1024, true, "K2 tmas", b2)
    TMA(3, 4, 1024, false, "K3 tma", b3)
    TMA(3, 4, 2048, false, "K3 tma", b3)
    TMA(3, 6, 1024, false, "K3 tma", b3)
    TMA(3, 3, 2048, true, "K3 tmas", b3)
    TMA(3, 4, 1024, true, "K3 tmas", b3)
    // copy-bandwidth reference: cudaMemcpy D2D of n doubles (reads n, writes n)
    report("memcpy d2d", 16.0 * n, [&] { cudaMemcpyAsync(x, r, n * 8, cudaMemcpyDeviceToDevice); });
    // ---- sequence K1-like -> K2 -> K3 with sweep directions: L2 reuse of the
    // vector the previous kernel wrote last (event-timed per kernel, no flush)
    {
        const int64_t per_row = 17; // ~270 B/row of matrix, as K1's 10 B/nnz x 27
        double2* mat;
        const size_t mb = (size_t)(n / 2) * per_row * 16;
        if (cudaMalloc(&mat, mb) == cudaSuccess) {
            cudaMemset(mat, 0, mb);
            double* Apv;
            cudaMalloc(&Apv, n * 8);
            cudaEvent_t ev[4];
            for (auto& e : ev) cudaEventCreate(&e);
            const int g = sms * 4;
            auto seqrun = [&](auto k2, auto k3, const char* name) {
                std::vector<float> t1, t2, t3;
                for (int it = 0; it < 12; ++it) {
                    cudaEventRecord(ev[0]);
                    k1_like<<<g, 256>>>(n, per_row, mat, Apv, parts);
                    cudaEventRecord(ev[1]);
                    k2<<<g, 256>>>(n, r, Apv, -0.5, parts);
                    cudaEventRecord(ev[2]);
                    k3<<<g, 256>>>(n, r, q, x, 0.5, 0.25);
                    cudaEventRecord(ev[3]);
                    cudaEventSynchronize(ev[3]);
                    float a, b, c;
                    cudaEventElapsedTime(&a, ev[0], ev[1]);
                    cudaEventElapsedTime(&b, ev[1], ev[2]);
                    cudaEventElapsedTime(&c, ev[2], ev[3]);
                    if (it >= 2) { t1.push_back(a); t2.push_back(b); t3.push_back(c); }
                }
                auto med = [](std::vector<float> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
                printf("seq %-22s K1like %7.1f us  K2 %6.1f us (%5.0f GB/s)  K3 %6.1f us (%5.0f GB/s)\n", name,
                       med(t1) * 1e3, med(t2) * 1e3, b2 / (med(t2) * 1e-3) / 1e9, med(t3) * 1e3,
                       b3 / (med(t3) * 1e-3) / 1e9);
            };
            seqrun(k2_dir<false, false>, k3_dir<false, false>, "asc/asc evict-first");
            seqrun(k2_dir<true, false>, k3_dir<false, false>, "desc/asc evict-first");
            seqrun(k2_dir<true, true>, k3_dir<false, false>, "desc(keep r)/asc");
            seqrun(k2_dir<false, true>, k3_dir<false, false>, "asc(keep r)/asc");
            seqrun(k2_dir<true, true>, k3_dir<true, false>, "desc(keep r)/desc");
            seqrun(k2_dir<false, true>, k3_dir<true, false>, "asc(keep r)/desc");
        }
    }
    return 0;
}
