// Read-only HBM stream ceiling on this GPU (context for the roofline):
// 128-bit loads (evict-first), several in flight per thread, grid = SMs x resident blocks.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o readbw scripts/readbw.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(256) read_kernel(const double2* __restrict__ a, size_t n4,
                                                   double* out) {
    double acc = 0.0;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n4; i += U * stride) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(a + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
    }
    for (; i < n4; i += stride) {
        double2 v = __ldcs(a + i);
        acc += v.x + v.y;
    }
    if (acc == 12345.678) *out = acc; // keep the loads
}

template <int U>
float run(const double2* a, size_t n4, double* out, int blocks) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 8; ++r) {
        cudaEventRecord(e0);
        read_kernel<U><<<blocks, 256>>>(a, n4, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    return best;
}

int main() {
    const size_t bytes = size_t(8) << 30; // 8 GiB
    double2* a;
    double* out;
    if (cudaMalloc(&a, bytes) != cudaSuccess) return 1;
    cudaMalloc(&out, 8);
    cudaMemset(a, 0, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t n4 = bytes / sizeof(double2);
    for (int bps : {4, 8, 16}) {
        const int blocks = sms * bps;
        printf("blocks %d: U1 %.0f  U2 %.0f  U4 %.0f  U8 %.0f GB/s\n", blocks,
               bytes / (run<1>(a, n4, out, blocks) * 1e6), bytes / (run<2>(a, n4, out, blocks) * 1e6),
               bytes / (run<4>(a, n4, out, blocks) * 1e6), bytes / (run<8>(a, n4, out, blocks) * 1e6));
    }
    return 0;
}
