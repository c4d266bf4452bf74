// Probe (tuning tool): does griddepcontrol.wait cover the grandparent of a
// programmatic chain?  kA (sleeps, then sets a flag) -> kB (triggers at
// once, never waits, exits) -> kC (griddepcontrol.wait, then reads the
// flag), each launched with programmatic stream serialisation on one
// stream, plainly and captured in a CUDA graph.  If kC ever reads the flag
// unset, a wait covers only the direct predecessor.  No kernel waits on
// another's memory (kA sleeps on the clock only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/pdl_t scripts/pdl_transitive.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__global__ void kA(volatile int* flag, unsigned long long ns, unsigned long long* t) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const unsigned long long t0 = now();
    while (now() - t0 < ns) {
    }
    *flag = 1;
    __threadfence();
    t[0] = now();
}
__global__ void kB(unsigned long long* t) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    t[1] = now();
}
__global__ void kC(volatile int* flag, int* seen, unsigned long long* t) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    t[2] = now();
    *seen = *flag;
}

template <typename K, typename... A>
void launch(K k, cudaStream_t s, A... a) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(32);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, a...);
}

int main() {
    int *flag, *seen;
    unsigned long long* t;
    cudaMalloc(&flag, 4);
    cudaMalloc(&seen, 4);
    cudaMalloc(&t, 24);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int graph = 0; graph < 2; ++graph) {
        int unset = 0, runs = 0;
        long long lag_min = 1LL << 62, lag_max = -(1LL << 62), bstart = 0;
        for (int rep = 0; rep < 50; ++rep) {
            cudaMemsetAsync(flag, 0, 4, s);
            cudaMemsetAsync(seen, -1, 4, s);
            cudaGraphExec_t ex = nullptr;
            if (graph) {
                cudaGraph_t g;
                cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
                launch(kA, s, (volatile int*)flag, 200000ull, t);
                launch(kB, s, t);
                launch(kC, s, (volatile int*)flag, seen, t);
                cudaStreamEndCapture(s, &g);
                cudaGraphInstantiate(&ex, g, 0);
                cudaGraphDestroy(g);
                cudaGraphLaunch(ex, s);
            } else {
                launch(kA, s, (volatile int*)flag, 200000ull, t);
                launch(kB, s, t);
                launch(kC, s, (volatile int*)flag, seen, t);
            }
            cudaError_t e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) {
                printf("error %s\n", cudaGetErrorString(e));
                return 1;
            }
            if (ex) cudaGraphExecDestroy(ex);
            int h = -1;
            unsigned long long ht[3];
            cudaMemcpy(&h, seen, 4, cudaMemcpyDeviceToHost);
            cudaMemcpy(ht, t, 24, cudaMemcpyDeviceToHost);
            ++runs;
            unset += h != 1;
            const long long lag = (long long)(ht[2] - ht[0]); // kC after kA's end
            lag_min = lag < lag_min ? lag : lag_min;
            lag_max = lag > lag_max ? lag : lag_max;
            bstart += (long long)(ht[0] - ht[1]); // kB's end before kA's end (> 0: B ran early)
        }
        printf("%s: %d runs, flag unset in kC after its wait: %d; kC - kA end %lld..%lld ns; "
               "kB ended before kA by %lld ns on average\n",
               graph ? "graph" : "stream", runs, unset, lag_min, lag_max, bstart / runs);
    }
    return 0;
}
