// NVLink peer-memory transport of the multi-rank CG iteration.
//
// Replaces the NCCL halo and the two NCCL allgathers inside the iteration,
// fused into the compute kernels (tw_kernels.cu, helpers in tw_device.cuh):
//   * K3 (update_p) stores the rank's first / last owned plane of p straight
//     into the neighbours' ghost planes (the fused halo); its last block
//     raises the neighbours' ghost flags;
//   * the boundary SpMV (K1b) and K2 finish with FIN_PUBLISH_A / _B: the last
//     block stores this rank's p.Ap / r.r partial into every rank's receive
//     slot [rank] and raises flag [rank] there;
//   * K1b, K2 and K3 start with block_wait_flags: acquire-spin until the
//     flags they consume carry this iteration's stamp.
// This file holds the stand-alone kernels: the initial ghost push of a solve
// (p = b before iteration 0) and the transport check (ping send / check).
// Flags hold stamps (solve epoch << 32 | iteration + 1), so they never need
// resetting.  Peer pointers come from CUDA IPC (one process per GPU) or are
// plain device pointers (the emulated rank group on one GPU, where the host
// sequences the phases so every flag is already set when it is checked).
#include <cuda_runtime.h>

#include <cstdint>

#include "tw_device.cuh"
#include "tw_internal.h"

namespace tw {

namespace {

using namespace dev;

// Initial ghost planes of a solve (p = b): push this rank's boundary planes
// into the neighbours' ghosts and raise their flags for iteration 0.
__global__ void peer_push_kernel(const double* p_owned, int64_t n, int64_t plane, PeerLinks L,
                                 const CgScalars* sc, unsigned* ticket) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < plane;
         i += stride) {
        if (L.ghost_lo_dst) L.ghost_lo_dst[i] = p_owned[i];
        if (L.ghost_hi_dst) L.ghost_hi_dst[i] = p_owned[n - plane + i];
    }
    __threadfence_system();
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) last = atomicInc(ticket, gridDim.x - 1) == gridDim.x - 1;
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence_system();
        const unsigned long long st = stamp_of(sc, 0);
        if (L.ghost_lo_flag) st_release_sys(L.ghost_lo_flag, st);
        if (L.ghost_hi_flag) st_release_sys(L.ghost_hi_flag, st);
    }
}

__global__ void peer_ping_send_kernel(PeerLinks L, unsigned long long token) {
    for (int q = threadIdx.x; q < L.nranks; q += blockDim.x) st_release_sys(L.win[q]->ping + L.rank, token);
}

// Bounded wait that reports instead of trapping: the caller falls back to
// another transport when a peer's store never becomes visible.
__global__ void peer_ping_check_kernel(const PeerWindow* win, int nranks, unsigned long long token,
                                       long long timeout_ns, int* ok) {
    __shared__ int good;
    if (threadIdx.x == 0) good = 1;
    __syncthreads();
    const unsigned long long t0 = global_ns();
    for (int q = threadIdx.x; q < nranks; q += blockDim.x) {
        while (ld_acquire_sys(win->ping + q) != token) {
            if (static_cast<long long>(global_ns() - t0) > timeout_ns) {
                atomicAnd(&good, 0);
                break;
            }
            __nanosleep(256);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) *ok = good;
}

} // namespace

void launch_peer_ping_send(const PeerLinks& L, unsigned long long token, cudaStream_t s) {
    peer_ping_send_kernel<<<1, 64, 0, s>>>(L, token);
    TW_CUDA(cudaGetLastError());
}

void launch_peer_ping_check(const PeerWindow* win, int nranks, unsigned long long token,
                            long long timeout_ns, int* ok, cudaStream_t s) {
    peer_ping_check_kernel<<<1, 64, 0, s>>>(win, nranks, token, timeout_ns, ok);
    TW_CUDA(cudaGetLastError());
}

void launch_peer_push(const double* p_owned, int64_t n, int64_t plane, const PeerLinks& L,
                      const CgScalars* sc, unsigned* ticket, cudaStream_t s) {
    int g = static_cast<int>((plane + 255) / 256);
    if (g < 1) g = 1;
    if (g > 1024) g = 1024;
    peer_push_kernel<<<g, 256, 0, s>>>(p_owned, n, plane, L, sc, ticket);
    TW_CUDA(cudaGetLastError());
}

} // namespace tw
