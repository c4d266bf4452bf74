// sm_100a builders of the sliced-ELL matrix (K0) and their helpers:
//   stencil_widths / stencil_fill   gen_stencil_matrix (csr.cpp:29-59) on the
//                                   device, rows in the reference's order
//   csr_widths / csr_fill           any CSR matrix (tw_ell_from_csr)
//   band                            min / max column of a row range
//                                   (make_tile_plan's band, cg.cpp:358-367)
//   scan_*                          int64 exclusive scan for slice offsets
// One warp per 32-row slice, lane = row; the chunked entry layout is the
// one tw_internal.h documents (ell_val_pos / ell_col_pos).
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "tw_device.cuh"
#include "tw_internal.h"

namespace tw {

namespace {

using namespace dev;

// --------------------------------------------------------------- K0 generator

__device__ __forceinline__ int64_t axis_span(int64_t c, int64_t d) {
    return 1 + (c > 0) + (c + 1 < d);
}

// Width of each 32-row slice = longest stencil row in it (closed form).
__global__ void stencil_widths_kernel(int64_t nx, int64_t ny, int64_t nz, int64_t row_offset,
                                      int64_t n_rows, int64_t n_slices, int64_t* widths) {
    const int lane = threadIdx.x & 31;
    const int64_t warp_g = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const int64_t plane = nx * ny;
    for (int64_t s = warp_g; s < n_slices; s += nwarps) {
        const int64_t row = s * 32 + lane;
        int len = 0;
        if (row < n_rows) {
            const int64_t g = row + row_offset;
            const int64_t z = g / plane, rem = g - z * plane, y = rem / nx, x = rem - y * nx;
            len = static_cast<int>(axis_span(x, nx) * axis_span(y, ny) * axis_span(z, nz));
        }
        const int w = __reduce_max_sync(0xffffffffu, len);
        if (lane == 0) widths[s] = 32LL * w;
    }
}

// One warp per slice, lane = row: walk the row's neighbours in the
// reference's (dz, dy, dx) order (csr.cpp:46-54) into registers, then write
// the slice block in its chunked layout with 128-bit stores -- 2 values, 4
// int32 columns or 8 x-staged 16-bit columns per lane and store, a warp
// writing 512 contiguous bytes -- padding to the slice width (value 0,
// column -1, staged 0xFFFF).  With c16 (nx % 32 == 0: each slice is one
// x-line segment starting at x0) the staged index of neighbour (dz, dy, cx)
// is run (dz + 1) * 3 + (dy + 1), offset cx - x0 + 2 (stage_run_start).
constexpr int kMaxStencilWidth = 27;
__global__ void __launch_bounds__(kThreads)
stencil_fill_kernel(int64_t nx, int64_t ny, int64_t nz, int64_t row_offset, int64_t col_offset,
                    int64_t n_rows, int64_t n_slices, const int64_t* __restrict__ slice_off,
                    double* vals, int32_t* cols, uint16_t* c16) {
    const int lane = threadIdx.x & 31;
    const int64_t warp_g = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const int64_t plane = nx * ny;
    for (int64_t s = warp_g; s < n_slices; s += nwarps) {
        const int64_t off = slice_off[s];
        const int w = static_cast<int>((slice_off[s + 1] - off) >> 5);
        const int64_t row = s * 32 + lane;
        const int64_t x0 = (s * 32 + row_offset) % nx;
        // entry k of the row is neighbour (iz, iy, ix) of its per-axis spans,
        // (dz, dy, dx) lexicographic = ascending column (csr.cpp:46-53)
        int len = 0, sx = 0, sxy = 0;
        int64_t x = 0, y = 0, z = 0, xlo = 0, ylo = 0, zlo = 0;
        if (row < n_rows) {
            const int64_t g = row + row_offset;
            z = g / plane;
            const int64_t rem = g - z * plane;
            y = rem / nx;
            x = rem - y * nx;
            xlo = x > 0 ? x - 1 : x;
            ylo = y > 0 ? y - 1 : y;
            zlo = z > 0 ? z - 1 : z;
            sx = static_cast<int>(axis_span(x, nx));
            sxy = sx * static_cast<int>(axis_span(y, ny));
            len = sxy * static_cast<int>(axis_span(z, nz));
        }
        // Interior slices (every row a full 27-point row, the bulk of any
        // large grid) take a body whose spans are compile-time constants, so
        // the neighbour decode of each unrolled entry folds to constants.
        const bool full = w == kMaxStencilWidth && __all_sync(0xffffffffu, len == kMaxStencilWidth);
        auto body = [&](auto full_tag) {
        constexpr bool F = decltype(full_tag)::value;
        const int SX = F ? 3 : sx, SXY = F ? 9 : sxy, LEN = F ? kMaxStencilWidth : len;
        auto nb = [&](int k, int64_t& cx, int64_t& cy, int64_t& cz) {
            const int iz = k / SXY, t = k - iz * SXY, iy = t / SX;
            cz = zlo + iz;
            cy = ylo + iy;
            cx = xlo + (t - iy * sx);
        };
        auto val = [&](int k) {
            if (F) return k == 13 ? 27.0 : -1.0;
            if (k >= LEN) return 0.0;
            int64_t cx, cy, cz;
            nb(k, cx, cy, cz);
            return cx == x && cy == y && cz == z ? 27.0 : -1.0;
        };
        auto cl = [&](int k) {
            if (F) // (z + dz, y + dy, x + dx) = row + dz * plane + dy * nx + dx
                return static_cast<int32_t>(row + row_offset - col_offset + (k / 9 - 1) * plane +
                                            ((k % 9) / 3 - 1) * nx + (k % 3 - 1));
            if (k >= LEN) return -1;
            int64_t cx, cy, cz;
            nb(k, cx, cy, cz);
            return static_cast<int32_t>((cz * ny + cy) * nx + cx - col_offset);
        };
        auto s16 = [&](int k) {
            if (F) // run (dz + 1) * 3 + (dy + 1), offset x + dx - x0 + 2
                return static_cast<uint32_t>((k / 3) * kStageRunLen + (k % 3) + 1 + (x - x0));
            if (k >= LEN) return uint32_t(kStagePad);
            int64_t cx, cy, cz;
            nb(k, cx, cy, cz);
            TW_DCHECK(cx - x0 + 2 >= 0 && cx - x0 + 2 < kStageRunLen);
            return static_cast<uint32_t>(((cz - z + 1) * 3 + (cy - y + 1)) * kStageRunLen +
                                         (cx - x0 + 2));
        };
        double* vb = vals + off;
        int32_t* cb = cols + off;
        // values: pairs [k/2][l][2] (one double2 per lane), odd tail [w-1][l]
#pragma unroll
        for (int j = 0; j < kMaxStencilWidth / 2; ++j)
            if (2 * j + 1 < w)
                __stcs(reinterpret_cast<double2*>(vb + 64 * j) + lane,
                       make_double2(val(2 * j), val(2 * j + 1)));
        if (w & 1) vb[32 * (w - 1) + lane] = val(w - 1);
        // int32 columns: quads [k/4][l][4], then a pair, then a single
        const int f4 = w & ~3;
#pragma unroll
        for (int q = 0; q < kMaxStencilWidth / 4; ++q)
            if (4 * q < f4)
                __stcs(reinterpret_cast<int4*>(cb + 128 * q) + lane,
                       make_int4(cl(4 * q), cl(4 * q + 1), cl(4 * q + 2), cl(4 * q + 3)));
        if (w - f4 >= 2)
            reinterpret_cast<int2*>(cb + 32 * f4)[lane] = make_int2(cl(f4), cl(f4 + 1));
        if ((w - f4) & 1) cb[32 * (w - 1) + lane] = cl(w - 1);
        if (!c16) return;
        // staged columns: [k/8][l][8] (one uint4 per lane), then 4, 2, 1
        uint16_t* hb = c16 + off;
        const int f8 = w & ~7;
        auto pk = [&](int k) { return s16(k) | (s16(k + 1) << 16); };
#pragma unroll
        for (int q = 0; q < kMaxStencilWidth / 8; ++q)
            if (8 * q < f8)
                __stcs(reinterpret_cast<uint4*>(hb + 256 * q) + lane,
                       make_uint4(pk(8 * q), pk(8 * q + 2), pk(8 * q + 4), pk(8 * q + 6)));
        int base = f8, rem = w - f8;
        if (rem >= 4) {
            reinterpret_cast<uint2*>(hb + 32 * base)[lane] = make_uint2(pk(base), pk(base + 2));
            base += 4;
            rem -= 4;
        }
        if (rem >= 2) {
            reinterpret_cast<uint32_t*>(hb + 32 * base)[lane] = pk(base);
            base += 2;
            rem -= 2;
        }
        if (rem) hb[32 * base + lane] = static_cast<uint16_t>(s16(base));
        };
        if (full)
            body(std::true_type{});
        else
            body(std::false_type{});
    }
}

__global__ void csr_widths_kernel(const int64_t* __restrict__ row_ptr, int64_t n_rows,
                                  int64_t n_slices, int64_t* widths) {
    const int lane = threadIdx.x & 31;
    const int64_t warp_g = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t s = warp_g; s < n_slices; s += nwarps) {
        const int64_t row = s * 32 + lane;
        unsigned len = row < n_rows ? static_cast<unsigned>(row_ptr[row + 1] - row_ptr[row]) : 0u;
        const unsigned w = __reduce_max_sync(0xffffffffu, len);
        if (lane == 0) widths[s] = 32LL * w;
    }
}

__global__ void csr_fill_kernel(const int64_t* __restrict__ row_ptr,
                                const int64_t* __restrict__ col_idx,
                                const double* __restrict__ values, int64_t n_rows,
                                int64_t n_slices, const int64_t* __restrict__ slice_off,
                                double* vals, int32_t* cols) {
    const int lane = threadIdx.x & 31;
    const int64_t warp_g = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t s = warp_g; s < n_slices; s += nwarps) {
        const int64_t off = slice_off[s];
        const int w = static_cast<int>((slice_off[s + 1] - off) >> 5);
        const int64_t row = s * 32 + lane;
        int k = 0;
        if (row < n_rows) {
            for (int64_t e = row_ptr[row]; e < row_ptr[row + 1]; ++e, ++k) {
                vals[off + ell_val_pos(k, lane, w)] = values[e];
                cols[off + ell_col_pos(k, lane, w)] = static_cast<int32_t>(col_idx[e]);
            }
        }
        for (; k < w; ++k) {
            vals[off + ell_val_pos(k, lane, w)] = 0.0;
            cols[off + ell_col_pos(k, lane, w)] = -1;
        }
    }
}

// Per-tile column band (make_tile_plan, cg.cpp:358-367): min and max local
// column over the rows [r0, r1), packed as atomics on 64-bit slots.
__global__ void band_kernel(EllView A, int64_t r0, int64_t r1, unsigned long long* minmax) {
    const int lane = threadIdx.x & 31;
    const int64_t warp_g = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const int64_t s0 = r0 >> 5, s1 = (r1 + 31) >> 5;
    long long lo = 0x7fffffffffffffffLL, hi = -1;
    for (int64_t s = s0 + warp_g; s < s1; s += nwarps) {
        const int64_t off = A.slice_off[s];
        const int w = static_cast<int>((A.slice_off[s + 1] - off) >> 5);
        const int64_t row = s * 32 + lane;
        if (row < r0 || row >= r1) continue;
        for (int k = 0; k < w; ++k) {
            const int c = A.cols[off + ell_col_pos(k, lane, w)];
            if (c < 0) break;
            lo = c < lo ? c : lo;
            hi = c > hi ? c : hi;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        long long l2 = __shfl_xor_sync(0xffffffffu, lo, o), h2 = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = l2 < lo ? l2 : lo;
        hi = h2 > hi ? h2 : hi;
    }
    if (lane == 0 && hi >= 0) {
        atomicMin(minmax, static_cast<unsigned long long>(lo));
        atomicMax(minmax + 1, static_cast<unsigned long long>(hi));
    }
}

// ------------------------------------------------------------------- scan
// Three-phase exclusive scan of int64 (slice offsets): per-block sums, one
// block scanning the block sums, per-block rescan with the carried base.
constexpr int kScanItems = 8; // per thread
constexpr int kScanTile = kThreads * kScanItems;

__device__ int64_t block_exclusive_scan(int64_t v, int64_t* smem, int64_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) smem[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        int64_t w = lane < (kThreads >> 5) ? smem[lane] : 0;
        int64_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < (kThreads >> 5)) smem[lane] = wi - w;
        if (lane == (kThreads >> 5) - 1) smem[32] = wi;
    }
    __syncthreads();
    int64_t excl = smem[warp] + inc - v;
    *total = smem[32];
    __syncthreads();
    return excl;
}

__global__ void scan_sums_kernel(const int64_t* in, int64_t n, int64_t* sums) {
    __shared__ int64_t smem[33];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    int64_t v = 0;
    for (int j = 0; j < kScanItems; ++j)
        if (base + j < n) v += in[base + j];
    int64_t total;
    block_exclusive_scan(v, smem, &total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void scan_top_kernel(int64_t* sums, int64_t nb) {
    __shared__ int64_t smem[33];
    int64_t carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += kThreads) {
        const int64_t i = b0 + threadIdx.x;
        int64_t v = i < nb ? sums[i] : 0;
        int64_t total;
        int64_t e = block_exclusive_scan(v, smem, &total);
        if (i < nb) sums[i] = e + carry;
        carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) sums[nb] = carry;
}

__global__ void scan_apply_kernel(const int64_t* in, int64_t n, const int64_t* sums,
                                  int64_t* out) {
    __shared__ int64_t smem[33];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    int64_t loc[kScanItems];
    int64_t v = 0;
    for (int j = 0; j < kScanItems; ++j) {
        loc[j] = base + j < n ? in[base + j] : 0;
        v += loc[j];
    }
    int64_t total;
    int64_t e = block_exclusive_scan(v, smem, &total) + sums[blockIdx.x];
    for (int j = 0; j < kScanItems; ++j) {
        if (base + j < n) out[base + j] = e;
        e += loc[j];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = sums[gridDim.x];
}

// 16-bit staged columns (ell_c16_pos layout) from the 32-bit ones: column c
// of a row in slice s maps to run r (its (dz, dy) line) at c - start(r).
// Slab matrices work in global coordinates: local row + sx_row_off, local
// column + sx_col_off.
__global__ void stencil_cols16_kernel(EllView A, uint16_t* cols16, unsigned* bad) {
    const int lane = threadIdx.x & 31;
    const int64_t warp_g = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const int64_t nx = A.sx_nx, ny = A.sx_ny, nz = A.sx_nz, plane = nx * ny;
    for (int64_t s = warp_g; s < A.n_slices; s += nwarps) {
        const int64_t off = A.slice_off[s];
        const int w = static_cast<int>((A.slice_off[s + 1] - off) >> 5);
        const int64_t row0 = s * 32 + A.sx_row_off, z0 = row0 / plane, y0 = (row0 / nx) % ny;
        for (int k = 0; k < w; ++k) {
            const int c = A.cols[off + ell_col_pos(k, lane, w)];
            uint16_t v = kStagePad;
            if (c >= 0) {
                const int64_t cg = c + A.sx_col_off;
                const int64_t dz = cg / plane - z0, dy = (cg / nx) % ny - y0;
                const int r = static_cast<int>((dz + 1) * 3 + (dy + 1));
                const int64_t o =
                    (dz < -1 || dz > 1 || dy < -1 || dy > 1)
                        ? -1
                        : c - stage_run_start(s, r, nx, ny, nz, A.sx_row_off, A.sx_col_off);
                if (o < 0 || o >= kStageRunLen) atomicOr(bad, 1u);
                else v = static_cast<uint16_t>(r * kStageRunLen + o);
            }
            cols16[off + ell_c16_pos(k, lane, w)] = v;
        }
    }
}

// Run table + 16-bit columns of a general matrix (tw_ell_from_csr), one warp
// per slice, lane = row.  Run 4 is the window of the slice's own rows
// ([row0 - 2, row0 + 34) in x: K1's p.Ap reads p[row] from it); the other 8
// runs cover the remaining columns greedily: each starts at the smallest
// column not yet covered (rounded down to the 16-byte grid of x) and takes
// every column below its end.  A column maps to the first run covering it.
// Slices whose columns need more than 9 runs flag *bad.
__global__ void csr_runs_kernel(EllView A, int32_t* runs, uint16_t* cols16, unsigned* bad) {
    constexpr int64_t kNone = INT64_MAX;
    const int lane = threadIdx.x & 31;
    const int64_t warp_g = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t s = warp_g; s < A.n_slices; s += nwarps) {
        const int64_t off = A.slice_off[s];
        const int w = static_cast<int>((A.slice_off[s + 1] - off) >> 5);
        const int64_t own = s * 32 + A.diag_shift - 2;
        auto col = [&](int k) -> int64_t {
            if (k >= w) return kNone;
            const int c = A.cols[off + ell_col_pos(k, lane, w)];
            return c < 0 ? kNone : c;
        };
        auto in_own = [&](int64_t c) { return c >= own && c < own + kStageRunLen; };
        int64_t start[kStageRuns];
        int k = 0; // this lane's next column not yet covered
        auto skip = [&](int64_t end) {
            for (int64_t c = col(k); c != kNone && (c < end || in_own(c)); c = col(++k)) {
            }
        };
        skip(INT64_MIN); // the columns inside run 4 only
        for (int r = 0; r < kStageRuns; ++r) {
            if (r == 4) {
                start[r] = own;
                continue;
            }
            int64_t m = col(k);
            for (int o = 16; o; o >>= 1) {
                const int64_t t = __shfl_xor_sync(0xffffffffu, m, o);
                m = t < m ? t : m;
            }
            if (m == kNone) {
                start[r] = own; // unused: any in-bounds window
                continue;
            }
            start[r] = m - ((m - A.diag_shift) & 1);
            skip(start[r] + kStageRunLen);
        }
        if (col(k) != kNone) atomicOr(bad, 1u);
        if (lane < kStageRuns) {
            TW_DCHECK(start[lane < kStageRuns ? lane : 0] >= -2);
            int64_t v = start[0];
            for (int r = 1; r < kStageRuns; ++r)
                if (lane == r) v = start[r];
            runs[s * kStageRuns + lane] = static_cast<int32_t>(v);
        }
        for (int e = 0; e < w; ++e) {
            const int64_t c = col(e);
            uint16_t v = kStagePad;
            if (c != kNone) {
                int rr = -1;
                if (in_own(c)) rr = 4;
                for (int r = 0; r < kStageRuns && rr < 0; ++r)
                    if (c >= start[r] && c < start[r] + kStageRunLen) rr = r;
                if (rr >= 0) v = static_cast<uint16_t>(rr * kStageRunLen + (c - start[rr]));
            }
            cols16[off + ell_c16_pos(e, lane, w)] = v;
        }
    }
}

#ifdef TW_CHECKS
// Checked build: one warp per slice, lane = row.
__global__ void ell_check_kernel(EllView A) {
    const int lane = threadIdx.x & 31;
    const int64_t warp_g = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t s = warp_g; s < A.n_slices; s += nwarps) {
        const int64_t off = A.slice_off[s], ents = A.slice_off[s + 1] - off;
        TW_DCHECK(ents >= 0 && ents % 32 == 0 && ents / 32 <= A.max_width);
        const int w = static_cast<int>(ents / 32);
        bool pad = false;
        for (int k = 0; k < w; ++k) {
            const int c = A.cols[off + ell_col_pos(k, lane, w)];
            TW_DCHECK(c >= -1 && c < A.x_len);
            if (c < 0) pad = true;
            else TW_DCHECK(!pad); // padding only ever trails a row
        }
    }
}
#endif

} // namespace

void launch_csr_runs(const EllView& A, int32_t* runs, uint16_t* cols16, unsigned* bad,
                     cudaStream_t s) {
    csr_runs_kernel<<<clamp_blocks(A.n_slices * 32, 4096), kThreads, 0, s>>>(A, runs, cols16, bad);
    TW_CUDA(cudaGetLastError());
}

void launch_stencil_cols16(const EllView& A, uint16_t* cols16, unsigned* bad, cudaStream_t s) {
    stencil_cols16_kernel<<<clamp_blocks(A.n_slices * 32, 4096), kThreads, 0, s>>>(A, cols16, bad);
    TW_CUDA(cudaGetLastError());
}

#ifdef TW_CHECKS
void launch_ell_check(const EllView& A, cudaStream_t s) {
    ell_check_kernel<<<clamp_blocks(A.n_slices * 32, 1024), kThreads, 0, s>>>(A);
    TW_CUDA(cudaGetLastError());
}
#endif

void launch_stencil_widths(int64_t nx, int64_t ny, int64_t nz, int64_t row_offset,
                           int64_t n_rows, int64_t n_slices, int64_t* widths_out, int blocks,
                           cudaStream_t s) {
    stencil_widths_kernel<<<clamp_blocks(n_slices * 32, blocks), kThreads, 0, s>>>(
        nx, ny, nz, row_offset, n_rows, n_slices, widths_out);
    TW_CUDA(cudaGetLastError());
}

void launch_stencil_fill(int64_t nx, int64_t ny, int64_t nz, int64_t row_offset,
                         int64_t col_offset, int64_t n_rows, int64_t n_slices,
                         const int64_t* slice_off, double* vals, int32_t* cols, uint16_t* c16,
                         int blocks, cudaStream_t s) {
    stencil_fill_kernel<<<clamp_blocks(n_slices * 32, blocks), kThreads, 0, s>>>(
        nx, ny, nz, row_offset, col_offset, n_rows, n_slices, slice_off, vals, cols, c16);
    TW_CUDA(cudaGetLastError());
}

void launch_csr_widths(const int64_t* row_ptr, int64_t n_rows, int64_t n_slices,
                       int64_t* widths_out, int blocks, cudaStream_t s) {
    csr_widths_kernel<<<clamp_blocks(n_slices * 32, blocks), kThreads, 0, s>>>(
        row_ptr, n_rows, n_slices, widths_out);
    TW_CUDA(cudaGetLastError());
}

void launch_csr_fill(const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                     int64_t n_rows, int64_t n_slices, const int64_t* slice_off, double* vals,
                     int32_t* cols, int blocks, cudaStream_t s) {
    csr_fill_kernel<<<clamp_blocks(n_slices * 32, blocks), kThreads, 0, s>>>(
        row_ptr, col_idx, values, n_rows, n_slices, slice_off, vals, cols);
    TW_CUDA(cudaGetLastError());
}

int64_t scan_tmp_elems(int64_t n) { return (n + kScanTile - 1) / kScanTile + 1; }

void scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* tmp,
                        cudaStream_t s) {
    const int64_t nb = (n + kScanTile - 1) / kScanTile;
    if (nb == 0) {
        TW_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
        return;
    }
    scan_sums_kernel<<<static_cast<unsigned>(nb), kThreads, 0, s>>>(in, n, tmp);
    scan_top_kernel<<<1, kThreads, 0, s>>>(tmp, nb);
    scan_apply_kernel<<<static_cast<unsigned>(nb), kThreads, 0, s>>>(in, n, tmp, out);
    TW_CUDA(cudaGetLastError());
}

void launch_band(const EllView& A, int64_t r0, int64_t r1, unsigned long long* minmax, int blocks,
                 cudaStream_t s) {
    const int64_t ns = ((r1 + 31) >> 5) - (r0 >> 5);
    band_kernel<<<clamp_blocks(ns * 32, blocks), kThreads, 0, s>>>(A, r0, r1, minmax);
    TW_CUDA(cudaGetLastError());
}

} // namespace tw
