// Internal declarations shared by the libtw_hpccg translation units.
// Public C ABI: include/tw_hpccg.h.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "tw_hpccg.h"
#include "tw_hpccg_emulation.h"

namespace tw {

// Where a tile kernel waits for the grids before it and where it lets the
// next one launch (programmatic dependent launch; tw_device.cuh
// pdl_role_entry / pdl_role_exit).  PDL_DEFAULT: trigger at entry, wait
// before the inputs -- the monolithic chain's K1 and every plain launch.
enum PdlRole : int {
    PDL_DEFAULT = 0,
    PDL_GATE = 1,      // a phase's first tile: wait, then trigger
    PDL_INNER = 2,     // a later tile: trigger at entry, no wait (its gate waited)
    PDL_LAST = 3,      // the phase's last tile: no wait, trigger after the main loop
    PDL_GATE_LAST = 4, // the phase's only tile: wait, trigger after the main loop
};

// Exceptions mapped 1:1 onto the ABI status codes at the extern "C" boundary
// (mirrors the reference's ConfigError / ContractViolation, types.hpp:23-33).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void config_error(const std::string& m) { throw Error(TW_ERR_CONFIG, m); }
[[noreturn]] inline void contract_error(const std::string& m) { throw Error(TW_ERR_CONTRACT, m); }
void cuda_check(cudaError_t e, const char* what, const char* file, int line);
#define TW_CUDA(x) ::tw::cuda_check((x), #x, __FILE__, __LINE__)

constexpr int kSliceRows = 32; // one warp per slice: lane = row within slice

// ---------------------------------------------------------------- device views

// Sliced ELL, 32-row slices.  Slice s stores its rows' entries in a block of
// 32*w entries starting at slice_off[s] (w = slice width = longest row).
// Inside a block entry k of lane l sits at a chunked position chosen so one
// 128-bit load gives a lane several consecutive entries of ITS row:
//   values  (f64): pairs  [k/2][l][2], odd tail k=w-1 at [w-1][l]
//   columns (i32): quads  [k/4][l][4], then a pair, then a single for w%4
// Rows keep the reference's entry order (csr.cpp:46-53); padding entries
// (k >= row length) carry col = -1 and are skipped, never accumulated.
struct EllView {
    const int64_t* slice_off; // [n_slices + 1], in entries
    const double* vals;
    const int32_t* cols;      // local column = global column - col_offset
    int64_t n_rows;
    int64_t n_slices;
    int64_t diag_shift;       // x index of local row i is i + diag_shift
    int max_width;            // widest slice (sizes the TMA stages)
    int tma_blocks;           // persistent grid of the TMA SpMV (0 = plain kernel)
    int64_t x_len;            // entries of the gathered vector (owned + ghost planes)
    // x-staged form (stencil or z-slab of one, nx % 32 == 0; null otherwise):
    // every stored column as a 16-bit index into the slice's staged window of
    // x -- 9 runs of 36 doubles, one per (dz, dy) neighbour line -- in the
    // chunked layout of ell_c16_pos; sx_* is the global grid the runs come
    // from and the slab's global row / column offsets
    const uint16_t* cols16 = nullptr;
    int64_t sx_nx = 0, sx_ny = 0, sx_nz = 0;
    int64_t sx_row_off = 0, sx_col_off = 0;
    // stage the x runs with an L2 evict_last hint (x up to 8M entries: it
    // then stays in L2 across the iteration; measured 128^3 K1 -2.4 %,
    // neutral at 256^3, profiles/r01_ab_k1_k2_k3_variants.md)
    int sx_keep = 0;
    // run-table form (a CSR matrix whose slices' columns fall into at most 9
    // windows of 36 doubles, tw_ell_from_csr): the run starts per slice,
    // int32[n_slices * 9], run 4 = the slice's own rows' window; null for
    // the closed-form runs of a stencil (sx_* above)
    const int32_t* sx_runs = nullptr;
};

// x-staged windows: run r = (dz + 1) * 3 + (dy + 1) of a slice starts 2
// doubles before the slice's x0 on line (z + dz, y + dy) and holds 36.
constexpr int kStageRuns = 9, kStageRunLen = 36;
constexpr uint16_t kStagePad = 0xFFFF;

// Position of entry k of lane l in a slice block of 16-bit columns: blocks of
// 8 per lane (one 128-bit load), then 4, then 2, then 1.
__host__ __device__ inline int64_t ell_c16_pos(int k, int lane, int w) {
    const int f8 = w & ~7;
    if (k < f8) return 32LL * (k & ~7) + 8 * lane + (k & 7);
    int base = f8, rem = w - f8;
    if (rem >= 4) {
        if (k < base + 4) return 32LL * base + 4 * lane + (k - base);
        base += 4;
        rem -= 4;
    }
    if (rem >= 2) {
        if (k < base + 2) return 32LL * base + 2 * lane + (k - base);
        base += 2;
    }
    return 32LL * base + lane;
}

// Start (in local x indices) of staged run r of slice s of an x-staged
// matrix whose local row 0 is global row row_off and local column 0 global
// column col_off; a neighbour line outside the global grid stages the
// slice's own line instead (no stored column refers to it).  A slab's
// neighbour lines in the planes next to it are its ghost planes.
__host__ __device__ inline int64_t stage_run_start(int64_t s, int r, int64_t nx, int64_t ny,
                                                   int64_t nz, int64_t row_off = 0,
                                                   int64_t col_off = 0) {
    const int64_t row0 = s * 32 + row_off, x0 = row0 % nx, t = row0 / nx, y = t % ny, z = t / ny;
    const int64_t zz = z + r / 3 - 1, yy = y + r % 3 - 1;
    const bool in = zz >= 0 && zz < nz && yy >= 0 && yy < ny;
    return (in ? zz * ny + yy : z * ny + y) * nx + x0 - 2 - col_off;
}

// Starts of the 9 staged runs of slice s, from the run table or the closed
// form (its divisions done once per slice, not per run: lane 0 computes
// them on K1's issue path, between one slice's copies and the next).
__host__ __device__ inline void run_starts(const EllView& A, int64_t s, int64_t st[kStageRuns]) {
    if (A.sx_runs) {
        for (int r = 0; r < kStageRuns; ++r) st[r] = A.sx_runs[s * kStageRuns + r];
        return;
    }
    const int64_t nx = A.sx_nx, ny = A.sx_ny, nz = A.sx_nz;
    const int64_t row0 = s * 32 + A.sx_row_off, x0 = row0 % nx, t = row0 / nx, y = t % ny,
                  z = t / ny;
    const int64_t own = (z * ny + y) * nx + x0 - 2 - A.sx_col_off;
    for (int r = 0; r < kStageRuns; ++r) {
        const int64_t dz = r / 3 - 1, dy = r % 3 - 1;
        const bool in = z + dz >= 0 && z + dz < nz && y + dy >= 0 && y + dy < ny;
        st[r] = in ? own + (dz * ny + dy) * nx : own;
    }
}

__host__ __device__ inline int64_t ell_val_pos(int k, int lane, int w) {
    const int full = w & ~1;
    if (k < full) return 32LL * (k & ~1) + 2 * lane + (k & 1);
    return 32LL * (w - 1) + lane;
}
__host__ __device__ inline int64_t ell_col_pos(int k, int lane, int w) {
    const int full = w & ~3;
    if (k < full) return 32LL * (k & ~3) + 4 * lane + (k & 3);
    const int rem = w - full;
    if (rem >= 2 && k < full + 2) return 32LL * full + 2 * lane + (k - full);
    return 32LL * (w - 1) + lane;
}

// Scalar state of one solve, resident on the device (never round-trips to
// the host inside the iteration loop).
struct CgScalars {
    double rtrans; // r.r of the current residual
    double alpha;
    double beta;
    double pAp;
    double rr;
    int iter;      // iterations completed (index into history)
    int history_cap;
    unsigned epoch; // solve number (set_rhs count): high half of the peer flag stamps
    unsigned pad_;
    double alpha_prev; // the previous iteration's alpha (FIN_ALPHA keeps it: paired x update)
};

// ------------------------------------------------- NVLink peer transport

constexpr int kMaxRanks = 64;

// Per-rank receive window in device memory; peers store into it over NVLink.
struct PeerWindow {
    double recv_a[kMaxRanks];               // p.Ap partial of rank q
    double recv_b[kMaxRanks];               // r.r partial of rank q
    unsigned long long flag_a[kMaxRanks];   // stamp of recv_a[q]
    unsigned long long flag_b[kMaxRanks];   // stamp of recv_b[q]
    unsigned long long flag_ghost_lo;       // my lower ghost plane holds rank-1's data
    unsigned long long flag_ghost_hi;       // my upper ghost plane holds rank+1's data
    unsigned long long ping[kMaxRanks];     // transport check: token from rank q
};

// Where this rank's data goes (device pointers: own, IPC-mapped or, for the
// emulated group, other ranks' buffers on the same device).
struct PeerLinks {
    int rank, nranks;
    PeerWindow* win[kMaxRanks];         // every rank's window (own included)
    double* ghost_lo_dst;               // rank-1's upper ghost plane <- my first plane
    double* ghost_hi_dst;               // rank+1's lower ghost plane <- my last plane
    unsigned long long* ghost_lo_flag;  // rank-1's flag_ghost_hi
    unsigned long long* ghost_hi_flag;  // rank+1's flag_ghost_lo
    int64_t plane;
};

// Scratch for fixed-order grid reductions: one partial per block plus a
// wrap-around ticket so the last block to finish combines them.
struct RedScratch {
    double* block_part;
    unsigned* ticket;
};

enum FinMode : int {
    FIN_NONE = 0,
    FIN_STORE = 1, // *out = total
    FIN_ALPHA = 2, // pAp = total; alpha = rtrans / pAp
    FIN_BETA = 3,  // rr = total; beta = rr / rtrans; rtrans = rr; history[iter++] = sqrt(rr)
    FIN_RTRANS = 4, // rtrans = total; iter = 0 (setup_state, cg.cpp:126)
    // peer transport: *out = total (if out); v = pre ? (0 + *pre) + total :
    // total; v -> recv_a / recv_b [rank] of every rank's window over NVLink,
    // then the matching flags get this iteration's stamp (release, .sys)
    FIN_PUBLISH_A = 5,
    FIN_PUBLISH_B = 6,
    // tasks variant, one rank: the alpha / beta_res reduction tasks
    // (cg.cpp:209-225, 290-311) folded into the tile kernels: *out = this
    // tile's partial, then a ticket over the `ntiles` tile kernels; the last
    // to finish sums tparts[0..ntiles) in tile order and finalizes with
    // `then` (FIN_ALPHA / FIN_BETA) -- the sum combine_kernel would form
    FIN_TILES = 7
};

struct PeerLinks;

struct Fin {
    int mode;
    double* out;
    CgScalars* sc;
    double* history;
    const PeerLinks* links = nullptr; // FIN_PUBLISH_*: device copy of the links
    const double* pre = nullptr;      // FIN_PUBLISH_A: the interior rows' partial
    // FIN_TILES: tile partials, their count, the cross-kernel ticket, the
    // finalize of the last tile
    const double* tparts = nullptr;
    int ntiles = 0;
    int then = FIN_NONE;
    unsigned* tticket = nullptr;
};

// Where an update kernel takes its scalar from: sc->alpha / sc->beta when
// count == 0, else recomputed per block from `count` partials summed in
// order (the cross-rank allgather result); with sc == nullptr (the
// standalone tw_update_* ops) the scalar itself is *parts.
// With `flags` (peer transport) every block first acquire-waits until the
// `count` flags carry this iteration's stamp, then reads the partials.
struct ScalarSrc {
    const double* parts;
    int count;
    const unsigned long long* flags = nullptr;
};

// ---------------------------------------------------------------- launchers

struct LaunchCfg {
    int spmv_blocks;   // grid for the SpMV family (SMs x resident blocks)
    int stream_blocks; // grid for streaming vector kernels
    int threads;       // 256
    int tma_blocks;    // one CTA per SM for the TMA-staged SpMV
};

struct RowRange {
    int64_t r0, r1;
};

// K1: y = A x over up to two local row ranges; optional fused dot(x_diag, y).
// With `wait_flags` (peer transport: the ghost-plane flags) every block
// first acquire-waits for this iteration's stamp (fin.sc) before gathering.
// pdl: programmatic dependent launch (the single-domain monolithic chain).
void launch_spmv(const EllView& A, const double* x, double* y, RowRange a, RowRange b,
                 bool with_dot, RedScratch rs, Fin fin, int blocks, cudaStream_t s,
                 const unsigned long long* wait_flags = nullptr, int nwait = 0, bool pdl = false);
// K2: x += alpha p; r -= alpha Ap; r.r partial/finalize.  x == nullptr:
// r only (K3 applies the x update, launch_update_p's x).
void launch_update_xr(int64_t i0, int64_t i1, double* x, const double* p, double* r,
                      const double* Ap, CgScalars* sc, ScalarSrc alpha_src, RedScratch rs,
                      Fin fin, int blocks, cudaStream_t s, bool pdl = false, int role = PDL_DEFAULT);
// K3: p = r + beta p (beta from sc or recomputed from partials; with x,
// also x += alpha p_old, alpha = sc->alpha; with
// partials, the last block also commits rtrans/history/iter).
// With `links` (device copy), K3 also stores the first / last owned plane
// into the neighbours' ghost planes and its last block raises their flags.
void launch_update_p(int64_t i0, int64_t i1, const double* r, double* p, CgScalars* sc,
                     ScalarSrc beta_src, RedScratch rs, double* history, int blocks,
                     cudaStream_t s, const PeerLinks* links = nullptr,
                     const double* psrc = nullptr, bool pdl = false, double* x = nullptr,
                     const double* p0 = nullptr, int role = PDL_DEFAULT);
// (with p0: the K3 of an x-update pair's second iteration, p = r + beta psrc,
// x = (x + alpha_prev p0) + alpha psrc; p may alias p0)
// K1 of the peer transport as one launch (interior, then the two boundary
// ranges after a per-warp ghost-flag acquire), partials bit-identical to
// the two launches; pm[0] = interior p.Ap into *fin.pre, fin (FIN_PUBLISH_A)
// for the boundary.  False when it does not apply (then two launches).
bool launch_spmv_split(const EllView& A, const double* x, double* y, RowRange interior,
                       RowRange b0, RowRange b1, RedScratch rs, Fin fin, cudaStream_t s,
                       const unsigned long long* wait_flags, int nwait, bool pdl = false);
// Transport check: ping_send stores `token` into ping[rank] of every rank's
// window (release, .sys); ping_check waits (bounded, no trap) until every
// ping[q] of this rank's window holds it and writes 1 / 0 to *ok.
void launch_peer_ping_send(const PeerLinks& L, unsigned long long token, cudaStream_t s);
void launch_peer_ping_check(const PeerWindow* win, int nranks, unsigned long long token,
                            long long timeout_ns, int* ok, cudaStream_t s);
void launch_peer_push(const double* p_owned, int64_t n, int64_t plane, const PeerLinks& L,
                      const CgScalars* sc, unsigned* ticket, cudaStream_t s);
// One rank of the concurrent rank-group kernel (tw_cg_group_iterate_concurrent).
struct GroupRank {
    EllView A;
    double *x, *r, *p_local, *p_owned, *Ap, *pm, *send_b, *history;
    CgScalars* sc;
    RedScratch rs;
    PeerWindow* win;
    const PeerLinks* links; // device copy
    const unsigned long long* ghost_flags;
    int n_ghost, P;
    int64_t n, int_r0, int_r1;
    unsigned* bar; // [count, generation]
    int stage_bytes, val_bytes, c16_bytes; // x-staged K1 stages (A.cols16 set)
};
constexpr int kGroupThreads = 256; // threads per rank-group block (= kThreads)
// smem: dynamic shared memory per block (the staged K1's stages, or 0)
int rank_group_blocks_per_rank(int nranks, int smem);
void launch_rank_group(const GroupRank* ranks_dev, int nranks, int blocks_per_rank,
                       int iterations, int jitter, int smem, cudaStream_t s);
// Per-warp stage of the x-staged K1: values, 16-bit columns, 9 x runs.
int staged_stage_bytes(int max_width, int* val_bytes, int* c16_bytes);
// Builds the 16-bit staged columns of a stencil matrix or z-slab
// (nx % 32 == 0; A carries sx_*) from its 32-bit columns; flags *bad if any
// stored column falls outside its slice's staged runs (then the matrix
// stays unstaged).
void launch_stencil_cols16(const EllView& A, uint16_t* cols16, unsigned* bad, cudaStream_t s);
// Run table (int32[n_slices * 9]) + 16-bit columns of a general matrix from
// its 32-bit columns (tw_ell_from_csr); flags *bad if a slice's columns need
// more than 9 runs of 36 (then the matrix stays unstaged).
void launch_csr_runs(const EllView& A, int32_t* runs, uint16_t* cols16, unsigned* bad,
                     cudaStream_t s);
// K1 on an x-staged matrix: the slice block and its 9 x runs arrive in one
// TMA transaction per slice; x must have 2 readable doubles of slack before
// index 0 and after x_len.  The three ranges form ONE index space (walked
// like launch_spmv's two), or with split = true two -- ra, then rb0 ++ rb1
// with its own p.Ap partial (grid_reduce2_finalize), the x runs of its
// slices staged only after the warp's acquire of wait_flags (the peer
// transport's ghost planes; launch_spmv_split's contract).  Without split a
// non-zero nwait holds every slice's x runs until the flags are up.
bool launch_spmv_staged(const EllView& A, const double* x, double* y, RowRange ra, RowRange rb0,
                        RowRange rb1, bool split, RedScratch rs, Fin fin, cudaStream_t s,
                        const unsigned long long* wait_flags = nullptr, int nwait = 0,
                        bool pdl = false, int role = PDL_DEFAULT);
inline bool launch_spmv_staged(const EllView& A, const double* x, double* y, RowRange rows,
                               RedScratch rs, Fin fin, cudaStream_t s, bool pdl = false,
                               int role = PDL_DEFAULT) {
    return launch_spmv_staged(A, x, y, rows, RowRange{0, 0}, RowRange{0, 0}, false, rs, fin, s,
                              nullptr, 0, pdl, role);
}
int spmv_staged_smem_bytes(int max_width);
// Checked build only: every stored column in [-1, x_len), padding only
// trailing a row, slice widths within max_width (traps otherwise).
void launch_ell_check(const EllView& A, cudaStream_t s);
// K4: dot(a, b) over [i0, i1) with finalize.
void launch_dot(const double* a, const double* b, int64_t i0, int64_t i1, RedScratch rs, Fin fin,
                int blocks, cudaStream_t s);
void launch_waxpby(double alpha, const double* x, double beta, const double* y, double* w,
                   int64_t i0, int64_t i1, int blocks, cudaStream_t s);
// Sum `count` partials in order, then finalize (1 warp).
void launch_combine(const double* parts, int count, Fin fin, cudaStream_t s);
void launch_fill(double* p, int64_t n, double v, int blocks, cudaStream_t s);
void launch_rhs_splitmix(uint64_t seed, int64_t first, int64_t count, double* out, int blocks,
                         cudaStream_t s);
void launch_rhs_xorshift(const uint64_t* chunk_states, int64_t chunk, int64_t count,
                         int64_t skip, double* out, int blocks, cudaStream_t s);

// K0 pieces
void launch_stencil_widths(int64_t nx, int64_t ny, int64_t nz, int64_t row_offset,
                           int64_t n_rows, int64_t n_slices, int64_t* widths_out, int blocks,
                           cudaStream_t s);
void launch_stencil_fill(int64_t nx, int64_t ny, int64_t nz, int64_t row_offset,
                         int64_t col_offset, int64_t n_rows, int64_t n_slices,
                         const int64_t* slice_off, double* vals, int32_t* cols, uint16_t* c16,
                         int blocks, cudaStream_t s);
void launch_csr_fill(const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                     int64_t n_rows, int64_t n_slices, const int64_t* slice_off, double* vals,
                     int32_t* cols, int blocks, cudaStream_t s);
void launch_csr_widths(const int64_t* row_ptr, int64_t n_rows, int64_t n_slices,
                       int64_t* widths_out, int blocks, cudaStream_t s);
// In-place exclusive scan of int64 (n + 1 entries written: out[0] = 0).
void scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* tmp,
                        cudaStream_t s);
int64_t scan_tmp_elems(int64_t n);
void launch_band(const EllView& A, int64_t r0, int64_t r1, unsigned long long* minmax,
                 int blocks, cudaStream_t s);

int spmv_tma_smem_bytes(int max_width);
int spmv_tma_warps(); // consumer warps per CTA of the TMA SpMV

// ------------------------------------------------- persistent DAG dispatcher

enum DagKind : int { DK_SPMV = 0, DK_ALPHA = 1, DK_UPD = 2, DK_BETA = 3, DK_UPDP = 4, DK_HALO = 5 };

// DagTask::flags: an SpMV tile whose band reads a ghost plane waits for that
// plane's flag (the neighbour's halo task of the same iteration) first.
constexpr int kDagGhostLo = 1, kDagGhostHi = 2;
// paired x updates (one rank): the SpMV of a pair's second iteration reads
// p from the pair buffer; the pair's first p update writes it there and
// leaves x, the second applies both x updates and writes p back
constexpr int kDagReadP2 = 4, kDagXDefer = 8, kDagXPair = 16;

// One physical task of the flattened K-iteration DAG (tw_dag.cu).
struct DagTask {
    int kind;
    int tile;
    int rank;         // index into DagParams::rk (0 on one rank)
    int iter;         // iteration within the launch (stamps of the peer flags)
    int flags;        // kDagGhost*, kDagReadP2, kDagXDefer, kDagXPair
    int64_t r0, r1;   // local rows of the tile
    int chunk0;       // first index in the global chunk list
    int nchunks;
    int succ0, nsucc; // successor task ids in DagParams::succ
};

// One rank's solver state as the dispatcher reads it.  Across ranks (the
// NVLink peer transport) the cross-rank edges of the DAG are the peer
// protocol of the monolithic path: the halo task stores the rank's first /
// last owned plane into the neighbours' ghost planes and raises their ghost
// flags; alpha / beta_res publish the rank's tile-order partial into every
// rank's window and wait for all P (sums in rank order).  Flags carry the
// stamp epoch << 32 | (iter0 + task.iter + 1).
struct DagRank {
    EllView A;
    const double* p_local;   // gathered (owned + ghost planes)
    double* p_owned;
    const double* p2_local;  // the pair buffer (paired x updates), else null
    double* p2_owned;
    double* x;
    double* r;
    double* Ap;
    CgScalars* sc;
    double* history;
    unsigned long long* stamps; // globaltimer at each iteration end (index iter + 1)
    double* pa;              // tile partials of p.Ap
    double* rr;              // tile partials of r.r
    const PeerLinks* links;  // device copy; null on one rank
    const PeerLinks* links2; // the same with the pair-buffer ghost targets (paired x updates)
    PeerWindow* win;         // this rank's window (flags it waits on)
    unsigned* tctr;          // [2] SpMV / x-r tiles done this iteration (publication)
    int iter0;               // iterations done before this launch
};
constexpr int kDagMaxRanks = 16; // ranks of one launch (a real GPU: 1; an emulated group: P)

struct DagParams {
    const DagTask* tasks;
    const int* chunk_task;   // chunk -> task
    const int* succ;
    int* remaining;          // unfinished predecessors per task
    unsigned* chunk_done;    // finished chunks per task
    double* chunk_part;      // per-chunk dot partial
    unsigned* ticket;        // next chunk to hand out
    int nchunks;
    int ntasks;              // entries of tasks (bounds of the checked build)
    int T;                   // tiles per iteration and rank
    int nranks;              // entries of rk
    int max_width;           // widest slice over the ranks (sizes the stages)
    unsigned long long* start_stamp; // globaltimer when chunk 0 is taken
    int64_t spmv_chunk_slices;
    int64_t vec_chunk_rows;
    int stage_bytes, val_bytes, c16_bytes; // c16_bytes: the column block (16- or 32-bit)
    // rows per TMA block of the update chunks (x, p, r, Ap / r, p in the
    // warp's stage); 0 = register path
    int upd_block_rows, updp_block_rows;
    int x_in_updp; // x += alpha p_old in the p-update chunks (TMA path only)
    int x_pairs;   // paired x updates (the dag_kernel<true> instantiation)
    DagRank rk[kDagMaxRanks];
};

int dag_smem_bytes(int max_width, bool staged, int* stage_bytes, int* val_bytes, int* c16_bytes);
int dag_threads();
int dag_compute_warps();
int dag_blocks(int max_width, bool staged, int sm_count);
void launch_dag(const DagParams& P, int blocks, cudaStream_t s);

// Occupancy-derived launch configuration for this device.
LaunchCfg query_launch_cfg(int sm_count);

} // namespace tw
