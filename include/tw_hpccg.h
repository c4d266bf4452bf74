/*
 * tw_hpccg.h -- C ABI of the B200-native HPCCG hot path (libtw_hpccg.so).
 *
 * Drop-in boundary for the reference's CG path (taskweave, arXiv 2602.21897
 * artifact).  Every entry point names the reference interface it replaces
 * (file:line under /root/reference/proj).  Plain pointers and sizes only; no
 * C++ or torch types cross this boundary and no exception escapes it.
 *
 * Errors follow the reference's two exception classes
 * (include/taskweave/types.hpp:23-33): TW_ERR_CONFIG for malformed input
 * (ConfigError, CLI exit 1), TW_ERR_CONTRACT for API misuse
 * (ContractViolation, CLI exit 2), plus TW_ERR_CUDA / TW_ERR_NCCL for device
 * and communicator failures.  tw_last_error_string() returns the message of
 * the last failing call on the calling thread.
 *
 * Pointers documented "device" are CUDA device pointers on the context's
 * device; "host" pointers are ordinary (preferably pinned) host memory.
 * `stream` arguments are cudaStream_t passed as void* (NULL = the context's
 * compute stream).
 */
#ifndef TW_HPCCG_H
#define TW_HPCCG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TW_OK 0
#define TW_ERR_CONFIG 1
#define TW_ERR_CONTRACT 2
#define TW_ERR_CUDA 3
#define TW_ERR_NCCL 4

#define TW_ABI_VERSION 3

typedef struct tw_ctx tw_ctx; /* replaces tw::Runtime + sim::Device (runtime.hpp:25-55, sim_device.hpp:91-166) */
typedef struct tw_ell tw_ell; /* replaces tw::bench::CsrMatrix on the device (csr.hpp:9-17) */
typedef struct tw_cg tw_cg;   /* replaces the CgRun solve state (cg.cpp:24-48) */

const char* tw_last_error_string(void);
int tw_abi_version(void);

/* ---------------------------------------------------------------- context */

/* Runtime(RuntimeConfig) + Device(...) (runtime.cpp:5-34, sim_device.cpp:77-85):
 * binds `device`, creates the compute stream and a pool of
 * `stream_pool_capacity` streams (QueuePool capacity, task_aware.hpp:83-109;
 * CgOptions::stream_pool_capacity default 4, cg.hpp:42). */
int tw_ctx_create(int device, unsigned stream_pool_capacity, tw_ctx** out);
int tw_ctx_destroy(tw_ctx* ctx);
int tw_ctx_compute_stream(tw_ctx* ctx, void** stream_out);
int tw_ctx_synchronize(tw_ctx* ctx);
/* Number of SMs and device ordinal, for launch sizing reports. */
int tw_ctx_device_info(tw_ctx* ctx, int* device, int* sm_count);

/* Multi-GPU (no reference equivalent: SPEC.md:291 lists multiple devices as a
 * non-goal).  One rank per GPU; the 128-byte id comes from
 * rank 0's tw_comm_unique_id and is broadcast by the caller.  NCCL is loaded
 * at run time (libnccl.so.2). */
int tw_comm_unique_id(unsigned char id_out[128]);
int tw_ctx_init_comm(tw_ctx* ctx, int rank, int nranks, const unsigned char id[128]);
int tw_ctx_comm_info(tw_ctx* ctx, int* rank, int* nranks);
/* (Emulated ranks on one device for the multi-rank tests: tw_hpccg_emulation.h.) */

/* Device buffers for callers without another allocator (tests, bench). */
int tw_malloc(tw_ctx* ctx, void** ptr, int64_t bytes);
int tw_free(tw_ctx* ctx, void* ptr);
int tw_malloc_host(void** ptr, int64_t bytes); /* pinned */
int tw_free_host(void* ptr);
int tw_memcpy(tw_ctx* ctx, void* dst, const void* src, int64_t bytes, void* stream); /* any direction, async */

/* ----------------------------------------------------------- matrix (K0) */

typedef struct tw_ell_info_t {
    int64_t nx, ny, nz;      /* 0 for matrices not generated as a stencil   */
    int64_t z_begin, z_end;  /* owned z-planes of the slab                  */
    int64_t n_global;        /* rows of the global operator                 */
    int64_t n_rows;          /* owned rows (local)                          */
    int64_t row_offset;      /* global row of local row 0                   */
    int64_t col_offset;      /* global column of local column 0             */
    int64_t x_len;           /* local length of a gathered vector (owned + ghost planes) */
    int64_t nnz;             /* true nonzeros of the owned rows             */
    int64_t n_slices;        /* 32-row slices                               */
    int64_t ell_entries;     /* stored entries incl. padding                */
    int32_t max_width;       /* widest slice                                */
    int32_t slice_rows;      /* 32                                          */
} tw_ell_info_t;

/* z-slab decomposition (no reference equivalent; the reference's row tiles,
 * cg.cpp:348-370, are the single-address-space analogue): the geometry of
 * the owned planes [z_begin, z_end) of an nx*ny*nz grid.  Host only. */
typedef struct tw_slab_t {
    int64_t nx, ny, nz, z_begin, z_end, plane;
    int64_t n_rows, row_offset, col_offset, x_len, diag_shift, nnz;
    int64_t interior_r0, interior_r1;           /* local rows that read no ghost plane */
    int64_t send_lo, recv_lo, send_hi, recv_hi; /* halo planes, local x coordinates    */
    int32_t ghost_lo, ghost_hi;
} tw_slab_t;
int tw_slab_plan(int64_t nx, int64_t ny, int64_t nz, int64_t z_begin, int64_t z_end,
                 tw_slab_t* out);
/* Strong-scaling split of nz planes over ranks: [nz*r/R, nz*(r+1)/R). */
int tw_slab_partition(int64_t nz, int rank, int nranks, int64_t* z_begin, int64_t* z_end);

/* gen_stencil_matrix(nx,ny,nz) (csr.cpp:29-59), generated on the device into
 * sliced ELL, for the z-slab [z_begin, z_end) (pass 0, nz for the whole grid).
 * Per-row entry order, columns and values are the reference's exactly.
 * TW_ERR_CONFIG on dims < 1 or overflow (csr.cpp:30-34). */
int tw_gen_stencil_ell(tw_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, int64_t z_begin,
                       int64_t z_end, tw_ell** out);
/* CsrMatrix -> device ELL (load_csr interop, csr.cpp:76-98).  Host arrays;
 * validated like CsrMatrix::validate (csr.cpp:13-27). */
int tw_ell_from_csr(tw_ctx* ctx, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                    const double* values, tw_ell** out);
int tw_ell_info(const tw_ell* A, tw_ell_info_t* out);
/* 1 when the matrix also carries the x-staged form the CG's K1 uses (16-bit
 * column indices into 9 per-slice windows of x: closed-form windows for a
 * stencil or z-slab with nx % 32 == 0, a per-slice run table otherwise),
 * else 0. */
int tw_ell_x_staged(const tw_ell* A, int* staged);
/* Builds (enable != 0) or drops the x-staged form; *staged (optional) says
 * whether the matrix carries it afterwards.  tw_ell_from_csr matrices get it
 * as a per-slice run table when every 32-row slice's columns fall into at
 * most 9 windows of 36 entries (the 27-point stencil does for nx % 32 == 0:
 * the reference's own gen_stencil_matrix output passed as a CsrMatrix runs
 * the same K1 as a device-generated grid); dropping it frees 2 B per entry
 * and makes the CG run the gather K1 (the results are bit-identical).  Call
 * it before creating solvers on A (their graphs and dispatcher tables hold
 * the form they were built with); tw_cg_solve's cached solvers of A are
 * dropped here. */
int tw_ell_set_x_staged(tw_ell* A, int enable, int* staged);
/* Device ELL -> host CSR with GLOBAL column indices (row_ptr int64[n_rows+1],
 * col_idx int64[nnz], values double[nnz]); the structure parity check. */
int tw_ell_to_csr(const tw_ell* A, int64_t* row_ptr, int64_t* col_idx, double* values);
/* Rows [row_begin, row_end) only (row_ptr relative: row_end - row_begin + 1
 * entries; col_idx / values sized max_width per row), so a grid whose CSR
 * does not fit host memory is checked a z-slab at a time.  staged != 0
 * decodes the 16-bit x-staged columns (the form the CG's K1 reads) through
 * the slices' run starts instead of the int32 columns (TW_ERR_CONTRACT when
 * the matrix has no x-staged form). */
int tw_ell_to_csr_rows(const tw_ell* A, int64_t row_begin, int64_t row_end, int staged,
                       int64_t* row_ptr, int64_t* col_idx, double* values);
int tw_ell_destroy(tw_ell* A);

/* ------------------------------------------------- streams and events
 * The reference's device / task-aware layer over real CUDA objects, for
 * callers that keep their own task graph.  Streams and
 * events are cudaStream_t / cudaEvent_t passed as void*. */

/* QueuePool::acquire / release (task_aware.cpp:122-166): one of the
 * context's pooled streams (capacity from tw_ctx_create); blocks, FIFO,
 * while every pooled stream is out.  Releasing a foreign stream is
 * TW_ERR_CONTRACT. */
int tw_stream_acquire(tw_ctx* ctx, void** stream);
int tw_stream_release(tw_ctx* ctx, void* stream);
/* sim::Device record_event / query / synchronize (sim_device.hpp:101-123). */
int tw_event_create(void** ev);
int tw_event_destroy(void* ev);
int tw_event_record(void* ev, void* stream);
int tw_event_query(void* ev, int* done); /* non-blocking: *done = 0 / 1 */
/* TaskAware::wait_transformed (task_aware.cpp:50-60): poll and yield until
 * ev completes; never a blocking driver wait. */
int tw_event_wait(tw_ctx* ctx, void* ev);
/* A device-side edge: later work on `stream` waits for ev. */
int tw_stream_wait_event(void* stream, void* ev);
/* TaskAware::bind_event_async (task_aware.cpp:43-48, 92-96): the context's
 * polling thread calls done(arg) once it observes ev complete (the
 * release-dependents hook).  The caller keeps ev alive until then;
 * callbacks still pending at tw_ctx_destroy are dropped. */
int tw_event_bind_async(tw_ctx* ctx, void* ev, void (*done)(void* arg), void* arg);

/* ------------------------------------------------------- kernels (K1-K4) */

/* spmv_range(A, x, y, r0, r1) (kernels.cpp:5-13): y[i] for local rows
 * [r0, r1); x is a device vector of length x_len (owned + ghost planes),
 * y of length n_rows.  Bit-identical to the reference (per-row order kept,
 * no FMA, padding masked). */
int tw_spmv_range(const tw_ell* A, const double* x, double* y, int64_t r0, int64_t r1,
                  void* stream);
/* spmv_range + dot_range(p, Ap, r0, r1) fused (K1): *dot_dev (device double)
 * receives sum_{i in [r0,r1)} p[i]*Ap[i] (fixed-order tree reduction). */
int tw_spmv_dot(const tw_ell* A, const double* p, double* Ap, int64_t r0, int64_t r1,
                double* dot_dev, void* stream);
/* dot_range(a, b, i0, i1) (kernels.cpp:15-20) into *out_dev (device double). */
int tw_dot_range(tw_ctx* ctx, const double* a, const double* b, int64_t i0, int64_t i1,
                 double* out_dev, void* stream);
/* waxpby_range(alpha, x, beta, y, w, i0, i1) (kernels.cpp:22-26): three
 * roundings per element, w may alias x or y; bit-identical. */
int tw_waxpby_range(tw_ctx* ctx, double alpha, const double* x, double beta, const double* y,
                    double* w, int64_t i0, int64_t i1, void* stream);

/* exchange_externals (HPCCG's halo step; in the reference, the column band
 * of make_tile_plan, cg.cpp:356-367, declared as the read region of p,
 * cg.cpp:177-180): on a z-slab matrix A (tw_gen_stencil_ell with z_begin /
 * z_end) of a communicator rank, send the first / last owned plane of the
 * local vector x (x_len entries: [ghost lo] owned [ghost hi]) to the
 * neighbours and receive theirs into the ghost planes -- one NCCL send/recv
 * group on `stream`, collective over the ranks.  A no-op for one rank. */
int tw_halo_exchange(const tw_ell* A, double* x, void* stream);

/* The CG's fused update kernels as standalone operators, scalars read on
 * the device (no host round trip inside a caller's DAG):
 *   K2 (x_up + r_up + dot_rr, cg.cpp:380-386 / 262-288):
 *      x += a p; r += (-a) Ap; *rr_dev = sum r[i]^2 over [i0, i1), a = *alpha_dev
 *   K3 (p_up, cg.cpp:389 / 313-332): p = r + b p, b = *beta_dev
 * Same roundings as waxpby_range (bit-identical); the dot is a fixed-order
 * tree. */
int tw_update_xr_rr(tw_ctx* ctx, const double* alpha_dev, double* x, const double* p, double* r,
                    const double* Ap, int64_t i0, int64_t i1, double* rr_dev, void* stream);
int tw_update_p(tw_ctx* ctx, const double* beta_dev, const double* r, double* p, int64_t i0,
                int64_t i1, void* stream);

/* make_tile_plan(A, tiles) (cg.cpp:348-370) over the owned rows; band in
 * GLOBAL columns like the reference.  TW_ERR_CONFIG if tiles < 1 or > rows. */
int tw_make_tile_plan(const tw_ell* A, int tiles, int64_t* r0, int64_t* r1, int64_t* band_lo,
                      int64_t* band_hi);

/* Right-hand sides generated on the device, element offset `first` of the
 * global sequence: xorshift64 (acceptance.cpp:48-58 / test_bench.cpp:26-36)
 * and SplitMix64 (scenario.cpp:46-55). */
int tw_rhs_xorshift(tw_ctx* ctx, uint64_t seed, int64_t first, int64_t count, double* out_dev,
                    void* stream);
int tw_rhs_splitmix(tw_ctx* ctx, uint64_t seed, int64_t first, int64_t count, double* out_dev,
                    void* stream);

/* ------------------------------------------------------------------- CG */

#define TW_CG_MONOLITHIC 0 /* cg_monolithic (cg.cpp:397-436)                    */
#define TW_CG_TASKS 1      /* cg_tasks block-task DAG (cg.cpp:166-334, 438-447)  */

typedef struct tw_cg_options {
    int variant;                   /* TW_CG_MONOLITHIC | TW_CG_TASKS                  */
    int tiles;                     /* CgOptions::tiles (cg.hpp:38); forced 1 for monolithic */
    unsigned stream_pool_capacity; /* CgOptions::stream_pool_capacity (cg.hpp:42)    */
    int use_graph;                 /* capture one iteration as a CUDA graph            */
    int iteration_marks;           /* CgOptions::iteration_marks: host poller stamps cg_iter=i */
    double tol;                    /* CgOptions::tol: converged = last residual < tol  */
    int dispatch;                  /* TW_DISPATCH_AUTO (default) | _STREAMS | _PERSISTENT | _CHAIN */
    /* Placement and tuning choices that change no result bit (x_update,
     * l2_keep) or only the dispatcher's chunk-order reduction tree (chunk
     * sizes; within the SURVEY 8(c) rule).  0 = the library's choice. */
    int x_update;                  /* TW_XUPD_AUTO | _K2 | _K3: where x += alpha p runs    */
    int l2_keep;                   /* TW_L2KEEP_AUTO | _ON | _OFF: staged K1's x-run policy */
    int64_t dag_spmv_slices;       /* persistent dispatcher: slices per SpMV chunk         */
    int64_t dag_vec_rows;          /* persistent dispatcher: rows per update chunk         */
} tw_cg_options;

#define TW_XUPD_AUTO 0   /* K3 pairs from 512k rows per rank (monolithic, tasks on streams /
                          * graphs) or 4M (the persistent dispatcher; across ranks the global
                          * rows per rank decide, alike on every rank); else K3 from 4M rows
                          * per rank (8n bytes less per iteration), else K2                  */
#define TW_XUPD_K2 1     /* in K2 with r -= alpha Ap                                        */
#define TW_XUPD_K3 2     /* in K3, reading p before it is overwritten                       */
#define TW_XUPD_K3_PAIRS 3 /* in K3 once per pair of iterations, x = (x + a_k p_k) + a_k+1 p_k+1
                            * (every executor, one rank or across ranks; 4n bytes less per
                            * iteration than _K3)                                              */
#define TW_L2KEEP_AUTO 0 /* evict_last on the staged x runs while x has <= 8M entries       */
#define TW_L2KEEP_ON 1
#define TW_L2KEEP_OFF 2

#define TW_DISPATCH_STREAMS 0    /* one launch per task, cudaStreamWaitEvent edges (or graph) */
#define TW_DISPATCH_PERSISTENT 1 /* one persistent kernel runs the whole DAG: chunked tasks,
                                    device-side dependency counters (tasks variant, 1 rank) */
#define TW_DISPATCH_AUTO 2       /* tasks variant on one rank, no graph requested: the
                                    programmatic chain for 2-8 tiles of >= 50k rows on an
                                    x-staged matrix, the persistent dispatcher for more / smaller
                                    tiles, streams otherwise (the measured winners) */
#define TW_DISPATCH_CHAIN 3      /* the tasks variant's tile kernels in DAG order on ONE
                                    stream, each launched programmatically: a phase's
                                    first tile waits for the grids before it
                                    (griddepcontrol.wait), its other tiles start behind it
                                    and run side by side (tasks variant, 1 rank, x-staged
                                    matrix; also under use_graph) */

/* Fills the defaults of CgOptions (cg.hpp:37-45) with the cuda backend. */
void tw_cg_options_default(tw_cg_options* opt);

/* setup_state (cg.cpp:75-128): allocates x|r|p|Ap and the scalar block on the
 * device for up to `max_iterations` history entries. */
int tw_cg_create(tw_ctx* ctx, const tw_ell* A, const tw_cg_options* opt, int max_iterations,
                 tw_cg** out);
int tw_cg_destroy(tw_cg* cg);
/* x = 0, r = p = b, rtrans = dot(r, r) (cg.cpp:124-127); b has n_rows entries
 * (this rank's rows), on the host or the device. */
int tw_cg_set_rhs(tw_cg* cg, const double* b, int b_is_device);
/* Enqueues `iterations` CG iterations (asynchronous; scalars stay on the
 * device, no host round trip). */
int tw_cg_iterate(tw_cg* cg, int iterations);
/* Waits for everything enqueued (host poll of the completion events,
 * TaskAware::wait_transformed semantics, task_aware.cpp:50-60). */
int tw_cg_wait(tw_cg* cg);
int tw_cg_iterations_done(tw_cg* cg, int* done);
/* residual_history (cg.hpp:13): sqrt(r.r) after each iteration run so far. */
int tw_cg_history(tw_cg* cg, double* host_out, int count);
/* x of this rank's rows, to host. */
int tw_cg_solution(tw_cg* cg, double* host_x);
/* Device pointers of the state vectors (x, r, p incl. ghosts, Ap). */
int tw_cg_vectors(tw_cg* cg, double** x, double** r, double** p, double** Ap);
/* Host wall time (seconds since tw_cg_set_rhs) at which the poller saw each
 * iteration complete (the cg_iter=i marks, cg.cpp:307-308); 0 if unseen. */
int tw_cg_iteration_marks(tw_cg* cg, double* host_out, int count);
/* Device-timed duration (seconds) of each iteration since tw_cg_set_rhs:
 * the difference of consecutive iteration-end events (the scenario CSV's
 * iter_time, scenario.cpp:115-124, in seconds instead of virtual units).
 * Needs iteration_marks. */
int tw_cg_iteration_times(tw_cg* cg, double* seconds, int count);
/* Logical block-task DAG of the tasks variant for the iterations enqueued so
 * far: edges as "pred succ\n" label pairs (labels "spmv:i:t", "dot_pAp:i:t",
 * "alpha:i:0", ... as in cg.cpp:168-170).  Returns needed size in *needed. */
int tw_cg_task_edges(tw_cg* cg, char* buf, int64_t cap, int64_t* needed);
/* Per-kernel device timing of the monolithic variant (graph capture off):
 * when enabled, each iteration brackets K1 (spmv_pAp), K2 (update_xr) and
 * K3 (update_p) with CUDA timing events on the stream they launch on.
 * tw_cg_kernel_times returns the summed milliseconds per kernel and the
 * number of timed iterations since the last enable; it synchronises. */
int tw_cg_enable_kernel_timing(tw_cg* cg, int enable);
int tw_cg_kernel_times(tw_cg* cg, double* k1_ms, double* k2_ms, double* k3_ms, int* iterations);
/* The same logical DAG without a device: dependency inference over the
 * access regions of spawn_iteration (cg.cpp:173-333) for the given tile plan
 * (rows local, band in local x coordinates, inclusive), `iterations`
 * iterations, optional ghost planes (a rank's halo task).  Runs on the host
 * only; the edge list is what tw_cg_task_edges reports for a real solve. */
int tw_task_dag_edges(int64_t n_rows, int tiles, const int64_t* r0, const int64_t* r1,
                      const int64_t* band_lo, const int64_t* band_hi, int64_t diag_shift,
                      int64_t plane, int ghost_lo, int ghost_hi, int iterations, char* buf,
                      int64_t cap, int64_t* needed);
/* Physical launches per iteration (kernels + NCCL calls), for reports:
 * monolithic 3 kernels (K1, K2, K3; across ranks 5 over NCCL, 3-4 over the
 * peer transport); tasks 3 per tile plus the alpha / beta_res combines (none
 * when folded into the tiles, 4 across ranks); the persistent dispatcher is
 * one launch per tw_cg_iterate call (reported as 0). */
int tw_cg_launches_per_iteration(tw_cg* cg, int* kernels, int* collectives);

/* What a solver actually executes (for reports and tests: the bench line
 * names the kernel instantiation its roofline is measured on). */
#define TW_K1_REGISTER 0       /* register-path gather SpMV (rows wider than the TMA stages) */
#define TW_K1_TMA_GATHER 1     /* spmv_tma_kernel: TMA-staged matrix, gathered x              */
#define TW_K1_STAGED 2         /* spmv_tma_staged_kernel, closed-form x runs (nx % 32 == 0)   */
#define TW_K1_STAGED_TABLE 3   /* spmv_tma_staged_kernel, per-slice run table                 */
#define TW_TRANSPORT_NONE 0
#define TW_TRANSPORT_NCCL 1
#define TW_TRANSPORT_PEER 2
#define TW_TRANSPORT_LOOPBACK 3 /* emulated rank group on one device */
typedef struct tw_cg_mode_t {
    int32_t variant;   /* TW_CG_MONOLITHIC | TW_CG_TASKS                     */
    int32_t tiles;
    int32_t dispatch;  /* TW_DISPATCH_STREAMS | _PERSISTENT | _CHAIN (AUTO resolved) */
    int32_t use_graph;
    int32_t k1_form;   /* TW_K1_*                                            */
    int32_t k1_l2_keep; /* staged K1 stages the x runs with L2 evict_last     */
    int32_t x_in_k3;   /* x += alpha p runs in K3 (else in K2); 2: in pairs  */
    int32_t transport; /* TW_TRANSPORT_*                                     */
    int32_t nranks;
    int32_t kernels_per_iteration;
    int32_t collectives_per_iteration;
} tw_cg_mode_t;
int tw_cg_mode(tw_cg* cg, tw_cg_mode_t* out);


/* NVLink peer transport for the monolithic multi-rank iteration: the halo is
 * stored by K3 straight into the neighbours' ghost planes and the rank
 * partials of p.Ap / r.r into every rank's receive window, each followed by
 * a release flag the consumer acquires (no NCCL inside the iteration; NCCL
 * stays for set_rhs).  Setup: every rank exports a blob (CUDA IPC handles
 * of its window and p buffer), the blobs are all-gathered in rank order by
 * the caller, then every rank connects. */
#define TW_PEER_BLOB_BYTES 256
int tw_cg_peer_export(tw_cg* cg, unsigned char* blob);
int tw_cg_peer_connect(tw_cg* cg, const unsigned char* blobs);
/* Transport check after connecting: every rank calls ping_send, then (after
 * a host barrier) ping_check, which waits at most timeout_ms for every
 * rank's store to be visible in this rank's window and sets *ok = 1 / 0
 * (never traps).  A caller falls back to NCCL when any rank reports 0. */
int tw_cg_peer_ping_send(tw_cg* cg);
int tw_cg_peer_ping_check(tw_cg* cg, int timeout_ms, int* ok);

/* cg_monolithic / cg_tasks in one call (cg.cpp:397-447): host b in, host
 * history[iterations] and x[n_rows] out, *converged per CgResult (cg.hpp:12-17).
 * The context keeps one solver per matrix between calls (rebuilt when the
 * options change or more iterations are asked for; dropped with the matrix
 * or the context); calls on one context are serialised.  Pageable host
 * buffers move through pinned staging buffers filled / drained by host
 * threads while the copy engine runs (tw_cg_set_rhs, tw_cg_solution and
 * tw_ell_from_csr do the same). */
int tw_cg_solve(tw_ctx* ctx, const tw_ell* A, const double* b_host, int iterations,
                const tw_cg_options* opt, double* history_out, double* x_out, int* converged);

#ifdef __cplusplus
}
#endif

#endif /* TW_HPCCG_H */
