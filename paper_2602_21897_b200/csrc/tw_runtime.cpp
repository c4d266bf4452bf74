// Host runtime of libtw_hpccg: errors, context (device + streams + pool +
// NCCL), device sliced-ELL matrices, the kernel entry points and right-hand
// side generators.  The CG drivers live in tw_cg.cpp.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>

#include "tw_objects.h"

namespace tw {

thread_local std::string g_last_error;

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e == cudaSuccess) return;
    throw Error(TW_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file +
                                 ":" + std::to_string(line) + ")");
}

double host_seconds() {
    using clk = std::chrono::steady_clock;
    return std::chrono::duration<double>(clk::now().time_since_epoch()).count();
}

// ------------------------------------------------------------------- NCCL

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        auto sym = [h](const char* n) { return dlsym(h, n); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.GetErrorString =
            reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        api.loaded = api.GetUniqueId && api.CommInitRank && api.AllGather && api.Send &&
                     api.Recv && api.GroupStart && api.GroupEnd;
    });
    if (!api.loaded) throw Error(TW_ERR_NCCL, "libnccl.so.2 could not be loaded");
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    const char* s = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
    throw Error(TW_ERR_NCCL, std::string(what) + ": " + s);
}

// -------------------------------------------------------------- StreamPool

void StreamPool::init(int device, unsigned capacity) {
    TW_CUDA(cudaSetDevice(device));
    for (unsigned i = 0; i < capacity; ++i) {
        cudaStream_t s;
        TW_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        streams_.push_back(s);
        free_.push_back(static_cast<int>(i));
        held_.push_back(0);
    }
}

void StreamPool::destroy() {
    for (auto s : streams_) cudaStreamDestroy(s);
    streams_.clear();
    free_.clear();
    held_.clear();
}

int StreamPool::acquire() {
    std::unique_lock lk(mu_);
    cv_.wait(lk, [this] { return !free_.empty(); });
    int i = free_.front();
    free_.pop_front();
    held_[static_cast<size_t>(i)] = 1;
    return i;
}

// Releasing a stream that is not held (never acquired, or released twice)
// is API misuse, as QueuePool::release treats it (task_aware.cpp:150-153):
// accepting it would hand one stream to two later acquirers.
void StreamPool::release(int idx) {
    {
        std::lock_guard lk(mu_);
        if (idx < 0 || static_cast<size_t>(idx) >= held_.size() || !held_[static_cast<size_t>(idx)])
            contract_error("release of a pool stream that is not held");
        held_[static_cast<size_t>(idx)] = 0;
        free_.push_back(idx);
    }
    cv_.notify_one();
}

int StreamPool::index_of(cudaStream_t s) const {
    for (size_t i = 0; i < streams_.size(); ++i)
        if (streams_[i] == s) return static_cast<int>(i);
    return -1;
}

size_t StreamPool::outstanding() const {
    std::lock_guard lk(mu_);
    return streams_.size() - free_.size();
}

// --------------------------------------------------------------- TaskAware

TaskAware::~TaskAware() {
    {
        std::lock_guard lk(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    if (th_.joinable()) th_.join();
    for (auto& b : binds_)
        if (b.owned) cudaEventDestroy(b.ev);
    for (auto e : spare_) cudaEventDestroy(e);
}

cudaEvent_t TaskAware::take_event() {
    std::lock_guard lk(mu_);
    if (!spare_.empty()) {
        cudaEvent_t e = spare_.back();
        spare_.pop_back();
        return e;
    }
    cudaEvent_t e;
    TW_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return e;
}

void TaskAware::add(const Bind& b) {
    {
        std::lock_guard lk(mu_);
        binds_.push_back(b);
        if (!started_) {
            started_ = true;
            th_ = std::thread([this] { loop(); });
        }
    }
    cv_.notify_all();
}

void TaskAware::bind(cudaEvent_t ev, double* slot, double t0) {
    add(Bind{ev, slot, t0, nullptr, nullptr, true});
}

void TaskAware::bind_callback(cudaEvent_t ev, void (*done)(void*), void* arg) {
    add(Bind{ev, nullptr, 0.0, done, arg, false});
}

size_t TaskAware::poll_once() {
    std::vector<std::pair<void (*)(void*), void*>> fire;
    size_t done = 0;
    {
        std::lock_guard lk(mu_);
        const double now = host_seconds();
        // One pass over every bound event (they may sit on different streams);
        // a completed one is stamped / released, the rest stay bound.
        for (auto it = binds_.begin(); it != binds_.end();) {
            const cudaError_t q = cudaEventQuery(it->ev);
            if (q == cudaErrorNotReady) {
                ++it;
                continue;
            }
            if (it->slot) *it->slot = now - it->t0;
            if (it->owned) spare_.push_back(it->ev);
            if (it->done) fire.emplace_back(it->done, it->arg);
            it = binds_.erase(it);
            ++done;
        }
        polled_ += done; // under the lock: polled() never runs ahead of binds_
    }
    // the callbacks run outside the lock: they may bind further events
    for (auto& f : fire) f.first(f.second);
    return done;
}

void TaskAware::loop() {
    cudaSetDevice(device_);
    std::unique_lock lk(mu_);
    while (!stop_) {
        if (binds_.empty()) {
            cv_.wait(lk, [this] { return stop_ || !binds_.empty(); });
            continue;
        }
        lk.unlock();
        poll_once();
        std::this_thread::sleep_for(std::chrono::duration<double>(period_));
        lk.lock();
    }
}

void TaskAware::wait(cudaEvent_t ev) { wait_static(ev); }

void TaskAware::wait_static(cudaEvent_t ev) {
    for (;;) {
        cudaError_t q = cudaEventQuery(ev);
        if (q == cudaSuccess) return;
        if (q != cudaErrorNotReady) TW_CUDA(q);
        std::this_thread::yield();
    }
}

size_t TaskAware::pending() const {
    std::lock_guard lk(mu_);
    return binds_.size();
}

// ------------------------------------------------------- host <-> device

constexpr size_t kStageBytes = size_t(32) << 20; // per staging buffer

static bool host_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// memcpy split over up to 8 host threads (>= 4 MB each)
static void par_memcpy(void* dst, const void* src, size_t n) {
    const size_t hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t k = std::min<size_t>({8, hw, std::max<size_t>(1, n >> 22)});
    std::vector<std::thread> th;
    for (size_t i = 1; i < k; ++i) {
        const size_t a = n * i / k, b = n * (i + 1) / k;
        th.emplace_back([=] {
            std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
        });
    }
    std::memcpy(dst, src, n / k);
    for (auto& t : th) t.join();
}

static void ensure_staging(tw_ctx* ctx) {
    for (int i = 0; i < 2; ++i) {
        if (!ctx->stage[i]) TW_CUDA(cudaMallocHost(&ctx->stage[i], kStageBytes));
        if (!ctx->stage_ev[i]) {
            TW_CUDA(cudaEventCreateWithFlags(&ctx->stage_ev[i], cudaEventDisableTiming));
            TW_CUDA(cudaEventRecord(ctx->stage_ev[i], ctx->compute));
        }
    }
}

void copy_h2d(tw_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes < (size_t(8) << 20) || host_pinned(src)) {
        TW_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    std::lock_guard lk(ctx->stage_mu);
    ensure_staging(ctx);
    for (size_t off = 0, i = 0; off < bytes; off += kStageBytes, ++i) {
        const int b = static_cast<int>(i & 1);
        const size_t n = std::min(kStageBytes, bytes - off);
        TW_CUDA(cudaEventSynchronize(ctx->stage_ev[b])); // its previous copy has left
        par_memcpy(ctx->stage[b], static_cast<const char*>(src) + off, n);
        TW_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, ctx->stage[b], n,
                                cudaMemcpyHostToDevice, s));
        TW_CUDA(cudaEventRecord(ctx->stage_ev[b], s));
    }
}

void copy_d2h(tw_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes < (size_t(8) << 20) || host_pinned(dst)) {
        TW_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        TW_CUDA(cudaStreamSynchronize(s));
        return;
    }
    std::lock_guard lk(ctx->stage_mu);
    ensure_staging(ctx);
    const size_t nch = (bytes + kStageBytes - 1) / kStageBytes;
    auto issue = [&](size_t i) {
        const int b = static_cast<int>(i & 1);
        const size_t off = i * kStageBytes, n = std::min(kStageBytes, bytes - off);
        TW_CUDA(cudaEventSynchronize(ctx->stage_ev[b]));
        TW_CUDA(cudaMemcpyAsync(ctx->stage[b], static_cast<const char*>(src) + off, n,
                                cudaMemcpyDeviceToHost, s));
        TW_CUDA(cudaEventRecord(ctx->stage_ev[b], s));
    };
    issue(0);
    if (nch > 1) issue(1);
    for (size_t i = 0; i < nch; ++i) {
        const int b = static_cast<int>(i & 1);
        const size_t off = i * kStageBytes, n = std::min(kStageBytes, bytes - off);
        TW_CUDA(cudaEventSynchronize(ctx->stage_ev[b]));
        par_memcpy(static_cast<char*>(dst) + off, ctx->stage[b], n);
        if (i + 2 < nch) issue(i + 2);
    }
}

// ------------------------------------------------------------------ helpers

RedScratch ctx_red_scratch(tw_ctx* ctx, cudaStream_t s) {
    std::lock_guard lk(ctx->red_mu);
    auto it = ctx->red.find(s);
    if (it != ctx->red.end()) return it->second;
    RedScratch rs{};
    TW_CUDA(cudaMalloc(&rs.block_part, sizeof(double) * static_cast<size_t>(ctx->red_blocks)));
    TW_CUDA(cudaMalloc(&rs.ticket, sizeof(unsigned) * 4));
    TW_CUDA(cudaMemset(rs.ticket, 0, sizeof(unsigned) * 4));
    ctx->red.emplace(s, rs);
    return rs;
}

static void check_ctx(const tw_ctx* c) {
    if (!c) contract_error("null tw_ctx");
}
static void check_ell(const tw_ell* a) {
    if (!a || !a->ctx) contract_error("null tw_ell");
}
static cudaStream_t pick(tw_ctx* c, void* s) {
    return s ? static_cast<cudaStream_t>(s) : c->compute;
}


static void finish_ell(tw_ell* A, int64_t* widths, int64_t n_slices, cudaStream_t s) {
    int64_t* tmp = nullptr;
    TW_CUDA(cudaMalloc(&A->slice_off, sizeof(int64_t) * (n_slices + 1)));
    TW_CUDA(cudaMalloc(&tmp, sizeof(int64_t) * scan_tmp_elems(n_slices)));
    scan_exclusive_i64(widths, A->slice_off, n_slices, tmp, s);
    int64_t entries = 0;
    TW_CUDA(cudaMemcpyAsync(&entries, A->slice_off + n_slices, sizeof(int64_t),
                            cudaMemcpyDeviceToHost, s));
    std::vector<int64_t> w(static_cast<size_t>(n_slices));
    if (n_slices)
        TW_CUDA(cudaMemcpyAsync(w.data(), widths, sizeof(int64_t) * n_slices,
                                cudaMemcpyDeviceToHost, s));
    TW_CUDA(cudaStreamSynchronize(s));
    cudaFree(tmp);
    int64_t mw = 0;
    for (int64_t v : w) mw = std::max(mw, v / 32);
    A->info.max_width = static_cast<int32_t>(mw);
    A->info.ell_entries = entries;
    A->info.n_slices = n_slices;
    A->info.slice_rows = kSliceRows;
    // +32 entries of slack so 128-bit loads of a final short slice stay in bounds
    TW_CUDA(cudaMalloc(&A->vals, sizeof(double) * (entries + 64)));
    TW_CUDA(cudaMalloc(&A->cols, sizeof(int32_t) * (entries + 128)));
}

static void free_ell(tw_ell* A) {
    if (!A) return;
    cudaFree(A->slice_off);
    cudaFree(A->vals);
    cudaFree(A->cols);
    cudaFree(A->cols16);
    cudaFree(A->runs);
    delete A;
}

// gen_stencil_matrix (csr.cpp:29-59) for the slab [z_begin, z_end).
} // namespace tw

// z-slab geometry shared by the generator, the solver and the host tests:
// owned planes [z_begin, z_end), one ghost plane on each side that has a
// neighbour, local x coordinates starting at the lower ghost plane.
extern "C" int tw_slab_plan(int64_t nx, int64_t ny, int64_t nz, int64_t zb, int64_t ze,
                            tw_slab_t* out) {
    return tw::guarded([&] {
        using namespace tw;
        if (nx < 1 || ny < 1 || nz < 1) config_error("stencil dims must be at least 1");
        __int128 cells = static_cast<__int128>(nx) * ny * nz;
        if (cells * 27 > std::numeric_limits<int64_t>::max() / 8) config_error("stencil dims overflow");
        if (zb < 0 || ze > nz || zb >= ze) contract_error("slab [z_begin, z_end) outside [0, nz)");
        tw_slab_t p{};
        p.nx = nx;
        p.ny = ny;
        p.nz = nz;
        p.z_begin = zb;
        p.z_end = ze;
        p.plane = nx * ny;
        p.ghost_lo = zb > 0;
        p.ghost_hi = ze < nz;
        p.n_rows = (ze - zb) * p.plane;
        p.row_offset = zb * p.plane;
        p.col_offset = (zb - p.ghost_lo) * p.plane;
        p.x_len = (ze + p.ghost_hi - (zb - p.ghost_lo)) * p.plane;
        p.diag_shift = p.row_offset - p.col_offset;
        // rows whose stencil never touches a ghost plane (overlap the halo)
        p.interior_r0 = p.ghost_lo ? p.plane : 0;
        p.interior_r1 = p.ghost_hi ? p.n_rows - p.plane : p.n_rows;
        if (p.interior_r1 < p.interior_r0) p.interior_r1 = p.interior_r0;
        // halo in local x coordinates: send the first/last owned plane, receive the ghosts
        p.send_lo = p.diag_shift;
        p.recv_lo = 0;
        p.send_hi = p.diag_shift + p.n_rows - p.plane;
        p.recv_hi = p.diag_shift + p.n_rows;
        int64_t zspan = 0;
        for (int64_t z = zb; z < ze; ++z) zspan += 1 + (z > 0) + (z + 1 < nz);
        auto ss = [](int64_t d) { return d == 1 ? int64_t{1} : 3 * d - 2; };
        p.nnz = ss(nx) * ss(ny) * zspan;
        *out = p;
    });
}

extern "C" int tw_slab_partition(int64_t nz, int rank, int nranks, int64_t* z_begin,
                                 int64_t* z_end) {
    return tw::guarded([&] {
        if (nranks < 1 || rank < 0 || rank >= nranks) tw::config_error("bad rank / world size");
        if (nz < nranks) tw::config_error("fewer planes than ranks");
        *z_begin = nz * rank / nranks;
        *z_end = nz * (rank + 1) / nranks;
    });
}

namespace tw {

// The x-staged form the CG's K1 reads (EllView::cols16), built from the
// int32 columns:
//  * a stencil matrix or z-slab with nx % 32 == 0: every slice is one x-line
//    segment and its 9 runs follow from the geometry (stage_run_start);
//  * any other matrix (stencils with nx % 32 != 0, tw_ell_from_csr): a
//    per-slice run table -- run 4 the window of the slice's own rows, the
//    other 8 cover the remaining columns greedily -- when every slice's
//    columns fit in 9 runs (any 27-point stencil does: the rows of a slice
//    are contiguous, so each (dz, dy) neighbour offset spans 34 columns).
// A matrix that does not fit stays unstaged (the gather K1 reads it).
static void build_x_staged(tw_ell* A, cudaStream_t s) {
    const tw_ell_info_t& in = A->info;
    if (A->cols16 || in.n_rows == 0 || in.max_width <= 0) return;
    if (spmv_staged_smem_bytes(static_cast<int>(in.max_width)) + 2048 > 227 * 1024) return;
    const bool stencil = in.nx > 0 && in.nx % 32 == 0;
    const int64_t ents = in.ell_entries;
    unsigned* bad = nullptr;
    TW_CUDA(cudaMalloc(&A->cols16, sizeof(uint16_t) * static_cast<size_t>(ents + 64)));
    if (!stencil)
        TW_CUDA(cudaMalloc(&A->runs, sizeof(int32_t) * kStageRuns * static_cast<size_t>(in.n_slices)));
    TW_CUDA(cudaMalloc(&bad, sizeof(unsigned)));
    TW_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned), s));
    if (stencil) {
        launch_stencil_cols16(A->view(), A->cols16, bad, s); // reads the 32-bit columns
    } else {
        EllView v = A->view();
        v.cols16 = nullptr; // not built yet
        launch_csr_runs(v, A->runs, A->cols16, bad, s);
    }
    unsigned hbad = 0;
    TW_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    TW_CUDA(cudaStreamSynchronize(s));
    cudaFree(bad);
    if (hbad) { // not representable: stay unstaged
        cudaFree(A->cols16);
        cudaFree(A->runs);
        A->cols16 = nullptr;
        A->runs = nullptr;
    }
}

static void drop_x_staged(tw_ell* A) {
    cudaFree(A->cols16);
    cudaFree(A->runs);
    A->cols16 = nullptr;
    A->runs = nullptr;
}

// gen_stencil_matrix (csr.cpp:29-59) for the slab [z_begin, z_end).
static tw_ell* gen_stencil(tw_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, int64_t zb,
                           int64_t ze) {
    tw_slab_t sp;
    if (int rc = tw_slab_plan(nx, ny, nz, zb, ze, &sp); rc != TW_OK) throw Error(rc, g_last_error);
    if (sp.x_len > std::numeric_limits<int32_t>::max())
        config_error("slab too large for 32-bit local column indices (" + std::to_string(sp.x_len) +
                     " columns); split it over more ranks");
    auto* A = new tw_ell;
    A->ctx = ctx;
    tw_ell_info_t& in = A->info;
    in.nx = nx;
    in.ny = ny;
    in.nz = nz;
    in.z_begin = zb;
    in.z_end = ze;
    in.n_global = nx * ny * nz;
    in.n_rows = sp.n_rows;
    in.row_offset = sp.row_offset;
    in.col_offset = sp.col_offset;
    in.x_len = sp.x_len;
    in.nnz = sp.nnz;
    A->diag_shift = sp.diag_shift;
    const int64_t n_slices = (in.n_rows + 31) / 32;
    cudaStream_t s = ctx->compute;
    int64_t* widths = nullptr;
    try {
        TW_CUDA(cudaMalloc(&widths, sizeof(int64_t) * std::max<int64_t>(n_slices, 1)));
        launch_stencil_widths(nx, ny, nz, in.row_offset, in.n_rows, n_slices, widths,
                              ctx->cfg.stream_blocks, s);
        finish_ell(A, widths, n_slices, s);
        // nx % 32 == 0: the fill writes the closed-form x-staged columns in
        // the same pass (otherwise build_x_staged adds a run table)
        if (nx % 32 == 0 &&
            spmv_staged_smem_bytes(static_cast<int>(in.max_width)) + 2048 <= 227 * 1024)
            TW_CUDA(cudaMalloc(&A->cols16, sizeof(uint16_t) * static_cast<size_t>(in.ell_entries + 64)));
        launch_stencil_fill(nx, ny, nz, in.row_offset, in.col_offset, in.n_rows, n_slices,
                            A->slice_off, A->vals, A->cols, A->cols16, ctx->cfg.stream_blocks, s);
#ifdef TW_CHECKS
        launch_ell_check(A->view(), s);
#endif
        build_x_staged(A, s);
        TW_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
        cudaFree(widths);
        free_ell(A);
        throw;
    }
    cudaFree(widths);
    return A;
}

// CsrMatrix::validate (csr.cpp:13-27) then device conversion.
static tw_ell* from_csr(tw_ctx* ctx, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                        const double* values) {
    if (n < 0 || !row_ptr) config_error("csr: row_ptr must hold n+1 offsets");
    if (row_ptr[0] != 0) config_error("csr: row_ptr must start at 0");
    for (int64_t i = 0; i < n; ++i)
        if (row_ptr[i] > row_ptr[i + 1])
            config_error("csr: row_ptr decreases at row " + std::to_string(i));
    const int64_t nnz = row_ptr[n];
    for (int64_t k = 0; k < nnz; ++k)
        if (col_idx[k] < 0 || col_idx[k] >= n)
            config_error("csr: column index " + std::to_string(col_idx[k]) + " out of range");
    if (n > std::numeric_limits<int32_t>::max())
        config_error("csr: more rows than 32-bit column indices address");
    auto* A = new tw_ell;
    A->ctx = ctx;
    tw_ell_info_t& in = A->info;
    in.n_global = n;
    in.n_rows = n;
    in.z_end = 0;
    in.x_len = n;
    in.nnz = nnz;
    const int64_t n_slices = (n + 31) / 32;
    cudaStream_t s = ctx->compute;
    int64_t *d_rp = nullptr, *d_ci = nullptr, *widths = nullptr;
    double* d_v = nullptr;
    try {
        TW_CUDA(cudaMalloc(&d_rp, sizeof(int64_t) * (n + 1)));
        TW_CUDA(cudaMalloc(&d_ci, sizeof(int64_t) * std::max<int64_t>(nnz, 1)));
        TW_CUDA(cudaMalloc(&d_v, sizeof(double) * std::max<int64_t>(nnz, 1)));
        TW_CUDA(cudaMalloc(&widths, sizeof(int64_t) * std::max<int64_t>(n_slices, 1)));
        copy_h2d(ctx, d_rp, row_ptr, sizeof(int64_t) * (n + 1), s);
        if (nnz) {
            copy_h2d(ctx, d_ci, col_idx, sizeof(int64_t) * nnz, s);
            copy_h2d(ctx, d_v, values, sizeof(double) * nnz, s);
        }
        launch_csr_widths(d_rp, n, n_slices, widths, ctx->cfg.stream_blocks, s);
        finish_ell(A, widths, n_slices, s);
        launch_csr_fill(d_rp, d_ci, d_v, n, n_slices, A->slice_off, A->vals, A->cols,
                        ctx->cfg.stream_blocks, s);
#ifdef TW_CHECKS
        launch_ell_check(A->view(), s);
#endif
        build_x_staged(A, s);
        TW_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
        cudaFree(d_rp);
        cudaFree(d_ci);
        cudaFree(d_v);
        cudaFree(widths);
        free_ell(A);
        throw;
    }
    cudaFree(d_rp);
    cudaFree(d_ci);
    cudaFree(d_v);
    cudaFree(widths);
    return A;
}

// Rows [r0, r1) of A as CSR with global columns; row_ptr relative to r0
// (r1 - r0 + 1 entries).  Copies only the slices the range touches, so a
// matrix whose CSR does not fit host memory is exported a z-slab at a time.
// staged: decode the 16-bit x-staged columns (the form the CG's K1 reads)
// through the slices' run starts instead of reading the int32 columns.
static void to_csr_rows(const tw_ell* A, int64_t r0, int64_t r1, bool staged, int64_t* row_ptr,
                        int64_t* col_idx, double* values) {
    const tw_ell_info_t& in = A->info;
    if (r0 < 0 || r1 > in.n_rows || r0 > r1) contract_error("csr export row range out of bounds");
    if (staged && !A->cols16) contract_error("matrix has no x-staged form");
    row_ptr[0] = 0;
    if (r0 == r1) return;
    const int64_t s0 = r0 / 32, s1 = (r1 + 31) / 32;
    std::vector<int64_t> off(static_cast<size_t>(s1 - s0 + 1));
    TW_CUDA(cudaMemcpy(off.data(), A->slice_off + s0, sizeof(int64_t) * off.size(),
                       cudaMemcpyDeviceToHost));
    const int64_t e0 = off.front(), ents = off.back() - e0;
    std::vector<double> v(static_cast<size_t>(ents));
    std::vector<int32_t> c(staged ? 0 : static_cast<size_t>(ents));
    std::vector<uint16_t> c16(staged ? static_cast<size_t>(ents) : 0);
    std::vector<int32_t> runs(staged && A->runs ? static_cast<size_t>(kStageRuns * (s1 - s0)) : 0);
    if (!runs.empty())
        TW_CUDA(cudaMemcpy(runs.data(), A->runs + kStageRuns * s0, sizeof(int32_t) * runs.size(),
                           cudaMemcpyDeviceToHost));
    if (ents) {
        TW_CUDA(cudaMemcpy(v.data(), A->vals + e0, sizeof(double) * ents, cudaMemcpyDeviceToHost));
        if (staged)
            TW_CUDA(cudaMemcpy(c16.data(), A->cols16 + e0, sizeof(uint16_t) * ents,
                               cudaMemcpyDeviceToHost));
        else
            TW_CUDA(cudaMemcpy(c.data(), A->cols + e0, sizeof(int32_t) * ents,
                               cudaMemcpyDeviceToHost));
    }
    int64_t k = 0;
    for (int64_t row = r0; row < r1; ++row) {
        const int64_t s = row / 32;
        const int lane = static_cast<int>(row % 32);
        const int64_t base = off[s - s0] - e0;
        const int w = static_cast<int>((off[s - s0 + 1] - off[s - s0]) / 32);
        bool padded = false;
        for (int e = 0; e < w; ++e) {
            int64_t col;
            if (staged) {
                const uint16_t j = c16[static_cast<size_t>(base + ell_c16_pos(e, lane, w))];
                const int r = j / kStageRunLen;
                const int64_t st =
                    runs.empty() ? stage_run_start(s, r, in.nx, in.ny, in.nz, in.row_offset,
                                                   in.col_offset)
                                 : runs[static_cast<size_t>((s - s0) * kStageRuns + r)];
                col = j == kStagePad ? -1 : st + j % kStageRunLen;
            } else {
                col = c[static_cast<size_t>(base + ell_col_pos(e, lane, w))];
            }
            if (col < 0) {
                padded = true;
                continue;
            }
            if (padded) contract_error("ELL row " + std::to_string(row) + " has an entry after padding");
            col_idx[k] = col + in.col_offset;
            values[k] = v[static_cast<size_t>(base + ell_val_pos(e, lane, w))];
            ++k;
        }
        row_ptr[row - r0 + 1] = k;
    }
}

static void to_csr(const tw_ell* A, int64_t* row_ptr, int64_t* col_idx, double* values) {
    to_csr_rows(A, 0, A->info.n_rows, false, row_ptr, col_idx, values);
}

void tile_plan(const tw_ell* A, int tiles, std::vector<int64_t>& r0, std::vector<int64_t>& r1,
               std::vector<int64_t>& lo, std::vector<int64_t>& hi) {
    const int64_t n = A->info.n_rows;
    if (tiles < 1) config_error("tile plan needs at least one tile");
    if (tiles > n) config_error("more tiles than matrix rows");
    tw_ctx* ctx = A->ctx;
    cudaStream_t s = ctx->compute;
    unsigned long long* mm = nullptr;
    TW_CUDA(cudaMalloc(&mm, sizeof(unsigned long long) * 2 * tiles));
    std::vector<unsigned long long> init(static_cast<size_t>(2 * tiles));
    for (int t = 0; t < tiles; ++t) {
        init[2 * t] = std::numeric_limits<unsigned long long>::max();
        init[2 * t + 1] = 0;
    }
    r0.resize(tiles);
    r1.resize(tiles);
    lo.resize(tiles);
    hi.resize(tiles);
    try {
        TW_CUDA(cudaMemcpyAsync(mm, init.data(), sizeof(unsigned long long) * 2 * tiles,
                                cudaMemcpyHostToDevice, s));
        for (int t = 0; t < tiles; ++t) {
            r0[t] = n * t / tiles;
            r1[t] = n * (t + 1) / tiles;
            launch_band(A->view(), r0[t], r1[t], mm + 2 * t, ctx->cfg.stream_blocks, s);
        }
        TW_CUDA(cudaMemcpyAsync(init.data(), mm, sizeof(unsigned long long) * 2 * tiles,
                                cudaMemcpyDeviceToHost, s));
        TW_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
        cudaFree(mm);
        throw;
    }
    cudaFree(mm);
    for (int t = 0; t < tiles; ++t) {
        if (init[2 * t] == std::numeric_limits<unsigned long long>::max()) {
            // empty tile: band collapses onto its first row (cg.cpp:364-367)
            lo[t] = hi[t] = r0[t] + A->diag_shift;
        } else {
            lo[t] = static_cast<int64_t>(init[2 * t]);
            hi[t] = static_cast<int64_t>(init[2 * t + 1]);
        }
    }
}

// xorshift64 jump-ahead: the step is linear over GF(2); columns[j] is the
// image of bit j.
struct Gf2 {
    uint64_t col[64];
    static Gf2 step() {
        Gf2 m;
        for (int j = 0; j < 64; ++j) {
            uint64_t s = 1ull << j;
            s ^= s << 13;
            s ^= s >> 7;
            s ^= s << 17;
            m.col[j] = s;
        }
        return m;
    }
    static Gf2 identity() {
        Gf2 m;
        for (int j = 0; j < 64; ++j) m.col[j] = 1ull << j;
        return m;
    }
    uint64_t apply(uint64_t v) const {
        uint64_t r = 0;
        for (int j = 0; j < 64; ++j)
            if (v >> j & 1) r ^= col[j];
        return r;
    }
    Gf2 mul(const Gf2& b) const { // this * b
        Gf2 m;
        for (int j = 0; j < 64; ++j) m.col[j] = apply(b.col[j]);
        return m;
    }
    static Gf2 power(uint64_t e) {
        Gf2 r = identity(), b = step();
        while (e) {
            if (e & 1) r = b.mul(r);
            b = b.mul(b);
            e >>= 1;
        }
        return r;
    }
};

static void rhs_xorshift(tw_ctx* ctx, uint64_t seed, int64_t first, int64_t count, double* out,
                         cudaStream_t s) {
    if (first < 0 || count < 0) contract_error("rhs: negative range");
    if (count == 0) return;
    const int64_t chunk = 1024;
    const int64_t nchunks = (count + chunk - 1) / chunk;
    std::vector<uint64_t> st(static_cast<size_t>(nchunks));
    const Gf2 jump = Gf2::power(static_cast<uint64_t>(chunk));
    uint64_t cur = Gf2::power(static_cast<uint64_t>(first)).apply(seed);
    for (int64_t c = 0; c < nchunks; ++c) {
        st[static_cast<size_t>(c)] = cur;
        cur = jump.apply(cur);
    }
    uint64_t* d = nullptr;
    TW_CUDA(cudaMalloc(&d, sizeof(uint64_t) * nchunks));
    try {
        TW_CUDA(cudaMemcpyAsync(d, st.data(), sizeof(uint64_t) * nchunks, cudaMemcpyHostToDevice, s));
        launch_rhs_xorshift(d, chunk, count, 0, out, ctx->cfg.stream_blocks, s);
        TW_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
        cudaFree(d);
        throw;
    }
    cudaFree(d);
}

} // namespace tw

using namespace tw;

extern "C" {

const char* tw_last_error_string(void) { return g_last_error.c_str(); }
int tw_abi_version(void) { return TW_ABI_VERSION; }

int tw_ctx_create(int device, unsigned cap, tw_ctx** out) {
    return guarded([&] {
        if (!out) contract_error("null out pointer");
        if (cap < 1) config_error("stream pool capacity must be at least 1");
        int ndev = 0;
        TW_CUDA(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev)
            config_error("device " + std::to_string(device) + " not present (" + std::to_string(ndev) + ")");
        TW_CUDA(cudaSetDevice(device));
        auto c = std::make_unique<tw_ctx>();
        c->device = device;
        TW_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
        int major = 0, minor = 0;
        TW_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
        TW_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
        if (major != 10 || minor != 0)
            config_error("libtw_hpccg is built for sm_100a (B200); device is sm_" +
                         std::to_string(major) + std::to_string(minor));
        c->cfg = query_launch_cfg(c->sm_count);
        TW_CUDA(cudaStreamCreateWithFlags(&c->compute, cudaStreamNonBlocking));
        TW_CUDA(cudaStreamCreateWithFlags(&c->comm, cudaStreamNonBlocking));
        c->pool.init(device, cap);
        c->red_blocks = std::max({c->cfg.spmv_blocks, c->cfg.stream_blocks, c->cfg.tma_blocks});
        *out = c.release();
    });
}

int tw_ctx_destroy(tw_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaDeviceSynchronize();
        drop_solve_cache(ctx, nullptr);
        for (int i = 0; i < 2; ++i) {
            if (ctx->stage[i]) cudaFreeHost(ctx->stage[i]);
            if (ctx->stage_ev[i]) cudaEventDestroy(ctx->stage_ev[i]);
        }
        if (ctx->ta) ctx->ta->poll_now(); // fire what completed, then stop the poller
        ctx->ta.reset();
        if (ctx->nccl_comm && nccl().CommDestroy) nccl().CommDestroy(ctx->nccl_comm);
        ctx->pool.destroy();
        cudaStreamDestroy(ctx->compute);
        cudaStreamDestroy(ctx->comm);
        for (auto& kv : ctx->red) {
            cudaFree(kv.second.block_part);
            cudaFree(kv.second.ticket);
        }
        delete ctx;
        (void)cudaGetLastError();
    });
}

int tw_ctx_compute_stream(tw_ctx* ctx, void** s) {
    return guarded([&] {
        check_ctx(ctx);
        *s = ctx->compute;
    });
}

int tw_ctx_synchronize(tw_ctx* ctx) {
    return guarded([&] {
        check_ctx(ctx);
        TW_CUDA(cudaSetDevice(ctx->device));
        TW_CUDA(cudaDeviceSynchronize());
    });
}

int tw_ctx_device_info(tw_ctx* ctx, int* device, int* sm_count) {
    return guarded([&] {
        check_ctx(ctx);
        if (device) *device = ctx->device;
        if (sm_count) *sm_count = ctx->sm_count;
    });
}

int tw_comm_unique_id(unsigned char id_out[128]) {
    return guarded([&] {
        ncclUniqueId id;
        TW_NCCL(nccl().GetUniqueId(&id));
        static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
        std::memcpy(id_out, &id, 128);
    });
}

int tw_ctx_init_comm(tw_ctx* ctx, int rank, int nranks, const unsigned char id[128]) {
    return guarded([&] {
        check_ctx(ctx);
        if (nranks < 1 || rank < 0 || rank >= nranks) config_error("bad rank / world size");
        if (ctx->nccl_comm) contract_error("communicator already initialised");
        if (ctx->emulated) contract_error("context is an emulated rank");
        ctx->rank = rank;
        ctx->nranks = nranks;
        // a 1-rank communicator is allowed: it runs the distributed code path
        ncclUniqueId uid;
        std::memcpy(&uid, id, 128);
        TW_CUDA(cudaSetDevice(ctx->device));
        TW_NCCL(nccl().CommInitRank(&ctx->nccl_comm, nranks, uid, rank));
    });
}

int tw_ctx_init_emulated_rank(tw_ctx* ctx, int rank, int nranks) {
    return guarded([&] {
        check_ctx(ctx);
        if (nranks < 1 || rank < 0 || rank >= nranks) config_error("bad rank / world size");
        if (ctx->nccl_comm) contract_error("context already has an NCCL communicator");
        ctx->rank = rank;
        ctx->nranks = nranks;
        ctx->emulated = true;
    });
}

int tw_ctx_comm_info(tw_ctx* ctx, int* rank, int* nranks) {
    return guarded([&] {
        check_ctx(ctx);
        if (rank) *rank = ctx->rank;
        if (nranks) *nranks = ctx->nranks;
    });
}

// ------------------------------------------------ streams and events
// The reference's QueuePool / sim::Device stream-event calls / TaskAware
// (task_aware.cpp:43-60, 122-166; sim_device.hpp:101-123) over real CUDA
// streams and events.

int tw_stream_acquire(tw_ctx* ctx, void** stream) {
    return guarded([&] {
        check_ctx(ctx);
        if (!stream) contract_error("null stream out");
        *stream = ctx->pool.stream(ctx->pool.acquire());
    });
}

int tw_stream_release(tw_ctx* ctx, void* stream) {
    return guarded([&] {
        check_ctx(ctx);
        const int i = ctx->pool.index_of(static_cast<cudaStream_t>(stream));
        if (i < 0) contract_error("not a stream of this context's pool");
        ctx->pool.release(i);
    });
}

int tw_event_create(void** ev) {
    return guarded([&] {
        if (!ev) contract_error("null event out");
        cudaEvent_t e;
        TW_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        *ev = e;
    });
}

int tw_event_destroy(void* ev) {
    return guarded([&] {
        if (!ev) contract_error("null event");
        TW_CUDA(cudaEventDestroy(static_cast<cudaEvent_t>(ev)));
    });
}

int tw_event_record(void* ev, void* stream) {
    return guarded([&] {
        if (!ev) contract_error("null event");
        TW_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(ev), static_cast<cudaStream_t>(stream)));
    });
}

int tw_event_query(void* ev, int* done) {
    return guarded([&] {
        if (!ev || !done) contract_error("null event or out");
        const cudaError_t q = cudaEventQuery(static_cast<cudaEvent_t>(ev));
        if (q == cudaErrorNotReady) {
            *done = 0;
            return;
        }
        TW_CUDA(q);
        *done = 1;
    });
}

int tw_event_wait(tw_ctx* ctx, void* ev) {
    return guarded([&] {
        check_ctx(ctx);
        if (!ev) contract_error("null event");
        TaskAware::wait_static(static_cast<cudaEvent_t>(ev));
    });
}

int tw_stream_wait_event(void* stream, void* ev) {
    return guarded([&] {
        if (!ev) contract_error("null event");
        TW_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), static_cast<cudaEvent_t>(ev), 0));
    });
}

int tw_event_bind_async(tw_ctx* ctx, void* ev, void (*done)(void* arg), void* arg) {
    return guarded([&] {
        check_ctx(ctx);
        if (!ev || !done) contract_error("null event or callback");
        {
            std::lock_guard lk(ctx->ta_mu);
            if (!ctx->ta) ctx->ta = std::make_unique<TaskAware>(ctx->device, 20e-6);
        }
        ctx->ta->bind_callback(static_cast<cudaEvent_t>(ev), done, arg);
    });
}

int tw_malloc(tw_ctx* ctx, void** ptr, int64_t bytes) {
    return guarded([&] {
        check_ctx(ctx);
        if (bytes < 0) contract_error("negative allocation");
        TW_CUDA(cudaSetDevice(ctx->device));
        TW_CUDA(cudaMalloc(ptr, static_cast<size_t>(std::max<int64_t>(bytes, 16))));
    });
}

int tw_free(tw_ctx* ctx, void* ptr) {
    return guarded([&] {
        check_ctx(ctx);
        TW_CUDA(cudaFree(ptr));
    });
}

int tw_malloc_host(void** ptr, int64_t bytes) {
    return guarded([&] { TW_CUDA(cudaMallocHost(ptr, static_cast<size_t>(std::max<int64_t>(bytes, 16)))); });
}

int tw_free_host(void* ptr) {
    return guarded([&] { TW_CUDA(cudaFreeHost(ptr)); });
}

int tw_memcpy(tw_ctx* ctx, void* dst, const void* src, int64_t bytes, void* stream) {
    return guarded([&] {
        check_ctx(ctx);
        if (bytes <= 0) return;
        TW_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDefault,
                                pick(ctx, stream)));
    });
}

int tw_gen_stencil_ell(tw_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, int64_t z_begin,
                       int64_t z_end, tw_ell** out) {
    return guarded([&] {
        check_ctx(ctx);
        TW_CUDA(cudaSetDevice(ctx->device));
        *out = gen_stencil(ctx, nx, ny, nz, z_begin, z_end);
    });
}

int tw_ell_from_csr(tw_ctx* ctx, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                    const double* values, tw_ell** out) {
    return guarded([&] {
        check_ctx(ctx);
        TW_CUDA(cudaSetDevice(ctx->device));
        *out = from_csr(ctx, n, row_ptr, col_idx, values);
    });
}

int tw_ell_info(const tw_ell* A, tw_ell_info_t* out) {
    return guarded([&] {
        check_ell(A);
        *out = A->info;
    });
}

int tw_ell_x_staged(const tw_ell* A, int* staged) {
    return guarded([&] {
        check_ell(A);
        if (!staged) contract_error("null out");
        *staged = A->cols16 ? 1 : 0;
    });
}

int tw_ell_set_x_staged(tw_ell* A, int enable, int* staged) {
    return guarded([&] {
        check_ell(A);
        TW_CUDA(cudaSetDevice(A->ctx->device));
        TW_CUDA(cudaStreamSynchronize(A->ctx->compute));
        drop_solve_cache(A->ctx, A); // their graphs / tables may hold the old form
        if (enable) build_x_staged(A, A->ctx->compute);
        else drop_x_staged(A);
        if (staged) *staged = A->cols16 ? 1 : 0;
    });
}

int tw_ell_to_csr(const tw_ell* A, int64_t* row_ptr, int64_t* col_idx, double* values) {
    return guarded([&] {
        check_ell(A);
        TW_CUDA(cudaSetDevice(A->ctx->device));
        to_csr(A, row_ptr, col_idx, values);
    });
}

int tw_ell_to_csr_rows(const tw_ell* A, int64_t row_begin, int64_t row_end, int staged,
                       int64_t* row_ptr, int64_t* col_idx, double* values) {
    return guarded([&] {
        check_ell(A);
        TW_CUDA(cudaSetDevice(A->ctx->device));
        to_csr_rows(A, row_begin, row_end, staged != 0, row_ptr, col_idx, values);
    });
}

int tw_ell_destroy(tw_ell* A) {
    return guarded([&] {
        if (!A) return;
        cudaSetDevice(A->ctx->device);
        drop_solve_cache(A->ctx, A); // tw_cg_solve's solvers of this matrix
        free_ell(A);
        (void)cudaGetLastError(); // teardown is best effort: leave no stale error behind
    });
}

int tw_spmv_range(const tw_ell* A, const double* x, double* y, int64_t r0, int64_t r1,
                  void* stream) {
    return guarded([&] {
        check_ell(A);
        if (r0 < 0 || r1 > A->info.n_rows || r0 > r1) contract_error("spmv row range out of bounds");
        if (r0 == r1) return;
        TW_CUDA(cudaSetDevice(A->ctx->device));
        RedScratch rs{};
        launch_spmv(A->view(), x, y, RowRange{r0, r1}, RowRange{0, 0}, false, rs,
                    Fin{FIN_NONE, nullptr, nullptr, nullptr}, A->ctx->cfg.spmv_blocks,
                    pick(A->ctx, stream));
    });
}

// exchange_externals for a z-slab: the first / last owned plane of x to the
// neighbours' ghost planes and theirs into ours, one NCCL send/recv group on
// `stream` (every rank of the communicator calls it).  Offsets from the slab
// plan, i.e. the same ones the solver's halo uses.
int tw_halo_exchange(const tw_ell* A, double* x, void* stream) {
    return guarded([&] {
        check_ell(A);
        tw_ctx* ctx = A->ctx;
        if (!ctx->nccl_comm) contract_error("halo exchange needs a communicator (tw_ctx_init_comm)");
        const tw_ell_info_t& in = A->info;
        if (in.nx == 0) contract_error("halo exchange needs a stencil slab (tw_gen_stencil_ell)");
        tw_slab_t sp{};
        if (int rc = tw_slab_plan(in.nx, in.ny, in.nz, in.z_begin, in.z_end, &sp); rc)
            throw Error(rc, g_last_error);
        if (sp.ghost_lo != (ctx->rank > 0) || sp.ghost_hi != (ctx->rank < ctx->nranks - 1))
            contract_error("slab z-range does not match this rank's position");
        TW_CUDA(cudaSetDevice(ctx->device));
        const auto& api = nccl();
        const size_t pl = static_cast<size_t>(in.nx * in.ny);
        cudaStream_t s = pick(ctx, stream);
        TW_NCCL(api.GroupStart());
        if (sp.ghost_lo) {
            TW_NCCL(api.Recv(x + sp.recv_lo, pl, ncclDouble, ctx->rank - 1, ctx->nccl_comm, s));
            TW_NCCL(api.Send(x + sp.send_lo, pl, ncclDouble, ctx->rank - 1, ctx->nccl_comm, s));
        }
        if (sp.ghost_hi) {
            TW_NCCL(api.Recv(x + sp.recv_hi, pl, ncclDouble, ctx->rank + 1, ctx->nccl_comm, s));
            TW_NCCL(api.Send(x + sp.send_hi, pl, ncclDouble, ctx->rank + 1, ctx->nccl_comm, s));
        }
        TW_NCCL(api.GroupEnd());
    });
}

int tw_spmv_dot(const tw_ell* A, const double* p, double* Ap, int64_t r0, int64_t r1,
                double* dot_dev, void* stream) {
    return guarded([&] {
        check_ell(A);
        if (r0 < 0 || r1 > A->info.n_rows || r0 > r1) contract_error("spmv row range out of bounds");
        tw_ctx* c = A->ctx;
        TW_CUDA(cudaSetDevice(c->device));
        cudaStream_t s = pick(c, stream);
        if (r0 == r1) {
            TW_CUDA(cudaMemsetAsync(dot_dev, 0, sizeof(double), s));
            return;
        }
        const RedScratch rs = ctx_red_scratch(c, s);
        launch_spmv(A->view(), p, Ap, RowRange{r0, r1}, RowRange{0, 0}, true, rs,
                    Fin{FIN_STORE, dot_dev, nullptr, nullptr}, c->cfg.spmv_blocks, s);
    });
}

int tw_dot_range(tw_ctx* ctx, const double* a, const double* b, int64_t i0, int64_t i1,
                 double* out_dev, void* stream) {
    return guarded([&] {
        check_ctx(ctx);
        if (i0 > i1) contract_error("dot range reversed");
        TW_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t s = pick(ctx, stream);
        if (i0 == i1) {
            TW_CUDA(cudaMemsetAsync(out_dev, 0, sizeof(double), s));
            return;
        }
        const RedScratch rs = ctx_red_scratch(ctx, s);
        launch_dot(a, b, i0, i1, rs, Fin{FIN_STORE, out_dev, nullptr, nullptr},
                   ctx->cfg.stream_blocks, s);
    });
}

// K2 / K3 as standalone operators (the fused forms of cg.cpp:380-389) with
// the scalar read on the device, so a caller's DAG never round-trips it.
int tw_update_xr_rr(tw_ctx* ctx, const double* alpha_dev, double* x, const double* p, double* r,
                    const double* Ap, int64_t i0, int64_t i1, double* rr_dev, void* stream) {
    return guarded([&] {
        check_ctx(ctx);
        if (!alpha_dev || !rr_dev) contract_error("null scalar pointer");
        if (i0 > i1) contract_error("update range reversed");
        TW_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t s = pick(ctx, stream);
        if (i0 == i1) {
            TW_CUDA(cudaMemsetAsync(rr_dev, 0, sizeof(double), s));
            return;
        }
        launch_update_xr(i0, i1, x, p, r, Ap, nullptr, ScalarSrc{alpha_dev, 0, nullptr},
                         ctx_red_scratch(ctx, s), Fin{FIN_STORE, rr_dev, nullptr, nullptr},
                         ctx->cfg.stream_blocks, s);
    });
}

int tw_update_p(tw_ctx* ctx, const double* beta_dev, const double* r, double* p, int64_t i0,
                int64_t i1, void* stream) {
    return guarded([&] {
        check_ctx(ctx);
        if (!beta_dev) contract_error("null scalar pointer");
        if (i0 > i1) contract_error("update range reversed");
        if (i0 == i1) return;
        TW_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t s = pick(ctx, stream);
        launch_update_p(i0, i1, r, p, nullptr, ScalarSrc{beta_dev, 0, nullptr},
                        ctx_red_scratch(ctx, s), nullptr, ctx->cfg.stream_blocks, s);
    });
}

int tw_waxpby_range(tw_ctx* ctx, double alpha, const double* x, double beta, const double* y,
                    double* w, int64_t i0, int64_t i1, void* stream) {
    return guarded([&] {
        check_ctx(ctx);
        if (i0 > i1) contract_error("waxpby range reversed");
        TW_CUDA(cudaSetDevice(ctx->device));
        launch_waxpby(alpha, x, beta, y, w, i0, i1, ctx->cfg.stream_blocks, pick(ctx, stream));
    });
}

int tw_make_tile_plan(const tw_ell* A, int tiles, int64_t* r0, int64_t* r1, int64_t* band_lo,
                      int64_t* band_hi) {
    return guarded([&] {
        check_ell(A);
        TW_CUDA(cudaSetDevice(A->ctx->device));
        std::vector<int64_t> a, b, lo, hi;
        tile_plan(A, tiles, a, b, lo, hi);
        for (int t = 0; t < tiles; ++t) {
            r0[t] = a[t];
            r1[t] = b[t];
            band_lo[t] = lo[t] + A->info.col_offset;
            band_hi[t] = hi[t] + A->info.col_offset;
        }
    });
}

int tw_rhs_xorshift(tw_ctx* ctx, uint64_t seed, int64_t first, int64_t count, double* out_dev,
                    void* stream) {
    return guarded([&] {
        check_ctx(ctx);
        TW_CUDA(cudaSetDevice(ctx->device));
        rhs_xorshift(ctx, seed, first, count, out_dev, pick(ctx, stream));
    });
}

int tw_rhs_splitmix(tw_ctx* ctx, uint64_t seed, int64_t first, int64_t count, double* out_dev,
                    void* stream) {
    return guarded([&] {
        check_ctx(ctx);
        if (first < 0 || count < 0) contract_error("rhs: negative range");
        TW_CUDA(cudaSetDevice(ctx->device));
        launch_rhs_splitmix(seed, first, count, out_dev, ctx->cfg.stream_blocks, pick(ctx, stream));
    });
}

} // extern "C"
