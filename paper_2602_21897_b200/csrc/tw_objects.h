// Host-side objects behind the opaque C handles.
#pragma once

#include <atomic>
#include <condition_variable>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <string>
#include <thread>
#include <vector>

#include "tw_internal.h"
#include "tw_nccl.h"

namespace tw {

// Fixed-capacity stream pool with FIFO acquisition: the QueuePool of the
// reference (task_aware.hpp:80-109) over real cudaStream_t.  A caller that
// asks while every stream is out waits (host side) for the next release.
class StreamPool {
public:
    void init(int device, unsigned capacity);
    void destroy();
    int acquire();               // index into streams()
    void release(int idx);
    cudaStream_t stream(int idx) const { return streams_[static_cast<size_t>(idx)]; }
    int index_of(cudaStream_t s) const; // -1 if s is not a pool stream
    unsigned capacity() const { return static_cast<unsigned>(streams_.size()); }
    size_t outstanding() const;

private:
    std::vector<cudaStream_t> streams_;
    mutable std::mutex mu_;
    std::condition_variable cv_;
    std::deque<int> free_;
    std::vector<char> held_; // held_[i]: stream i is acquired (release checks it)
};

// Task-aware completion layer over CUDA events: the TACUDA mechanism of
// ta::TaskAware (task_aware.cpp:16-100).  bind() ties an event to a
// completion slot that the polling thread fills with the host time at which
// it first observed the event complete (bind_event_async semantics);
// wait() polls until an event completes, yielding the thread between polls
// (wait_transformed semantics).  Device-to-device ordering never goes
// through here: it is expressed as cudaStreamWaitEvent edges.
class TaskAware {
public:
    explicit TaskAware(int device, double poll_period_s) : device_(device), period_(poll_period_s) {}
    ~TaskAware();
    void bind(cudaEvent_t ev, double* slot, double t0);          // event owned, recycled
    void bind_callback(cudaEvent_t ev, void (*done)(void*), void* arg); // caller's event
    void wait(cudaEvent_t ev);
    static void wait_static(cudaEvent_t ev); // poll + yield until ev completes
    size_t pending() const;
    size_t polled() const { return polled_.load(); }
    size_t poll_now() { return poll_once(); }
    cudaEvent_t take_event();

private:
    void loop();
    size_t poll_once();
    struct Bind {
        cudaEvent_t ev;
        double* slot;
        double t0;
        void (*done)(void*);
        void* arg;
        bool owned;
    };
    void add(const Bind& b);
    int device_;
    double period_;
    mutable std::mutex mu_;
    std::condition_variable cv_;
    std::deque<Bind> binds_;
    std::vector<cudaEvent_t> spare_;
    std::thread th_;
    bool stop_ = false;
    bool started_ = false;
    std::atomic<size_t> polled_{0};
};

double host_seconds();

extern thread_local std::string g_last_error;

// Runs f, mapping exceptions onto ABI status codes (never throws).
template <typename F>
int guarded(F&& f) {
    try {
        f();
        return TW_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return TW_ERR_CONFIG;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return TW_ERR_CONTRACT;
    }
}

} // namespace tw

struct tw_ctx {
    int device = 0;
    int sm_count = 0;
    tw::LaunchCfg cfg{};
    cudaStream_t compute = nullptr;
    cudaStream_t comm = nullptr;
    tw::StreamPool pool;
    // scratch for standalone reductions (tw_dot_range / tw_spmv_dot), one per
    // stream: calls on one stream run in order, calls on different streams
    // may run at the same time (the reference's kernels may be called from
    // any worker, kernels.hpp:7-9) and must not share a ticket
    std::unordered_map<cudaStream_t, tw::RedScratch> red;
    int red_blocks = 0;
    std::mutex red_mu;
    // multi-GPU
    ncclComm_t nccl_comm = nullptr;
    int rank = 0;
    int nranks = 1;
    bool emulated = false; // rank of an emulated group on one device (no NCCL)
    // task-aware completion for tw_event_bind_async (lazily started poller)
    std::unique_ptr<tw::TaskAware> ta;
    std::mutex ta_mu;
    // two pinned staging buffers for pageable host <-> device copies
    // (tw::copy_h2d / copy_d2h), allocated on first use
    void* stage[2] = {nullptr, nullptr};
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};
    std::mutex stage_mu;
    // tw_cg_solve's solvers, kept per matrix between calls (the matrix's
    // destroy and the context's release drop them)
    std::map<const tw_ell*, tw_cg*> solve_cache;
    std::mutex solve_mu;
};

struct tw_ell {
    tw_ctx* ctx = nullptr;
    tw_ell_info_t info{};
    int64_t diag_shift = 0;
    int64_t* slice_off = nullptr;
    double* vals = nullptr;
    int32_t* cols = nullptr;
    uint16_t* cols16 = nullptr; // x-staged columns (stencil or z-slab, nx % 32 == 0), or null
    int32_t* runs = nullptr;    // run table of a staged CSR matrix (EllView::sx_runs), or null
    tw::EllView view() const {
        tw::EllView v{slice_off, vals, cols, info.n_rows, info.n_slices, diag_shift,
                      info.max_width, ctx->cfg.tma_blocks, info.x_len};
        if (cols16) {
            v.cols16 = cols16;
            v.sx_nx = info.nx;
            v.sx_ny = info.ny;
            v.sx_nz = info.nz;
            v.sx_row_off = info.row_offset;
            v.sx_col_off = info.col_offset;
            v.sx_keep = info.x_len <= (int64_t(1) << 23) ? 1 : 0;
            v.sx_runs = runs;
        }
        return v;
    }
};

namespace tw {
// Host <-> device copies of caller buffers (tw_runtime.cpp).  Pinned memory
// goes straight to the copy engine; pageable memory -- a reference caller's
// std::vector -- through the context's two pinned staging buffers, host
// threads filling (draining) one while the copy engine moves the other.
// copy_h2d returns once the source may be reused; copy_d2h once dst holds
// the data (both order on stream s).
void copy_h2d(tw_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t s);
void copy_d2h(tw_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t s);
void drop_solve_cache(tw_ctx* ctx, const tw_ell* A); // A == nullptr: every entry
// helpers shared across translation units
RedScratch ctx_red_scratch(tw_ctx* ctx, cudaStream_t s);
void tile_plan(const tw_ell* A, int tiles, std::vector<int64_t>& r0, std::vector<int64_t>& r1,
               std::vector<int64_t>& band_lo_local, std::vector<int64_t>& band_hi_local);
} // namespace tw
