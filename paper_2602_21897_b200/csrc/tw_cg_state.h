// Solver state shared by the CG drivers (tw_cg.cpp: single-GPU monolithic
// and block-task DAG, graphs, the persistent dispatcher) and the multi-rank
// transports (tw_cg_dist.cpp: NCCL, NVLink peer, emulated rank groups).
// Internal header of libtw_hpccg; the C ABI is include/tw_hpccg.h.
#pragma once

#include <map>
#include <memory>
#include <vector>

#include "tw_dag_host.h"
#include "tw_objects.h"

using namespace tw; // internal header: tw_cg sits at global scope (C ABI type)

struct tw_cg {
    tw_ctx* ctx = nullptr;
    const tw_ell* A = nullptr;
    tw_cg_options opt{};
    tw_cg_options req{}; // the options as requested (tw_cg_solve's cache key)
    int max_iters = 0;
    int T = 1;
    int P = 1;
    bool dist = false; // communicator attached: halo + rank-ordered allgathers
    int64_t n = 0, plane = 0, x_len = 0, diag_shift = 0;
    bool glo = false, ghi = false;
    tw_slab_t slab{}; // z-slab geometry (multi-rank)
    // NVLink peer transport (tw_peer.cu): own receive window, links to the
    // other ranks, device copy of the links, IPC mappings to release
    bool peer = false;
    PeerWindow* win = nullptr;
    PeerLinks links{};
    PeerLinks* d_links = nullptr;
    // paired x updates: the same links with the neighbours' pair-buffer
    // ghost planes as the halo targets (the K3 that writes the pair buffer)
    PeerLinks links2{};
    PeerLinks* d_links2 = nullptr;
    unsigned long long ping_seq = 0; // transport-check round (same on every rank)
    std::vector<void*> ipc_mapped;
    unsigned epoch = 0; // set_rhs count

    double* x = nullptr;
    double* r = nullptr;      // r_base + 16: 2+ doubles of slack each side (staged runs of r)
    double* r_base = nullptr;
    double* p_base = nullptr;
    double* p2_base = nullptr; // pair buffer (x_pairs; inside the p_base allocation): p_k+1 between the two K3s of a pair
    double* p2_local = nullptr;
    double* p2_owned = nullptr;
    double* p_local = nullptr; // x_len entries: [ghost lo] owned [ghost hi]
    double* p_owned = nullptr;
    double* Ap = nullptr;
    CgScalars* sc = nullptr;
    double* history = nullptr;
    double* parts = nullptr;
    double* block_parts = nullptr;
    unsigned* tickets = nullptr;
    unsigned* tile_tickets = nullptr; // [2]: the folded alpha / beta_res (FIN_TILES)
    int maxg = 0;

    // partial slots (offsets into parts)
    double *pa = nullptr, *rrp = nullptr, *pm = nullptr, *send_a = nullptr, *send_b = nullptr,
           *recv_a = nullptr, *recv_b = nullptr, *send_r = nullptr, *recv_r = nullptr;

    std::vector<int64_t> t_r0, t_r1, t_lo, t_hi; // tile plan (local rows / local columns)
    DagSpec dag;                                 // inputs of the logical DAG
    std::vector<LTask> ltasks;                   // one iteration's logical tasks (template)
    std::vector<PNode> nodes;                    // one iteration's physical nodes
    std::vector<cudaEvent_t> ev[2];              // per node, by iteration parity
    std::vector<cudaEvent_t> tail_ev;            // per pool stream + comm
    cudaEvent_t fork_ev = nullptr, halo_ev = nullptr, pready_ev = nullptr;
    cudaEvent_t ag_in_ev = nullptr, ag_out_ev = nullptr;

    cudaGraphExec_t graph = nullptr;
    std::map<int, cudaGraphExec_t> timed_graphs; // K iterations + per-kernel timing events
    std::map<int, cudaGraphExec_t> chunk_graphs; // up to kGraphChunk iterations, untimed
    bool x_k3 = false; // x += alpha p_old in K3, not K2 (decided at creation)
    bool x_pairs = false; // ... once per pair of iterations (one rank; monolithic, tasks on streams)
    // programmatic chain: its x/r phase's first tile launched plainly (tiles of
    // 3M rows and more, where a programmatic x/r gate behind the SpMV tiles
    // costs 2 %; profiles/r02_ab_chain.md)
    bool chain_plain_upd = false;
    int enqueued = 0;
    // per-kernel timing (monolithic, no graph): 4 events per timed iteration
    bool timing = false;
    std::vector<cudaEvent_t> tev;
    int timed = 0;
    std::vector<cudaEvent_t> iter_ev; // iteration-end timing events (marks on)
    // persistent dispatcher (TW_DISPATCH_PERSISTENT): flattened K-iteration
    // DAG tables, cached per K
    struct DagTable {
        int ntasks = 0, nchunks = 0;
        DagTask* d_tasks = nullptr;
        int* d_chunk_task = nullptr;
        int* d_succ = nullptr;
        int* d_npred = nullptr;
        int* d_remaining = nullptr;
        unsigned* d_chunk_done = nullptr;
        double* d_chunk_part = nullptr;
    };
    std::map<int, DagTable> dag_tables;
    int dag_grid = 0;
    unsigned* d_ticket = nullptr;
    unsigned long long* d_stamps = nullptr;
    double t0 = 0.0;
    std::vector<double> marks;
    std::vector<char> mark_real; // persistent dispatch: the poller marked this iteration
    std::unique_ptr<TaskAware> ta;

    RedScratch slot(int i) const {
        return RedScratch{block_parts + static_cast<size_t>(i) * maxg, tickets + 4 * i};
    }
    // K1's view of A; l2_keep overrides the x-run L2 policy of the staged K1
    // tasks variant, one rank, up to 4 tiles: alpha / beta_res folded into
    // the last tile kernel of their phase (no combine launch between the
    // phases; 128^3, 4 tiles: streams 132.7 -> 130.0 us).  With more tiles
    // the empty join node turns into T x T edges between the phases (a
    // captured graph has no node left to join on): 16 tiles 193 -> 212 us,
    // 64 tiles 330 -> 523 us as one 16-iteration graph (profiles/
    // r02_ab_tasks_executors.md), so there the combine kernels stay.
#ifndef TW_FOLD_TILES
#define TW_FOLD_TILES 4 // most tiles folded
#endif
    bool fold_scalars() const {
        return opt.variant == TW_CG_TASKS && !dist && T <= TW_FOLD_TILES;
    }
    Fin tile_fin(double* parts, int t, int then, unsigned* ticket) const {
        Fin f{FIN_STORE, parts + t, nullptr, nullptr};
        if (fold_scalars()) {
            f.mode = FIN_TILES;
            f.sc = sc;
            f.history = history;
            f.tparts = parts;
            f.ntiles = T;
            f.then = then;
            f.tticket = ticket;
        }
        return f;
    }
    EllView view() const {
        EllView v = A->view();
        if (v.cols16 && opt.l2_keep == TW_L2KEEP_ON) v.sx_keep = 1;
        if (v.cols16 && opt.l2_keep == TW_L2KEEP_OFF) v.sx_keep = 0;
        return v;
    }
    // Across ranks every node that calls NCCL (the halo; alpha / beta_res:
    // combine, allgather, combine) runs on the comm stream, so one rank's
    // collectives are issued in program order on one stream -- the order
    // every rank shares (halo(i) < alpha(i) < beta_res(i) < halo(i+1)).
    cudaStream_t node_stream(const PNode& nd) const {
        if (nd.kind == PK_HALO) return ctx->comm;
        const unsigned C = ctx->pool.capacity();
        if (nd.kind == PK_ALPHA || nd.kind == PK_BETA) return dist ? ctx->comm : ctx->pool.stream(0);
        return ctx->pool.stream(static_cast<int>(static_cast<unsigned>(nd.tile) % C));
    }
};

namespace tw {
namespace cgi {

// tw_cg.cpp
bool x_in_k3(const tw_cg* cg);
void build_schedule(tw_cg* cg);
int launch_blocks(const tw_cg* cg, bool spmv);
cudaEvent_t tmark(tw_cg* cg, int k);
void record(cudaEvent_t e, cudaStream_t s);
#ifndef TW_XPAIRS_AUTO
#define TW_XPAIRS_AUTO 1 // TW_XUPD_AUTO pairs the x updates wherever it puts them in K3
#endif
enum { XPH_SINGLE = 0, XPH_DEFER = 1, XPH_PAIR = 2 };
int x_phase(const tw_cg* cg, int i, int k);
void enqueue_mono(tw_cg* cg, int xph = XPH_SINGLE);
int tile_share(const tw_cg* cg);
void launch_node(tw_cg* cg, const PNode& nd, cudaStream_t st, int xph = XPH_SINGLE,
                 int chain_role = -1);
void fork_streams(tw_cg* cg);
void join_streams(tw_cg* cg);
void enqueue_tasks(tw_cg* cg, int parity, bool first, int xph = XPH_SINGLE);
void enqueue_iteration_body(tw_cg* cg, int parity, bool first, int xph = XPH_SINGLE);
void build_graph(tw_cg* cg);
constexpr int kGraphChunk = 16;
cudaGraphExec_t build_chunk_graph(tw_cg* cg, int c);
void free_cg(tw_cg* cg);
tw_cg* create_cg(tw_ctx* ctx, const tw_ell* A, const tw_cg_options* o, int max_iters);
void set_rhs_prefix(tw_cg* cg, const double* b, bool on_device, cudaStream_t s);
void reset_solve_state(tw_cg* cg);
void set_rhs(tw_cg* cg, const double* b, bool on_device);
cudaEvent_t iter_event(tw_cg* cg, int i);
int64_t dag_spmv_chunk_slices(const tw_cg* cg);
int64_t dag_vec_chunk_rows(const tw_cg* cg);
void build_dag_table(tw_cg** g, int P, int k);
void enqueue_persistent(tw_cg** g, int P, int k);
void iterate(tw_cg* cg, int k);
void wait_cg(tw_cg* cg);

// tw_cg_dist.cpp
void allgather1(tw_cg* cg, const double* send, double* recv, cudaStream_t s);
void halo_exchange(tw_cg* cg, cudaStream_t s, double* p_local = nullptr);
void dist_spmv_interior(tw_cg* cg, cudaStream_t s, const double* p_local = nullptr);
void dist_spmv_boundary(tw_cg* cg, cudaStream_t s, const double* p_local = nullptr);
void dist_update_xr(tw_cg* cg, cudaStream_t s);
void dist_update_p(tw_cg* cg, cudaStream_t s, int xph = XPH_SINGLE);
bool peer_k1_fused(const tw_cg* cg);
void peer_spmv(tw_cg* cg, cudaStream_t s, int xph = XPH_SINGLE);
void peer_update_xr(tw_cg* cg, cudaStream_t s);
void peer_update_p(tw_cg* cg, cudaStream_t s, int xph = XPH_SINGLE);
void alloc_window(tw_cg* cg);
void finish_links(tw_cg* cg);
void group_check(tw_cg** g, int P);
void loopback_allgather(tw_cg** g, int P, double* tw_cg::*send, double* tw_cg::*recv,
                        cudaStream_t s);
void loopback_halo(tw_cg** g, int P, cudaStream_t s, int xph = XPH_SINGLE);
void group_join(tw_cg** g, int P, cudaStream_t s);
void group_enable_peer(tw_cg** g, int P);
void group_set_rhs(tw_cg** g, int P, const double* const* b, bool on_device);
void group_iterate(tw_cg** g, int P, int k);
void group_iterate_concurrent(tw_cg** g, int P, int k, int jitter);

} // namespace cgi
} // namespace tw
