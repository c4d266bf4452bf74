// CG drivers of libtw_hpccg: cg_monolithic and the cg_tasks block-task DAG
// (cg.cpp:166-447) re-expressed as CUDA streams, events and graphs, with all
// scalars resident on the device; the persistent DAG dispatcher's tables;
// the solver ABI.  Across ranks the iteration's phases come from
// tw_cg_dist.cpp (z-slab decomposition, NCCL or NVLink peer transport).
//
// Per iteration the device work is three HBM-bound kernels:
//   K1 spmv_pAp   Ap = A p, p.Ap            (spmv:i:t + dot_pAp:i:t)
//   K2 update_xr  x += a p, r -= a Ap, r.r  (x_up:i:t + r_up:i:t + dot_rr:i:t)
//   K3 update_p   p = r + b p               (p_up:i:t)
// with alpha:i / beta_res:i folded into the last block of K1 / K2 (one tile),
// into the last tile kernel of the phase (tiles, one rank), or run as one-warp
// combine kernels over the tile / rank partials (across ranks).
//
// The tasks variant keeps the reference's data-flow semantics: the depsys
// dependency rule infers the per-iteration logical DAG from the same byte-interval
// accesses spawn_iteration declares (cg.cpp:173-333); fused physical nodes
// inherit the union of their members' edges and become cudaStreamWaitEvent
// edges between pooled streams (or edges of a captured CUDA graph).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <optional>
#include <set>
#include <sstream>
#include <string>

#include "tw_cg_state.h"

namespace tw {
namespace cgi {

// The x update (x += alpha p_old) in K3 instead of K2: K3 reads p_old
// anyway, so the iteration moves 8 n bytes less from DRAM once the vectors
// no longer sit in L2 (measured, event-timed K2 + K3: 256^3 197.5 -> 179.7 us,
// 128^3 29.0 -> 29.6 us), hence from 4M rows per rank by default.  The
// placement changes no bit (each element's update is the same rounding).
bool x_in_k3(const tw_cg* cg) { return cg->x_k3; }

// Paired x updates (one rank, monolithic): x = (x + a_k p_k) + a_k+1 p_k+1
// in the second K3 of each pair of iterations, so x is read and written once
// per pair; the first K3 writes p_k+1 to a second buffer and keeps p_k.
// 4 n bytes less per iteration than the x update in every K3, no bit
// changes.  Measured per iteration (profiles/r02_ab_k2k3_sweep.md), K3
// every iteration / pairs / K2: 256^3 857-868 / 846-854 / 887-894 us,
// 128^3 114.0-114.5 / 113.4-113.8 / 116.9-117.1, 96^3 57.6-57.9 /
// 56.9-57.1 / 58.1-58.4, 64^3 29.0 / 28.7-28.8 / 28.4-28.6: pairs from
// 512k rows on such a solver.  The block-task DAG on streams / graphs (one
// rank) pairs them in its p-update tiles the same way: 256^3, 2 / 4 / 16
// tiles, 873-885 -> 859-872 us (streams), 868-874 -> 859-864 (4 tiles,
// chunked graphs), 941 -> 922 (16 tiles); 128^3 125.6 -> 123.5 (4 tiles,
// chunked graphs; 125.2 with x in the x/r tiles).  The persistent
// dispatcher pairs them where it moves x into the p updates, from 4M rows
// (256^3, 8 / 16 / 64 tiles: 888-892 -> 876-881 us; at 128^3 the x update in
// the x/r chunks stays best: 133 against 136 us either way).
static bool dag_pairs_fit(const tw_cg* cg);
// Across ranks (monolithic: the halo then alternates buffers too) every
// rank must make the same choice, so it rests on the global rows per rank.
static bool auto_pairs(const tw_cg* cg) {
    const int64_t rows = cg->dist ? cg->A->info.n_global / std::max(cg->P, 1) : cg->n;
    if (rows < (int64_t(1) << 19)) return false;
    if (cg->opt.variant == TW_CG_TASKS && cg->opt.dispatch == TW_DISPATCH_PERSISTENT)
        return rows >= (int64_t(1) << 22) && dag_pairs_fit(cg);
    return true;
}

static bool decide_x_in_k3(const tw_cg* cg) { // at solver creation
    const int xu = cg->opt.x_update;
    if (xu == TW_XUPD_K2) return false;
    if (xu == TW_XUPD_K3 || xu == TW_XUPD_K3_PAIRS) return true;
    return cg->n >= (int64_t(1) << 22) || (TW_XPAIRS_AUTO && auto_pairs(cg));
}

// The persistent dispatcher pairs them in its TMA update chunks, which need
// stages of >= 128 rows for 3 and 4 operand streams (else its register path
// runs, with single updates).
static bool dag_pairs_fit(const tw_cg* cg) {
    int sb, vb, cb;
    dag_smem_bytes(static_cast<int>(cg->A->info.max_width), cg->A->cols16 != nullptr, &sb, &vb, &cb);
    return ((sb / 24) & ~63) >= 128 && ((sb / 32) & ~63) >= 128;
}

static bool decide_x_pairs(const tw_cg* cg) {
    if (!cg->x_k3) return false;
    if (cg->opt.variant == TW_CG_TASKS && cg->opt.dispatch == TW_DISPATCH_PERSISTENT &&
        !dag_pairs_fit(cg))
        return false;
    if (cg->opt.x_update == TW_XUPD_K3_PAIRS) return true;
    return cg->opt.x_update == TW_XUPD_AUTO && TW_XPAIRS_AUTO && auto_pairs(cg);
}

// The x-update phase of iteration i of a run of k enqueued together: pairs
// inside the run, a single update for an odd run's last iteration, so x and
// p (in p_local) are current at the end of every run.
int x_phase(const tw_cg* cg, int i, int k) {
    if (!cg->x_pairs) return XPH_SINGLE;
    if (i & 1) return XPH_PAIR;
    return i + 1 < k ? XPH_DEFER : XPH_SINGLE;
}

// Physical predecessor lists from the logical DAG of iterations 0 and 1.
void build_schedule(tw_cg* cg) {
    build_logical(cg->dag, 0, cg->ltasks, &cg->nodes);
    const int L = static_cast<int>(cg->ltasks.size());
    std::vector<std::pair<int, int>> edges;
    std::vector<int> phys;
    logical_edges(cg->dag, 2, edges, nullptr, &phys);
    std::vector<std::set<int>> first(cg->nodes.size()), intra(cg->nodes.size()),
        cross(cg->nodes.size());
    for (auto [a, b] : edges) {
        const int pa = phys[static_cast<size_t>(a)], pb = phys[static_cast<size_t>(b)];
        const int ia = a / L, ib = b / L;
        if (ib == 0) {
            if (pa != pb) first[static_cast<size_t>(pb)].insert(pa);
        } else if (ia == 1) {
            if (pa != pb) intra[static_cast<size_t>(pb)].insert(pa);
        } else {
            cross[static_cast<size_t>(pb)].insert(pa);
        }
    }
    for (size_t j = 0; j < cg->nodes.size(); ++j) {
        cg->nodes[j].preds_first.assign(first[j].begin(), first[j].end());
        cg->nodes[j].preds_intra.assign(intra[j].begin(), intra[j].end());
        cg->nodes[j].preds_cross.assign(cross[j].begin(), cross[j].end());
        for (int p : cg->nodes[j].preds_first)
            if (p >= static_cast<int>(j)) contract_error("physical task order is not topological");
    }
}

int launch_blocks(const tw_cg* cg, bool spmv) {
    return spmv ? cg->ctx->cfg.spmv_blocks : cg->ctx->cfg.stream_blocks;
}

// Timing event k (0..3) of the current timed iteration, or null.
cudaEvent_t tmark(tw_cg* cg, int k) {
    if (!cg->timing) return nullptr;
    const size_t i = static_cast<size_t>(cg->timed) * 4 + static_cast<size_t>(k);
    while (cg->tev.size() <= i) {
        cudaEvent_t e;
        TW_CUDA(cudaEventCreate(&e));
        cg->tev.push_back(e);
    }
    return cg->tev[i];
}

// Timing marks: inside a stream capture a plain cudaEventRecord only forms
// graph edges, so the marks are captured as external event-record nodes.
void record(cudaEvent_t e, cudaStream_t s) {
    if (!e) return;
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    TW_CUDA(cudaStreamIsCapturing(s, &st));
    if (st == cudaStreamCaptureStatusActive)
        TW_CUDA(cudaEventRecordWithFlags(e, s, cudaEventRecordExternal));
    else
        TW_CUDA(cudaEventRecord(e, s));
}

// One monolithic iteration (cg_monolithic, cg.cpp:408-431) on the compute
// stream: K1 -> K2 -> K3 (x rides on K2 or on K3, x_in_k3); across ranks the
// SpMV is split so the interior rows overlap the halo exchange on the comm
// stream.
// Programmatic dependent launch in the one-rank chain (bit 0 K1, 1 K2, 2 K3).
// K1 only: its one 205 KB CTA per SM cannot co-reside with a full-occupancy
// K3 wave, so its blocks take each SM as K3's blocks leave it, stream their
// first matrix block and wait (griddepcontrol.wait) only before the x runs.
// 128^3: 114.1 -> 111.6 us per iteration, 256^3 842.7 -> 841.4-842.7; K2
// after K1 co-resides with K1 and loses (all three: 895 us at 256^3); the
// SpMV tiles of the tasks variant gain nothing (profiles/r02_ab_pdl.md).
#ifndef TW_MONO_PDL
#define TW_MONO_PDL 1
#endif
void enqueue_mono(tw_cg* cg, int xph) {
    cudaStream_t s = cg->ctx->compute;
    const EllView A = cg->view();
    const int bs = launch_blocks(cg, true), bv = launch_blocks(cg, false);
    const RedScratch rs = cg->slot(0);
    if (xph != XPH_SINGLE && !cg->x_pairs) contract_error("paired x update not enabled");
    if (!cg->dist) {
        // p_k of this iteration: in the pair buffer for the second of a pair
        double* pl = xph == XPH_PAIR ? cg->p2_local : cg->p_local;
        double* po = xph == XPH_PAIR ? cg->p2_owned : cg->p_owned;
        const Fin fa{FIN_ALPHA, nullptr, cg->sc, nullptr};
        record(tmark(cg, 0), s);
        const bool pdl1 = (TW_MONO_PDL & 1) && !cg->timing, pdl2 = (TW_MONO_PDL & 2) && !cg->timing,
                   pdl3 = (TW_MONO_PDL & 4) && !cg->timing;
        if (!launch_spmv_staged(A, pl, cg->Ap, RowRange{0, cg->n}, RowRange{0, 0}, RowRange{0, 0},
                                false, rs, fa, s, nullptr, 0, pdl1))
            launch_spmv(A, po, cg->Ap, RowRange{0, cg->n}, RowRange{0, 0}, true, rs, fa, bs, s);
        record(tmark(cg, 1), s);
        const bool xk3 = x_in_k3(cg);
        launch_update_xr(0, cg->n, xk3 ? nullptr : cg->x, po, cg->r, cg->Ap, cg->sc,
                         ScalarSrc{nullptr, 0}, rs, Fin{FIN_BETA, nullptr, cg->sc, cg->history}, bv,
                         s, pdl2);
        record(tmark(cg, 2), s);
        if (xph == XPH_DEFER) // p_k+1 into the pair buffer, p_k and x left as they are
            launch_update_p(0, cg->n, cg->r, cg->p2_owned, cg->sc, ScalarSrc{nullptr, 0}, rs,
                            cg->history, bv, s, nullptr, cg->p_owned, pdl3, nullptr);
        else if (xph == XPH_PAIR) // x gets a_k-1 p_k-1 + a_k p_k; p_k+1 back into p_owned
            launch_update_p(0, cg->n, cg->r, cg->p_owned, cg->sc, ScalarSrc{nullptr, 0}, rs,
                            cg->history, bv, s, nullptr, cg->p2_owned, pdl3, cg->x, cg->p_owned);
        else
            launch_update_p(0, cg->n, cg->r, cg->p_owned, cg->sc, ScalarSrc{nullptr, 0}, rs,
                            cg->history, bv, s, nullptr, nullptr, pdl3, xk3 ? cg->x : nullptr);
        record(tmark(cg, 3), s);
        if (cg->timing) ++cg->timed;
        return;
    }
    if (cg->peer) {
        record(tmark(cg, 0), s);
        peer_spmv(cg, s, xph);
        record(tmark(cg, 1), s);
        peer_update_xr(cg, s);
        record(tmark(cg, 2), s);
        peer_update_p(cg, s, xph);
        record(tmark(cg, 3), s);
        if (cg->timing) ++cg->timed;
        return;
    }
    // p of this iteration: the pair buffer in the second of an x pair (its
    // halo is exchanged, its ghost planes read)
    double* pl = xph == XPH_PAIR ? cg->p2_local : cg->p_local;
    cudaStream_t c = cg->ctx->comm;
    TW_CUDA(cudaEventRecord(cg->pready_ev, s));
    TW_CUDA(cudaStreamWaitEvent(c, cg->pready_ev, 0));
    halo_exchange(cg, c, pl);
    TW_CUDA(cudaEventRecord(cg->halo_ev, c));
    record(tmark(cg, 0), s);
    dist_spmv_interior(cg, s, pl);
    TW_CUDA(cudaStreamWaitEvent(s, cg->halo_ev, 0));
    dist_spmv_boundary(cg, s, pl);
    allgather1(cg, cg->send_a, cg->recv_a, s);
    record(tmark(cg, 1), s);
    dist_update_xr(cg, s);
    allgather1(cg, cg->send_b, cg->recv_b, s);
    record(tmark(cg, 2), s);
    dist_update_p(cg, s, xph);
    record(tmark(cg, 3), s);
    if (cg->timing) ++cg->timed;
}

// Tile kernels of one phase run side by side on the pool's streams (at most
// min(T, capacity) at once), so with few tiles each gets that share of the
// GPU's resident grid: a full grid per tile would make them queue behind one
// another, paying a ramp and a tail each (128^3, 4 tiles: 0.149 -> 0.142 ms
// per iteration with a graph).
int tile_share(const tw_cg* cg) {
    const int cap = static_cast<int>(cg->ctx->pool.capacity());
    // with many tiles each tile's grid is already bounded by its own size
    // (and measured: sharing then costs up to 15 %, profiles/r01_sweep_summary.md)
    if (cg->T > 2 * cap) return 1;
    return std::max(1, std::min(cg->T, cap));
}

void launch_node(tw_cg* cg, const PNode& nd, cudaStream_t st, int xph, int chain_role) {
    if (xph != XPH_SINGLE && !cg->x_pairs) contract_error("paired x update not enabled");
    // the iteration's p_old: in the pair buffer for the second of a pair
    double* pl = xph == XPH_PAIR ? cg->p2_local : cg->p_local;
    double* po = xph == XPH_PAIR ? cg->p2_owned : cg->p_owned;
    const int share = tile_share(cg);
    EllView A = cg->view();
    // rounded down: the side-by-side tiles' one-CTA-per-SM SpMV grids must
    // fit on the SMs together (3 tiles: 3 x 50 = 150 > 148 blocks would leave
    // one tile's last blocks waiting for another tile to finish)
    A.tma_blocks = std::max(1, A.tma_blocks / share);
    const int t = nd.tile;
    const int bs = (launch_blocks(cg, true) + share - 1) / share;
    const int bv = (launch_blocks(cg, false) + share - 1) / share;
    // the programmatic chain (chain_role >= 0): a programmatic launch with the role
    // (large tiles: the x/r phase's gate launched plainly, after the SpMV
    // tiles have completed; its role still lets the later tiles launch)
    const bool gate = chain_role == PDL_GATE || chain_role == PDL_GATE_LAST;
    const bool pdl = chain_role >= 0 && !(gate && nd.kind == PK_UPD && cg->chain_plain_upd);
    const int role = chain_role >= 0 ? chain_role : PDL_DEFAULT;
    switch (nd.kind) {
    case PK_HALO: // the buffer this iteration's SpMV tiles read
        halo_exchange(cg, st, xph == XPH_PAIR ? cg->p2_local : nullptr);
        break;
    case PK_SPMV: { // the x-staged K1 when the matrix has it
        const Fin f = cg->tile_fin(cg->pa, t, FIN_ALPHA, cg->tile_tickets);
        if (!launch_spmv_staged(A, pl, cg->Ap, RowRange{cg->t_r0[t], cg->t_r1[t]}, cg->slot(t), f,
                                st, pdl, role)) {
            if (pdl) contract_error("the programmatic chain needs the staged K1");
            launch_spmv(A, pl, cg->Ap, RowRange{cg->t_r0[t], cg->t_r1[t]}, RowRange{0, 0}, true,
                        cg->slot(t), f, bs, st);
        }
        break;
    }
    case PK_ALPHA: // folded into the last SpMV tile (an empty join node) on one rank
        if (cg->fold_scalars()) break;
        if (!cg->dist) {
            launch_combine(cg->pa, cg->T, Fin{FIN_ALPHA, nullptr, cg->sc, nullptr}, st);
        } else {
            launch_combine(cg->pa, cg->T, Fin{FIN_STORE, cg->send_a, nullptr, nullptr}, st);
            allgather1(cg, cg->send_a, cg->recv_a, st);
            launch_combine(cg->recv_a, cg->P, Fin{FIN_ALPHA, nullptr, cg->sc, nullptr}, st);
        }
        break;
    case PK_UPD: // x += alpha p moves into the p update from 4M rows (x_in_k3)
        launch_update_xr(cg->t_r0[t], cg->t_r1[t], x_in_k3(cg) ? nullptr : cg->x, po,
                         cg->r, cg->Ap, cg->sc,
                         ScalarSrc{nullptr, 0}, cg->slot(t),
                         cg->tile_fin(cg->rrp, t, FIN_BETA, cg->tile_tickets + 1), bv, st, pdl,
                         role);
        break;
    case PK_BETA: // folded into the last x/r-update tile on one rank
        if (cg->fold_scalars()) break;
        if (!cg->dist) {
            launch_combine(cg->rrp, cg->T, Fin{FIN_BETA, nullptr, cg->sc, cg->history}, st);
        } else {
            launch_combine(cg->rrp, cg->T, Fin{FIN_STORE, cg->send_b, nullptr, nullptr}, st);
            allgather1(cg, cg->send_b, cg->recv_b, st);
            launch_combine(cg->recv_b, cg->P, Fin{FIN_BETA, nullptr, cg->sc, cg->history}, st);
        }
        break;
    case PK_UPDP: // paired x updates: as in enqueue_mono, per tile
        if (xph == XPH_DEFER)
            launch_update_p(cg->t_r0[t], cg->t_r1[t], cg->r, cg->p2_owned, cg->sc,
                            ScalarSrc{nullptr, 0}, cg->slot(t), cg->history, bv, st, nullptr,
                            cg->p_owned, pdl, nullptr, nullptr, role);
        else if (xph == XPH_PAIR)
            launch_update_p(cg->t_r0[t], cg->t_r1[t], cg->r, cg->p_owned, cg->sc,
                            ScalarSrc{nullptr, 0}, cg->slot(t), cg->history, bv, st, nullptr,
                            cg->p2_owned, pdl, cg->x, cg->p_owned, role);
        else
            launch_update_p(cg->t_r0[t], cg->t_r1[t], cg->r, cg->p_owned, cg->sc,
                            ScalarSrc{nullptr, 0}, cg->slot(t), cg->history, bv, st, nullptr,
                            nullptr, pdl, x_in_k3(cg) ? cg->x : nullptr, nullptr, role);
        break;
    }
}

// All pooled streams (and the comm stream) start after everything already
// on the compute stream.
void fork_streams(tw_cg* cg) {
    if (cg->opt.dispatch == TW_DISPATCH_CHAIN) return; // one stream
    TW_CUDA(cudaEventRecord(cg->fork_ev, cg->ctx->compute));
    for (unsigned i = 0; i < cg->ctx->pool.capacity(); ++i)
        TW_CUDA(cudaStreamWaitEvent(cg->ctx->pool.stream(static_cast<int>(i)), cg->fork_ev, 0));
    TW_CUDA(cudaStreamWaitEvent(cg->ctx->comm, cg->fork_ev, 0));
}

void join_streams(tw_cg* cg) {
    if (cg->opt.dispatch == TW_DISPATCH_CHAIN) return;
    const unsigned C = cg->ctx->pool.capacity();
    for (unsigned i = 0; i <= C; ++i) {
        cudaStream_t st = i < C ? cg->ctx->pool.stream(static_cast<int>(i)) : cg->ctx->comm;
        TW_CUDA(cudaEventRecord(cg->tail_ev[i], st));
        TW_CUDA(cudaStreamWaitEvent(cg->ctx->compute, cg->tail_ev[i], 0));
    }
}

// One block-task iteration: physical nodes in topological order, each on its
// stream after waiting for predecessors on other streams.
// TW_DISPATCH_CHAIN: the iteration's physical nodes in DAG order on the
// compute stream, every tile kernel launched programmatically with its role
// in its phase (PdlRole): the first tile waits for every grid before it,
// the later ones start behind it without a wait, the last lets the next
// phase's first tile launch after its main loop.  alpha / beta_res combine
// kernels (more tiles than the fold takes) launch plainly.  Stream order is
// stronger than the DAG's edges (a p tile -> only its band's SpMV tiles)
// and replaces them: no events, one graph branch.
static void enqueue_tasks_chain(tw_cg* cg, int xph) {
    cudaStream_t s = cg->ctx->compute;
    const size_t m = cg->nodes.size();
    for (size_t j = 0; j < m; ++j) {
        const PNode& nd = cg->nodes[j];
        const bool tile = nd.kind == PK_SPMV || nd.kind == PK_UPD || nd.kind == PK_UPDP;
        int role = -1;
        if (tile) {
            const bool first = j == 0 || cg->nodes[j - 1].kind != nd.kind;
            const bool last = j + 1 == m || cg->nodes[j + 1].kind != nd.kind;
            role = first ? (last ? PDL_GATE_LAST : PDL_GATE) : (last ? PDL_LAST : PDL_INNER);
        }
        launch_node(cg, nd, s, xph, role);
    }
}

void enqueue_tasks(tw_cg* cg, int parity, bool first, int xph) {
    if (cg->opt.dispatch == TW_DISPATCH_CHAIN) {
        enqueue_tasks_chain(cg, xph);
        return;
    }
    for (size_t j = 0; j < cg->nodes.size(); ++j) {
        const PNode& nd = cg->nodes[j];
        cudaStream_t st = cg->node_stream(nd);
        for (int p : first ? nd.preds_first : nd.preds_intra)
            if (cg->node_stream(cg->nodes[static_cast<size_t>(p)]) != st)
                TW_CUDA(cudaStreamWaitEvent(st, cg->ev[parity][static_cast<size_t>(p)], 0));
        if (!first)
            for (int p : nd.preds_cross)
                if (cg->node_stream(cg->nodes[static_cast<size_t>(p)]) != st)
                    TW_CUDA(cudaStreamWaitEvent(st, cg->ev[parity ^ 1][static_cast<size_t>(p)], 0));
        launch_node(cg, nd, st, xph);
        TW_CUDA(cudaEventRecord(cg->ev[parity][j], st));
    }
}

void enqueue_iteration_body(tw_cg* cg, int parity, bool first, int xph) {
    if (cg->opt.variant == TW_CG_MONOLITHIC)
        enqueue_mono(cg, xph);
    else
        enqueue_tasks(cg, parity, first, xph);
}

void build_graph(tw_cg* cg) {
    cudaStream_t s = cg->ctx->compute;
    cudaGraph_t g = nullptr;
    TW_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    try {
        if (cg->opt.variant == TW_CG_TASKS) {
            fork_streams(cg);
            enqueue_tasks(cg, 0, true);
            join_streams(cg);
        } else {
            enqueue_mono(cg);
        }
    } catch (...) {
        cudaStreamEndCapture(s, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    TW_CUDA(cudaStreamEndCapture(s, &g));
    cudaError_t e = cudaGraphInstantiate(&cg->graph, g, 0);
    cudaGraphDestroy(g);
    TW_CUDA(e);
}

cudaGraphExec_t build_chunk_graph(tw_cg* cg, int c) {
    cudaStream_t s = cg->ctx->compute;
    cudaGraph_t g = nullptr;
    TW_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    try {
        if (cg->opt.variant == TW_CG_TASKS) {
            fork_streams(cg);
            for (int i = 0; i < c; ++i) enqueue_tasks(cg, i & 1, i == 0, x_phase(cg, i, c));
            join_streams(cg);
        } else {
            for (int i = 0; i < c; ++i) enqueue_mono(cg, x_phase(cg, i, c));
        }
    } catch (...) {
        cudaStreamEndCapture(s, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    TW_CUDA(cudaStreamEndCapture(s, &g));
    cudaGraphExec_t ge = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
    cudaGraphDestroy(g);
    TW_CUDA(e);
    return ge;
}

void free_cg(tw_cg* cg) {
    if (!cg) return;
    cudaSetDevice(cg->ctx->device);
    cudaDeviceSynchronize();
    cg->ta.reset();
    if (cg->graph) cudaGraphExecDestroy(cg->graph);
    for (auto& kv : cg->timed_graphs) cudaGraphExecDestroy(kv.second);
    for (auto& kv : cg->chunk_graphs) cudaGraphExecDestroy(kv.second);
    for (auto& v : cg->ev)
        for (auto e : v) cudaEventDestroy(e);
    for (auto e : cg->tail_ev) cudaEventDestroy(e);
    for (auto e : cg->tev) cudaEventDestroy(e);
    for (auto e : cg->iter_ev) cudaEventDestroy(e);
    if (cg->fork_ev) cudaEventDestroy(cg->fork_ev);
    if (cg->halo_ev) cudaEventDestroy(cg->halo_ev);
    if (cg->pready_ev) cudaEventDestroy(cg->pready_ev);
    if (cg->ag_in_ev) cudaEventDestroy(cg->ag_in_ev);
    if (cg->ag_out_ev) cudaEventDestroy(cg->ag_out_ev);
    cudaFree(cg->x);
    cudaFree(cg->r_base);
    cudaFree(cg->p_base); // (the pair buffer included)
    cudaFree(cg->Ap);
    cudaFree(cg->sc);
    cudaFree(cg->history);
    cudaFree(cg->parts);
    cudaFree(cg->block_parts);
    cudaFree(cg->tickets);
    cudaFree(cg->tile_tickets);
    for (void* m : cg->ipc_mapped) cudaIpcCloseMemHandle(m);
    cudaFree(cg->win);
    cudaFree(cg->d_links);
    cudaFree(cg->d_links2);
    for (auto& kv : cg->dag_tables) {
        auto& t = kv.second;
        cudaFree(t.d_tasks);
        cudaFree(t.d_chunk_task);
        cudaFree(t.d_succ);
        cudaFree(t.d_npred);
        cudaFree(t.d_remaining);
        cudaFree(t.d_chunk_done);
        cudaFree(t.d_chunk_part);
    }
    cudaFree(cg->d_ticket);
    cudaFree(cg->d_stamps);
    delete cg;
}

tw_cg* create_cg(tw_ctx* ctx, const tw_ell* A, const tw_cg_options* o, int max_iters) {
    if (!ctx || !A) contract_error("null context or matrix");
    if (A->ctx != ctx) contract_error("matrix belongs to another context");
    if (max_iters < 0) config_error("iterations must be non-negative");
    auto* cg = new tw_cg;
    try {
        cg->ctx = ctx;
        cg->A = A;
        if (o)
            cg->opt = *o;
        else
            tw_cg_options_default(&cg->opt);
        if (cg->opt.dispatch == TW_DISPATCH_AUTO) {
            // the persistent dispatcher where it wins (many tiles, one rank,
            // no graph requested; profiles/r01_sweep_summary.md), else streams
            // small tiles: on an x-staged matrix below ~400k rows per tile,
            // or from 8 tiles up below 3M rows per tile (measured crossovers:
            // 128^3 between 4 and 8 tiles, 256^3 at 4 tiles (a tie);
            // profiles/r01_dispatcher_summary.md); on a gather matrix, more
            // than 8 tiles
            int sb, vb, cb;
            const bool fits =
                dag_smem_bytes(A->info.max_width, A->cols16 != nullptr, &sb, &vb, &cb) <= 225 * 1024;
            const int64_t rows_per_tile = A->info.n_rows / std::max(cg->opt.tiles, 1);
            const bool small =
                cg->opt.tiles > 1 &&
                (A->cols16 ? rows_per_tile < 400000 || (cg->opt.tiles >= 8 && rows_per_tile < 3000000)
                           : cg->opt.tiles > 8);
            // the programmatic chain for 2 to 8 tiles of 50k rows and more on
            // an x-staged matrix (128^3: 2 / 4 / 8 tiles 118.5 / 119.0 / 128.5 us
            // against streams 124.2 / 126.3 and the dispatcher's 135.4 at 8;
            // 96^3, 4 tiles: 61.5 against the dispatcher's 82.5; 256^3, 2 / 4
            // / 8 tiles 853 / 853 / 861 against streams 858 / 858 and the
            // dispatcher's 875 at 8; below ~50k rows per tile (64^3, 8 tiles)
            // the dispatcher's one launch wins; profiles/r02_ab_chain.md)
            const bool chain = A->cols16 && cg->opt.tiles > 1 && cg->opt.tiles <= 8 &&
                               rows_per_tile >= 50000;
            const bool one_rank = cg->opt.variant == TW_CG_TASKS && !ctx->nccl_comm &&
                                  !ctx->emulated && !cg->opt.use_graph;
            cg->opt.dispatch = one_rank && chain            ? TW_DISPATCH_CHAIN
                               : one_rank && small && fits ? TW_DISPATCH_PERSISTENT
                                                           : TW_DISPATCH_STREAMS;
        }
        if (cg->opt.dispatch == TW_DISPATCH_PERSISTENT) {
            if (cg->opt.variant != TW_CG_TASKS)
                config_error("the persistent dispatcher runs the tasks variant");
            int sb, vb, cb;
            if (dag_smem_bytes(A->info.max_width, A->cols16 != nullptr, &sb, &vb, &cb) > 225 * 1024)
                config_error("matrix rows too wide for the dispatcher's shared-memory stages");
            if (cg->opt.use_graph) config_error("the persistent dispatcher is one launch; no graph");
        } else if (cg->opt.dispatch == TW_DISPATCH_CHAIN) {
            if (cg->opt.variant != TW_CG_TASKS) config_error("the programmatic chain runs the tasks variant");
            if (ctx->nccl_comm || ctx->emulated) config_error("the programmatic chain runs on one rank");
            if (!A->cols16) config_error("the programmatic chain needs the x-staged matrix form");
        } else if (cg->opt.dispatch != TW_DISPATCH_STREAMS) {
            config_error("unknown dispatch mode");
        }
        if (cg->opt.variant != TW_CG_MONOLITHIC && cg->opt.variant != TW_CG_TASKS)
            config_error("unknown CG variant");
        if (cg->opt.x_update < TW_XUPD_AUTO || cg->opt.x_update > TW_XUPD_K3_PAIRS)
            config_error("unknown x_update placement");
        if (cg->opt.l2_keep < TW_L2KEEP_AUTO || cg->opt.l2_keep > TW_L2KEEP_OFF)
            config_error("unknown l2_keep policy");
        cg->T = cg->opt.variant == TW_CG_MONOLITHIC ? 1 : cg->opt.tiles; // cg.cpp:400
        cg->P = ctx->nranks;
        // rank-partial path: an NCCL communicator (also 1 rank) or an emulated rank
        cg->dist = ctx->nccl_comm != nullptr || ctx->emulated;
        cg->max_iters = max_iters;
        const tw_ell_info_t& in = A->info;
        cg->n = in.n_rows;
        cg->chain_plain_upd = cg->opt.dispatch == TW_DISPATCH_CHAIN &&
                              cg->n / std::max(cg->T, 1) >= 3000000;
        cg->x_len = in.x_len;
        cg->diag_shift = A->diag_shift;
        if (cg->dist) {
            if (in.nx == 0) config_error("multi-GPU CG needs a stencil slab (tw_gen_stencil_ell)");
            cg->plane = in.nx * in.ny;
            cg->glo = in.z_begin > 0;
            cg->ghi = in.z_end < in.nz;
            if (cg->glo != (ctx->rank > 0) || cg->ghi != (ctx->rank < cg->P - 1))
                contract_error("slab z-range does not match this rank's position");
            if (int rc = tw_slab_plan(in.nx, in.ny, in.nz, in.z_begin, in.z_end, &cg->slab); rc)
                throw Error(rc, g_last_error);
            if (cg->slab.diag_shift != cg->diag_shift || cg->slab.x_len != cg->x_len)
                contract_error("matrix and slab plan disagree");
        } else if (cg->P > 1) {
            contract_error("multi-rank context without communicator");
        } else if (in.z_begin > 0 || (in.nx && in.z_end < in.nz)) {
            contract_error("a partial slab needs a multi-rank context");
        }
        tile_plan(A, cg->T, cg->t_r0, cg->t_r1, cg->t_lo, cg->t_hi);
        cg->dag = DagSpec{cg->T, cg->dist, cg->glo, cg->ghi, cg->n, cg->diag_shift, cg->plane,
                          cg->t_r0, cg->t_r1, cg->t_lo, cg->t_hi};
        TW_CUDA(cudaSetDevice(ctx->device));
        const size_t n = static_cast<size_t>(cg->n);
        TW_CUDA(cudaMalloc(&cg->x, sizeof(double) * (n + 2)));
        TW_CUDA(cudaMalloc(&cg->r_base, sizeof(double) * (n + 32)));
        cg->r = cg->r_base + 16; // 128-byte aligned, slack for the fused K1's staged r runs
        TW_CUDA(cudaMalloc(&cg->Ap, sizeof(double) * (n + 2)));
        // p_owned on a 128-byte line (the streaming kernels' 128-bit accesses
        // then never straddle lines) with at least 2 doubles of slack before
        // p_local and after its end: the x-staged K1 copies 36-double runs
        // that start 2 before a line
        int64_t front = (16 - cg->diag_shift % 16) % 16;
        if (front < 2) front += 16;
        // (and at least kStageRunLen after: a run-table run may start at the
        // last column)
        cg->x_k3 = decide_x_in_k3(cg);
        cg->x_pairs = decide_x_pairs(cg);
        // the pair buffer (paired x updates) sits in the same allocation, one
        // stride of whole 128-byte lines further: same line offset and slack
        // as p_local, and one IPC mapping of p_base reaches both (a peer
        // rank stores its halo planes into either buffer's ghost planes)
        const int64_t stride = (cg->x_len + front + 48 + 15) / 16 * 16;
        const size_t pbytes = sizeof(double) * static_cast<size_t>(stride * (cg->x_pairs ? 2 : 1));
        TW_CUDA(cudaMalloc(&cg->p_base, pbytes));
        TW_CUDA(cudaMemset(cg->p_base, 0, pbytes));
        cg->p_local = cg->p_base + front;
        cg->p_owned = cg->p_local + cg->diag_shift;
        if (cg->x_pairs) {
            cg->p2_base = cg->p_base + stride;
            cg->p2_local = cg->p2_base + front;
            cg->p2_owned = cg->p2_local + cg->diag_shift;
        }
        TW_CUDA(cudaMalloc(&cg->sc, sizeof(CgScalars)));
        TW_CUDA(cudaMalloc(&cg->history, sizeof(double) * std::max(max_iters, 1)));
        const int T = cg->T, P = cg->P;
        const size_t np = static_cast<size_t>(2 * T + 8 + 3 * P + 8);
        TW_CUDA(cudaMalloc(&cg->parts, sizeof(double) * np));
        TW_CUDA(cudaMemset(cg->parts, 0, sizeof(double) * np));
        cg->pa = cg->parts;
        cg->rrp = cg->pa + T;
        cg->pm = cg->rrp + T;
        cg->send_a = cg->pm + 4;
        cg->send_b = cg->send_a + 1;
        cg->send_r = cg->send_b + 1;
        cg->recv_a = cg->send_r + 1;
        cg->recv_b = cg->recv_a + P;
        cg->recv_r = cg->recv_b + P;
        cg->maxg = std::max(ctx->cfg.spmv_blocks, ctx->cfg.stream_blocks);
        TW_CUDA(cudaMalloc(&cg->block_parts, sizeof(double) * static_cast<size_t>(cg->maxg) * T));
        TW_CUDA(cudaMalloc(&cg->tickets, sizeof(unsigned) * 4 * T));
        TW_CUDA(cudaMemset(cg->tickets, 0, sizeof(unsigned) * 4 * T));
        TW_CUDA(cudaMalloc(&cg->tile_tickets, sizeof(unsigned) * 2));
        TW_CUDA(cudaMemset(cg->tile_tickets, 0, sizeof(unsigned) * 2));
        TW_CUDA(cudaEventCreateWithFlags(&cg->fork_ev, cudaEventDisableTiming));
        TW_CUDA(cudaEventCreateWithFlags(&cg->halo_ev, cudaEventDisableTiming));
        TW_CUDA(cudaEventCreateWithFlags(&cg->pready_ev, cudaEventDisableTiming));
        TW_CUDA(cudaEventCreateWithFlags(&cg->ag_in_ev, cudaEventDisableTiming));
        TW_CUDA(cudaEventCreateWithFlags(&cg->ag_out_ev, cudaEventDisableTiming));
        for (unsigned i = 0; i <= ctx->pool.capacity(); ++i) {
            cudaEvent_t e;
            TW_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            cg->tail_ev.push_back(e);
        }
        if (cg->opt.variant == TW_CG_TASKS) {
            build_schedule(cg);
            for (auto& v : cg->ev)
                for (size_t j = 0; j < cg->nodes.size(); ++j) {
                    cudaEvent_t e;
                    TW_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                    v.push_back(e);
                }
        }
        cg->marks.assign(static_cast<size_t>(std::max(max_iters, 1)), 0.0);
        cg->mark_real.assign(cg->marks.size(), 0);
        cg->ta = std::make_unique<TaskAware>(ctx->device, 20e-6);
        if (cg->opt.dispatch == TW_DISPATCH_PERSISTENT) {
            TW_CUDA(cudaMalloc(&cg->d_stamps, sizeof(unsigned long long) * (max_iters + 2)));
            TW_CUDA(cudaMemset(cg->d_stamps, 0, sizeof(unsigned long long) * (max_iters + 2)));
            TW_CUDA(cudaMalloc(&cg->d_ticket, sizeof(unsigned) * 4));
            cg->dag_grid = dag_blocks(A->info.max_width, A->cols16 != nullptr, ctx->sm_count);
        }
    } catch (...) {
        free_cg(cg);
        throw;
    }
    return cg;
}

// x = 0, r = p = b, and the local r.r into send_r (dist) or rtrans (single).
void set_rhs_prefix(tw_cg* cg, const double* b, bool on_device, cudaStream_t s) {
    tw_ctx* ctx = cg->ctx;
    const size_t bytes = sizeof(double) * static_cast<size_t>(cg->n);
    CgScalars init{};
    init.history_cap = cg->max_iters;
    init.epoch = ++cg->epoch;
    TW_CUDA(cudaMemcpyAsync(cg->sc, &init, sizeof(init), cudaMemcpyHostToDevice, s));
    TW_CUDA(cudaMemsetAsync(cg->x, 0, bytes, s));
    TW_CUDA(cudaMemsetAsync(cg->Ap, 0, bytes, s));
    TW_CUDA(cudaMemsetAsync(cg->p_local, 0, sizeof(double) * static_cast<size_t>(cg->x_len), s));
    if (on_device)
        TW_CUDA(cudaMemcpyAsync(cg->r, b, bytes, cudaMemcpyDeviceToDevice, s));
    else
        copy_h2d(ctx, cg->r, b, bytes, s);
    TW_CUDA(cudaMemcpyAsync(cg->p_owned, cg->r, bytes, cudaMemcpyDeviceToDevice, s));
    const RedScratch rs = cg->slot(0);
    if (!cg->dist)
        launch_dot(cg->r, cg->r, 0, cg->n, rs, Fin{FIN_RTRANS, nullptr, cg->sc, nullptr},
                   ctx->cfg.stream_blocks, s);
    else
        launch_dot(cg->r, cg->r, 0, cg->n, rs, Fin{FIN_STORE, cg->send_r, nullptr, nullptr},
                   ctx->cfg.stream_blocks, s);
}

void reset_solve_state(tw_cg* cg) {
    cg->enqueued = 0;
    std::fill(cg->marks.begin(), cg->marks.end(), 0.0);
    std::fill(cg->mark_real.begin(), cg->mark_real.end(), 0);
    cg->t0 = host_seconds();
}

void set_rhs(tw_cg* cg, const double* b, bool on_device) {
    tw_ctx* ctx = cg->ctx;
    if (ctx->emulated) contract_error("emulated ranks are driven as a group (tw_cg_group_set_rhs)");
    cudaStream_t s = ctx->compute;
    TW_CUDA(cudaSetDevice(ctx->device));
    TW_CUDA(cudaStreamSynchronize(s));
    set_rhs_prefix(cg, b, on_device, s);
    if (cg->dist) {
        // the allgather is also the barrier that orders every rank's memset of
        // its ghost planes before any neighbour's push into them
        allgather1(cg, cg->send_r, cg->recv_r, s);
        launch_combine(cg->recv_r, cg->P, Fin{FIN_RTRANS, nullptr, cg->sc, nullptr}, s);
        if (cg->peer)
            launch_peer_push(cg->p_owned, cg->n, cg->plane, cg->links, cg->sc, cg->tickets, s);
    }
    TW_CUDA(cudaStreamSynchronize(s));
    reset_solve_state(cg);
}

// Timing event at the end of iteration i-1 (i = 0: the start of the solve).
cudaEvent_t iter_event(tw_cg* cg, int i) {
    while (static_cast<int>(cg->iter_ev.size()) <= i) {
        cudaEvent_t e;
        TW_CUDA(cudaEventCreate(&e));
        cg->iter_ev.push_back(e);
    }
    return cg->iter_ev[static_cast<size_t>(i)];
}

// Flattens k iterations of the physical DAG into the dispatcher's task table
// (topological order, chunk list, successor lists, predecessor counts).
// Chunk sizes: up to 216 slices (12 per compute warp) per SpMV chunk and
// 32768 rows per update chunk (the 256^3 optimum); on smaller problems SpMV
// chunks in whole waves over the CTAs and update chunks of the next power
// of two above half a CTA's rows (round-2 sweeps at 128^3, 16 tiles: 144.7
// -> 132.7 us per iteration; profiles/r02_ab_tasks_executors.md).
// tw_cg_options::dag_spmv_slices / dag_vec_rows override (tuning sweeps).
int64_t dag_spmv_chunk_slices(const tw_cg* cg) {
    if (cg->opt.dag_spmv_slices > 0) return cg->opt.dag_spmv_slices;
    const int64_t w = dag_compute_warps(), grid = std::max(cg->dag_grid, 1);
    const int64_t ns_tile = ((cg->n + 31) / 32 + cg->T - 1) / cg->T;
    // a whole number of slices per compute warp (the warps of a CTA share a
    // chunk round-robin: one slice more than a multiple costs a round), and
    // the phase's chunks in whole waves over the CTAs: among 1..12 slices
    // per warp, the size whose chunk count fills its last wave best, with
    // 4 to 8 waves per phase; a problem with more waves than that at 12
    // slices per warp (256^3) takes 12
    int64_t best = 12 * w;
    double best_fill = -1.0;
    for (int64_t k = 1; k <= 12; ++k) {
        const int64_t sl = k * w;
        const int64_t chunks = cg->T * ((ns_tile + sl - 1) / sl);
        const double waves = static_cast<double>(chunks) / static_cast<double>(grid);
        if (waves < 4.0 || waves > 8.0) continue;
        const double fill = waves / std::ceil(waves);
        if (fill > best_fill + 1e-9 || (std::abs(fill - best_fill) <= 1e-9 && sl > best)) {
            best_fill = fill;
            best = sl;
        }
    }
    if (best_fill < 0.0) { // no size gives 4-8 waves: the largest that gives at least 4
        best = w;
        for (int64_t k = 12; k >= 1; --k)
            if (cg->T * ((ns_tile + k * w - 1) / (k * w)) >= 4 * grid) {
                best = k * w;
                break;
            }
    }
    return best;
}
int64_t dag_vec_chunk_rows(const tw_cg* cg) {
    if (cg->opt.dag_vec_rows > 0) return cg->opt.dag_vec_rows;
    const int64_t fit = cg->n / (2 * static_cast<int64_t>(std::max(cg->dag_grid, 1)));
    if (fit >= 24576) return 32768;
    int64_t rows = 2048;
    while (rows < fit) rows *= 2;
    return rows;
}

// The task table of k iterations of the ranks g[0..P) (one rank on a GPU;
// every rank of an emulated group in one launch), kept in g[0]->dag_tables[k].
// Order: per iteration, phase by phase (halo, SpMV tiles, alpha, x/r tiles,
// beta_res, p tiles), rank by rank inside a phase.  That order is
// topological for the local edges and for the cross-rank ones (a ghost
// plane's halo task precedes the SpMV tiles reading it; every rank's alpha
// / beta_res publishes before it waits), so with every CTA resident a chunk
// only ever waits on chunks already taken: no deadlock.
void build_dag_table(tw_cg** g, int P, int k) {
    const int64_t spmv_cs = dag_spmv_chunk_slices(g[0]);
    const int64_t vec_cr = dag_vec_chunk_rows(g[0]);
    // id of (rank, iteration, node), assigned in the launch order above (the
    // end ranks have no halo node: node lists differ by at most one entry)
    size_t L = 0;
    for (int r = 0; r < P; ++r) L = std::max(L, g[r]->nodes.size());
    std::vector<int> id_of(static_cast<size_t>(P) * k * L, -1);
    auto key = [&](int r, int it, int j) {
        return (static_cast<size_t>(r) * k + static_cast<size_t>(it)) * L + static_cast<size_t>(j);
    };
    std::vector<DagTask> tasks;
    std::vector<std::pair<int, int>> who; // (rank, node) of every task, for the preds pass
    std::vector<int> iter_of;
    static const PhysKind kPhases[] = {PK_HALO, PK_SPMV, PK_ALPHA, PK_UPD, PK_BETA, PK_UPDP};
    for (int it = 0; it < k; ++it)
        for (PhysKind ph : kPhases)
            for (int r = 0; r < P; ++r) {
                const tw_cg* cg = g[r];
                for (int j = 0; j < static_cast<int>(cg->nodes.size()); ++j) {
                    const PNode& nd = cg->nodes[static_cast<size_t>(j)];
                    if (nd.kind != ph) continue;
                    id_of[key(r, it, j)] = static_cast<int>(tasks.size());
                    DagTask t{};
                    t.tile = nd.tile;
                    t.rank = r;
                    t.iter = it;
                    t.r0 = cg->t_r0[static_cast<size_t>(nd.tile)];
                    t.r1 = cg->t_r1[static_cast<size_t>(nd.tile)];
                    t.nchunks = 1;
                    const int xph = x_phase(cg, it, k); // paired x updates (one rank)
                    switch (nd.kind) {
                    case PK_SPMV: {
                        t.kind = DK_SPMV;
                        if (xph == XPH_PAIR) t.flags |= kDagReadP2;
                        const int64_t ns = ((t.r1 + 31) >> 5) - (t.r0 >> 5);
                        t.nchunks = static_cast<int>((ns + spmv_cs - 1) / spmv_cs);
                        if (cg->peer) { // band (local x, inclusive) reaching a ghost plane
                            if (cg->glo && cg->t_lo[static_cast<size_t>(nd.tile)] < cg->diag_shift)
                                t.flags |= kDagGhostLo;
                            if (cg->ghi && cg->t_hi[static_cast<size_t>(nd.tile)] >= cg->diag_shift + cg->n)
                                t.flags |= kDagGhostHi;
                        }
                        break;
                    }
                    case PK_ALPHA: t.kind = DK_ALPHA; break;
                    case PK_UPD:
                        t.kind = DK_UPD;
                        t.nchunks = static_cast<int>((t.r1 - t.r0 + vec_cr - 1) / vec_cr);
                        break;
                    case PK_BETA: t.kind = DK_BETA; break;
                    case PK_UPDP:
                        t.kind = DK_UPDP;
                        t.nchunks = static_cast<int>((t.r1 - t.r0 + vec_cr - 1) / vec_cr);
                        if (xph == XPH_DEFER) t.flags |= kDagXDefer;
                        if (xph == XPH_PAIR) t.flags |= kDagXPair;
                        break;
                    case PK_HALO: // a no-op without neighbours (a 1-rank communicator)
                        if (!cg->peer && (cg->glo || cg->ghi))
                            contract_error("the dispatcher's halo task needs the peer transport");
                        t.kind = DK_HALO;
                        if (xph == XPH_PAIR) t.flags |= kDagReadP2; // the pair buffer's planes
                        break;
                    }
                    tasks.push_back(t);
                    who.emplace_back(r, j);
                    iter_of.push_back(it);
                }
            }
    std::vector<std::vector<int>> succ(tasks.size());
    std::vector<int> npred(tasks.size(), 0), chunk_task;
    for (size_t id = 0; id < tasks.size(); ++id) {
        const auto [r, j] = who[id];
        const int it = iter_of[id];
        const PNode& nd = g[r]->nodes[static_cast<size_t>(j)];
        auto add = [&](int pit, int pj) {
            const int pid = id_of[key(r, pit, pj)];
            if (pid < 0 || pid >= static_cast<int>(id)) contract_error("task order is not topological");
            succ[static_cast<size_t>(pid)].push_back(static_cast<int>(id));
            ++npred[id];
        };
        if (it == 0) {
            for (int p : nd.preds_first) add(0, p);
        } else {
            for (int p : nd.preds_intra) add(it, p);
            for (int p : nd.preds_cross) add(it - 1, p);
        }
        tasks[id].chunk0 = static_cast<int>(chunk_task.size());
        chunk_task.insert(chunk_task.end(), static_cast<size_t>(tasks[id].nchunks), static_cast<int>(id));
    }
    std::vector<int> flat;
    for (size_t i = 0; i < tasks.size(); ++i) {
        tasks[i].succ0 = static_cast<int>(flat.size());
        tasks[i].nsucc = static_cast<int>(succ[i].size());
        flat.insert(flat.end(), succ[i].begin(), succ[i].end());
    }
    if (flat.empty()) flat.push_back(0);
    auto realloc = [](auto*& p, size_t n) {
        cudaFree(p);
        p = nullptr;
        TW_CUDA(cudaMalloc(&p, sizeof(*p) * std::max<size_t>(n, 1)));
    };
    tw_cg::DagTable& tb = g[0]->dag_tables[k];
    realloc(tb.d_tasks, tasks.size());
    realloc(tb.d_chunk_task, chunk_task.size());
    realloc(tb.d_succ, flat.size());
    realloc(tb.d_npred, npred.size());
    realloc(tb.d_remaining, npred.size());
    realloc(tb.d_chunk_done, tasks.size());
    realloc(tb.d_chunk_part, chunk_task.size());
    TW_CUDA(cudaMemcpy(tb.d_tasks, tasks.data(), sizeof(DagTask) * tasks.size(), cudaMemcpyHostToDevice));
    TW_CUDA(cudaMemcpy(tb.d_chunk_task, chunk_task.data(), sizeof(int) * chunk_task.size(),
                       cudaMemcpyHostToDevice));
    TW_CUDA(cudaMemcpy(tb.d_succ, flat.data(), sizeof(int) * flat.size(), cudaMemcpyHostToDevice));
    TW_CUDA(cudaMemcpy(tb.d_npred, npred.data(), sizeof(int) * npred.size(), cudaMemcpyHostToDevice));
    tb.ntasks = static_cast<int>(tasks.size());
    tb.nchunks = static_cast<int>(chunk_task.size());
}

// k iterations of cg_tasks of the ranks g[0..P) as ONE persistent kernel
// (tw_dag.cu) on g[0]'s compute stream.
void enqueue_persistent(tw_cg** g, int P, int k) {
    tw_cg* cg = g[0];
    if (P > kDagMaxRanks) config_error("more ranks than one dispatcher launch holds");
    cudaStream_t s = cg->ctx->compute;
    if (!cg->dag_tables.count(k)) {
        TW_CUDA(cudaStreamSynchronize(s));
        build_dag_table(g, P, k);
    }
    const tw_cg::DagTable& tb = cg->dag_tables[k];
    TW_CUDA(cudaMemcpyAsync(tb.d_remaining, tb.d_npred, sizeof(int) * tb.ntasks,
                            cudaMemcpyDeviceToDevice, s));
    TW_CUDA(cudaMemsetAsync(tb.d_chunk_done, 0, sizeof(unsigned) * tb.ntasks, s));
    for (int r = 0; r < P; ++r) // the chunk ticket and the tile-publication counters
        TW_CUDA(cudaMemsetAsync(g[r]->d_ticket, 0, sizeof(unsigned) * 4, s));
    DagParams D{};
    D.tasks = tb.d_tasks;
    D.chunk_task = tb.d_chunk_task;
    D.succ = tb.d_succ;
    D.remaining = tb.d_remaining;
    D.chunk_done = tb.d_chunk_done;
    D.chunk_part = tb.d_chunk_part;
    D.ticket = cg->d_ticket;
    D.nchunks = tb.nchunks;
    D.ntasks = tb.ntasks;
    D.T = cg->T;
    D.nranks = P;
    for (int r = 0; r < P; ++r) {
        const tw_cg* c = g[r];
        DagRank& R = D.rk[r];
        R.A = c->view();
        R.p_local = c->p_local;
        R.p_owned = c->p_owned;
        R.p2_local = c->p2_local;
        R.p2_owned = c->p2_owned;
        R.x = c->x;
        R.r = c->r;
        R.Ap = c->Ap;
        R.sc = c->sc;
        R.history = c->history;
        R.stamps = c->d_stamps;
        R.pa = c->pa;
        R.rr = c->rrp;
        R.links = c->peer ? c->d_links : nullptr;
        R.links2 = c->peer && c->x_pairs ? c->d_links2 : nullptr;
        R.win = c->peer ? c->win : nullptr;
        R.tctr = c->d_ticket + 2;
        R.iter0 = c->enqueued;
    }
    D.start_stamp = cg->enqueued == 0 ? cg->d_stamps : cg->d_stamps + cg->max_iters + 1;
    D.spmv_chunk_slices = dag_spmv_chunk_slices(cg);
    D.vec_chunk_rows = dag_vec_chunk_rows(cg);
    // the stages hold the widest slice of ANY rank of the launch (an end
    // slab's rows reach one plane fewer than a middle slab's: 18 against 27
    // entries), and the grid is what fits on the device at that size
    int mw = 0;
    bool staged = true;
    for (int r = 0; r < P; ++r) {
        mw = std::max(mw, static_cast<int>(g[r]->A->info.max_width));
        staged = staged && D.rk[r].A.cols16 != nullptr;
    }
    if (!staged)
        for (int r = 0; r < P; ++r)
            if (D.rk[r].A.cols16) config_error("the ranks of one launch mix staged and gather matrices");
    D.max_width = mw;
    dag_smem_bytes(mw, staged, &D.stage_bytes, &D.val_bytes, &D.c16_bytes);
    const int grid = P == 1 ? cg->dag_grid : dag_blocks(mw, staged, cg->ctx->sm_count);
    // update chunks by TMA when the stage holds >= 128 rows of each operand
    // (multiples of 64 rows: one 16-byte pair per lane and step); the
    // register path remains for stages too small for that.  With the x
    // update in the p-update chunks (x_in_k3) x/r chunks stream r, Ap and p
    // chunks r, p, x; else x, p, r, Ap and r, p
    const int rows2 = (D.stage_bytes / 16) & ~63, rows3 = (D.stage_bytes / 24) & ~63,
              rows4 = (D.stage_bytes / 32) & ~63;
    // (only when BOTH update kinds take the TMA path: the register path of
    // the x/r chunks always updates x -- a stage too small for 4-operand
    // blocks but not for 3 once updated x twice; found by
    // scripts/stress_random.py on tiny grids)
    D.x_in_updp = x_in_k3(cg) && rows3 >= 128 && rows4 >= 128;
    // x/r chunks keep the 4-operand block size either way: a lane's rows (and
    // so its r.r partial) do not depend on where x is updated
    const int ru = rows4, rp = D.x_in_updp ? rows3 : rows2;
    D.upd_block_rows = ru >= 128 ? ru : 0;
    D.updp_block_rows = rp >= 128 ? rp : 0;
    for (int r = 0; r < P; ++r)
        if (g[r]->x_pairs != cg->x_pairs) contract_error("the ranks of a launch pair their x updates alike");
    if (cg->x_pairs && (!D.x_in_updp || !D.upd_block_rows))
        contract_error("paired x updates need the dispatcher's TMA update chunks");
    D.x_pairs = cg->x_pairs ? 1 : 0;
    // stamps[0] is the start of the first launch after set_rhs; later launches
    // write their start into a spare slot so iteration ends stay in place
    launch_dag(D, grid, s);
}

void iterate(tw_cg* cg, int k) {
    if (cg->ctx->emulated) contract_error("emulated ranks iterate as a group (tw_cg_group_iterate)");
    if (k < 0) config_error("negative iteration count");
    if (cg->enqueued + k > cg->max_iters)
        contract_error("iterations beyond max_iterations (" + std::to_string(cg->max_iters) + ")");
    if (k == 0) return;
    TW_CUDA(cudaSetDevice(cg->ctx->device));
    cudaStream_t s = cg->ctx->compute;
    if (cg->opt.dispatch == TW_DISPATCH_PERSISTENT) {
        // across ranks the dispatcher's cross edges are the peer protocol
        if (cg->dist && cg->P > 1 && !cg->peer)
            contract_error("the multi-rank dispatcher runs over the peer transport (tw_cg_peer_connect)");
        enqueue_persistent(&cg, 1, k);
        if (cg->opt.iteration_marks) {
            cudaEvent_t e = cg->ta->take_event();
            TW_CUDA(cudaEventRecord(e, s));
            cg->ta->bind(e, &cg->marks[static_cast<size_t>(cg->enqueued + k - 1)], cg->t0);
            cg->mark_real[static_cast<size_t>(cg->enqueued + k - 1)] = 1;
        }
        cg->enqueued += k;
        return;
    }
    if (cg->opt.use_graph && cg->opt.variant == TW_CG_MONOLITHIC && cg->timing) {
        // k iterations as ONE graph; timed: with the K1/K2/K3 timing events
        // inside (graph-launch efficiency and per-kernel durations of one run)
        auto& cache = cg->timed_graphs;
        auto it = cache.find(k);
        if (it == cache.end()) {
            cudaGraph_t g = nullptr;
            cg->timed = 0;
            TW_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            try {
                for (int i = 0; i < k; ++i) enqueue_mono(cg, x_phase(cg, i, k));
            } catch (...) {
                cudaStreamEndCapture(s, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            TW_CUDA(cudaStreamEndCapture(s, &g));
            cudaGraphExec_t ge = nullptr;
            cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
            cudaGraphDestroy(g);
            TW_CUDA(e);
            it = cache.emplace(k, ge).first;
        }
        TW_CUDA(cudaGraphLaunch(it->second, s));
        if (cg->timing) cg->timed = k; // the graph records timing slots 0..k-1
        cg->enqueued += k;
        return;
    }
    const bool tasks = cg->opt.variant == TW_CG_TASKS;
    if (cg->opt.use_graph && !cg->opt.iteration_marks) {
        // no per-iteration host marks: chunks of up to kGraphChunk iterations
        // per graph launch, so consecutive iterations overlap where the DAG
        // allows (tasks) and no graph boundary sits between two iterations
        // of a chunk; one graph per chunk length, cached
        for (int left = k; left > 0;) {
            const int c = std::min(left, kGraphChunk);
            auto it = cg->chunk_graphs.find(c);
            if (it == cg->chunk_graphs.end()) it = cg->chunk_graphs.emplace(c, build_chunk_graph(cg, c)).first;
            TW_CUDA(cudaGraphLaunch(it->second, s));
            left -= c;
        }
        cg->enqueued += k;
        return;
    }
    if (cg->opt.use_graph && !cg->graph) build_graph(cg);
    if (!cg->opt.use_graph && tasks) fork_streams(cg);
    if (cg->opt.iteration_marks && cg->enqueued == 0) TW_CUDA(cudaEventRecord(iter_event(cg, 0), s));
    for (int i = 0; i < k; ++i) {
        const int it = cg->enqueued + i;
        if (cg->opt.use_graph) {
            TW_CUDA(cudaGraphLaunch(cg->graph, s));
        } else if (!tasks) {
            enqueue_mono(cg, x_phase(cg, i, k));
        } else {
            enqueue_iteration_body(cg, it & 1, i == 0, x_phase(cg, i, k));
        }
        if (cg->opt.iteration_marks) {
            // cg_iter=i mark (cg.cpp:307-308): the poller stamps the host time
            // at which it first sees this iteration complete.
            cudaStream_t ms = s;
            if (tasks && !cg->opt.use_graph && cg->opt.dispatch != TW_DISPATCH_CHAIN) {
                for (const PNode& nd : cg->nodes)
                    if (nd.kind == PK_BETA) ms = cg->node_stream(nd);
            }
            cudaEvent_t e = cg->ta->take_event();
            TW_CUDA(cudaEventRecord(e, ms));
            cg->ta->bind(e, &cg->marks[static_cast<size_t>(it)], cg->t0);
            // device-timed iteration end (iter_time of the scenario CSV)
            TW_CUDA(cudaEventRecord(iter_event(cg, it + 1), ms));
        }
    }
    if (!cg->opt.use_graph && tasks) join_streams(cg);
    cg->enqueued += k;
}

void wait_cg(tw_cg* cg) {
    TW_CUDA(cudaSetDevice(cg->ctx->device));
    cudaEvent_t e = cg->ta->take_event();
    TW_CUDA(cudaEventRecord(e, cg->ctx->compute));
    cg->ta->wait(e); // wait_transformed: poll + yield, never a blocking device wait
    cudaEventDestroy(e);
    TW_CUDA(cudaGetLastError());
}

} // namespace cgi
} // namespace tw

using namespace tw::cgi;

namespace tw {
void drop_solve_cache(tw_ctx* ctx, const tw_ell* A) {
    std::lock_guard lk(ctx->solve_mu);
    for (auto it = ctx->solve_cache.begin(); it != ctx->solve_cache.end();) {
        if (A && it->first != A) {
            ++it;
            continue;
        }
        free_cg(it->second);
        it = ctx->solve_cache.erase(it);
    }
}
} // namespace tw

extern "C" {


void tw_cg_options_default(tw_cg_options* o) {
    if (!o) return;
    o->variant = TW_CG_TASKS;
    o->tiles = 16;
    o->stream_pool_capacity = 4;
    o->use_graph = 0;
    o->iteration_marks = 1;
    o->tol = 0.0;
    o->dispatch = TW_DISPATCH_AUTO;
    o->x_update = TW_XUPD_AUTO;
    o->l2_keep = TW_L2KEEP_AUTO;
    o->dag_spmv_slices = 0;
    o->dag_vec_rows = 0;
}

int tw_cg_create(tw_ctx* ctx, const tw_ell* A, const tw_cg_options* opt, int max_iterations,
                 tw_cg** out) {
    return guarded([&] { *out = create_cg(ctx, A, opt, max_iterations); });
}

int tw_cg_destroy(tw_cg* cg) {
    return guarded([&] {
        free_cg(cg);
        (void)cudaGetLastError(); // teardown is best effort: leave no stale error behind
    });
}

int tw_cg_set_rhs(tw_cg* cg, const double* b, int b_is_device) {
    return guarded([&] {
        if (!cg || !b) contract_error("null solver or rhs");
        set_rhs(cg, b, b_is_device != 0);
    });
}

int tw_cg_iterate(tw_cg* cg, int iterations) {
    return guarded([&] {
        if (!cg) contract_error("null solver");
        iterate(cg, iterations);
    });
}

int tw_cg_wait(tw_cg* cg) {
    return guarded([&] {
        if (!cg) contract_error("null solver");
        wait_cg(cg);
    });
}

int tw_cg_iterations_done(tw_cg* cg, int* done) {
    return guarded([&] {
        if (!cg) contract_error("null solver");
        CgScalars sc;
        TW_CUDA(cudaMemcpy(&sc, cg->sc, sizeof(sc), cudaMemcpyDeviceToHost));
        *done = sc.iter;
    });
}

int tw_cg_history(tw_cg* cg, double* host_out, int count) {
    return guarded([&] {
        if (!cg) contract_error("null solver");
        if (count < 0 || count > cg->max_iters) contract_error("history count out of range");
        wait_cg(cg);
        if (count)
            TW_CUDA(cudaMemcpy(host_out, cg->history, sizeof(double) * count, cudaMemcpyDeviceToHost));
    });
}

int tw_cg_solution(tw_cg* cg, double* host_x) {
    return guarded([&] {
        if (!cg) contract_error("null solver");
        wait_cg(cg);
        copy_d2h(cg->ctx, host_x, cg->x, sizeof(double) * static_cast<size_t>(cg->n),
                 cg->ctx->compute);
    });
}

int tw_cg_vectors(tw_cg* cg, double** x, double** r, double** p, double** Ap) {
    return guarded([&] {
        if (!cg) contract_error("null solver");
        if (x) *x = cg->x;
        if (r) *r = cg->r;
        if (p) *p = cg->p_local;
        if (Ap) *Ap = cg->Ap;
    });
}

int tw_cg_iteration_marks(tw_cg* cg, double* host_out, int count) {
    return guarded([&] {
        if (!cg) contract_error("null solver");
        if (count < 0 || count > cg->max_iters) contract_error("mark count out of range");
        wait_cg(cg);
        while (cg->ta->pending()) std::this_thread::yield();
        std::copy(cg->marks.begin(), cg->marks.begin() + count, host_out);
        if (cg->opt.dispatch == TW_DISPATCH_PERSISTENT && count > 0 && cg->opt.iteration_marks) {
            // one launch covers a whole tw_cg_iterate call, so the poller marks
            // only each call's last iteration; earlier ones are placed before
            // that mark by the device's per-iteration clock (d_stamps)
            const int done = std::min(count, cg->enqueued);
            std::vector<unsigned long long> st(static_cast<size_t>(done) + 1);
            TW_CUDA(cudaMemcpy(st.data(), cg->d_stamps, sizeof(unsigned long long) * (done + 1),
                               cudaMemcpyDeviceToHost));
            int real = -1; // the nearest later iteration the poller marked
            for (int i = done - 1; i >= 0; --i) {
                if (cg->mark_real[static_cast<size_t>(i)]) real = i;
                else if (real >= 0)
                    host_out[i] = cg->marks[static_cast<size_t>(real)] -
                                  static_cast<double>(st[real + 1] - st[i + 1]) * 1e-9;
            }
        }
    });
}

int tw_cg_iteration_times(tw_cg* cg, double* seconds, int count) {
    return guarded([&] {
        if (!cg) contract_error("null solver");
        if (!cg->opt.iteration_marks) config_error("iteration times need iteration_marks");
        if (count < 0 || count > cg->enqueued) contract_error("count beyond iterations run");
        wait_cg(cg);
        if (cg->opt.dispatch == TW_DISPATCH_PERSISTENT) {
            std::vector<unsigned long long> st(static_cast<size_t>(count) + 1);
            TW_CUDA(cudaMemcpy(st.data(), cg->d_stamps, sizeof(unsigned long long) * (count + 1),
                               cudaMemcpyDeviceToHost));
            for (int i = 0; i < count; ++i) seconds[i] = static_cast<double>(st[i + 1] - st[i]) * 1e-9;
            return;
        }
        for (int i = 0; i < count; ++i) {
            float ms = 0.f;
            TW_CUDA(cudaEventElapsedTime(&ms, cg->iter_ev[static_cast<size_t>(i)],
                                         cg->iter_ev[static_cast<size_t>(i + 1)]));
            seconds[i] = ms * 1e-3;
        }
    });
}

int tw_cg_task_edges(tw_cg* cg, char* buf, int64_t cap, int64_t* needed) {
    return guarded([&] {
        if (!cg) contract_error("null solver");
        const std::string s = edges_text(cg->dag, std::max(cg->enqueued, 1));
        if (needed) *needed = static_cast<int64_t>(s.size()) + 1;
        if (buf && cap > 0) {
            const int64_t k = std::min<int64_t>(cap - 1, static_cast<int64_t>(s.size()));
            std::memcpy(buf, s.data(), static_cast<size_t>(k));
            buf[k] = '\0';
        }
    });
}

int tw_cg_enable_kernel_timing(tw_cg* cg, int enable) {
    return guarded([&] {
        if (!cg) contract_error("null solver");
        if (enable && cg->opt.variant != TW_CG_MONOLITHIC)
            config_error("kernel timing needs the monolithic variant");
        cg->timing = enable != 0;
        cg->timed = 0;
    });
}

int tw_cg_kernel_times(tw_cg* cg, double* k1, double* k2, double* k3, int* iterations) {
    return guarded([&] {
        if (!cg) contract_error("null solver");
        wait_cg(cg);
        double acc[3] = {0, 0, 0};
        for (int i = 0; i < cg->timed; ++i)
            for (int k = 0; k < 3; ++k) {
                float ms = 0.f;
                TW_CUDA(cudaEventElapsedTime(&ms, cg->tev[static_cast<size_t>(4 * i + k)],
                                             cg->tev[static_cast<size_t>(4 * i + k + 1)]));
                acc[k] += ms;
            }
        if (k1) *k1 = acc[0];
        if (k2) *k2 = acc[1];
        if (k3) *k3 = acc[2];
        if (iterations) *iterations = cg->timed;
    });
}

int tw_cg_launches_per_iteration(tw_cg* cg, int* kernels, int* collectives) {
    return guarded([&] {
        if (!cg) contract_error("null solver");
        int k = 0, c = 0;
        if (cg->opt.dispatch == TW_DISPATCH_PERSISTENT) {
            k = 0; // one launch per tw_cg_iterate call, whatever its iteration count
        } else if (cg->opt.variant == TW_CG_MONOLITHIC && cg->peer) {
            // K1 (one launch, or interior + boundary), K2 (+wait, publish), K3 (+wait, halo)
            k = peer_k1_fused(cg) ? 3 : 4;
        } else if (cg->opt.variant == TW_CG_MONOLITHIC) {
            k = cg->dist ? 5 : 3;
            c = cg->dist ? 3 : 0;
        } else {
            k = 3 * cg->T + (cg->dist ? 4 : cg->fold_scalars() ? 0 : 2); // one rank: alpha / beta_res fold into the tiles
            c = cg->dist ? 3 : 0;
        }
        if (kernels) *kernels = k;
        if (collectives) *collectives = c;
    });
}

int tw_cg_mode(tw_cg* cg, tw_cg_mode_t* out) {
    return guarded([&] {
        if (!cg || !out) contract_error("null solver / out");
        const EllView v = cg->view();
        tw_cg_mode_t m{};
        m.variant = cg->opt.variant;
        m.tiles = cg->T;
        m.dispatch = cg->opt.dispatch;
        m.use_graph = cg->opt.use_graph;
        if (v.cols16) {
            m.k1_form = v.sx_runs ? TW_K1_STAGED_TABLE : TW_K1_STAGED;
            m.k1_l2_keep = v.sx_keep;
        } else {
            m.k1_form = v.tma_blocks > 0 && v.max_width > 0 &&
                                spmv_tma_smem_bytes(v.max_width) + 4096 <= 227 * 1024
                            ? TW_K1_TMA_GATHER
                            : TW_K1_REGISTER;
        }
        m.x_in_k3 = cg->x_pairs ? 2 : x_in_k3(cg);
        m.transport = cg->ctx->emulated ? TW_TRANSPORT_LOOPBACK
                      : cg->peer        ? TW_TRANSPORT_PEER
                      : cg->dist        ? TW_TRANSPORT_NCCL
                                        : TW_TRANSPORT_NONE;
        m.nranks = cg->P;
        int k = 0, c = 0;
        if (tw_cg_launches_per_iteration(cg, &k, &c) != TW_OK) throw Error(TW_ERR_CONTRACT, g_last_error);
        m.kernels_per_iteration = k;
        m.collectives_per_iteration = c;
        *out = m;
    });
}

int tw_cg_solve(tw_ctx* ctx, const tw_ell* A, const double* b_host, int iterations,
                const tw_cg_options* opt, double* history_out, double* x_out, int* converged) {
    return guarded([&] {
        if (!ctx || !A) contract_error("null context or matrix");
        // one solver per matrix kept between calls (no per-call allocation of
        // x | r | p | Ap); reused when the options match and it holds enough
        // history, rebuilt otherwise; set_rhs resets its whole state
        std::lock_guard lk(ctx->solve_mu);
        tw_cg_options o;
        tw_cg_options_default(&o);
        if (opt) o = *opt;
        tw_cg*& cg = ctx->solve_cache[A];
        const tw_cg_options& q = cg ? cg->req : o;
        const bool same = q.variant == o.variant && q.tiles == o.tiles &&
                          q.stream_pool_capacity == o.stream_pool_capacity &&
                          q.use_graph == o.use_graph && q.iteration_marks == o.iteration_marks &&
                          q.tol == o.tol && q.dispatch == o.dispatch && q.x_update == o.x_update &&
                          q.l2_keep == o.l2_keep && q.dag_spmv_slices == o.dag_spmv_slices &&
                          q.dag_vec_rows == o.dag_vec_rows;
        if (cg && (!same || cg->max_iters < iterations)) {
            free_cg(cg);
            cg = nullptr;
        }
        if (!cg) {
            cg = create_cg(ctx, A, &o, std::max(iterations, 1));
            cg->req = o;
        }
        try {
            set_rhs(cg, b_host, false);
            iterate(cg, iterations);
            wait_cg(cg);
            std::vector<double> h(static_cast<size_t>(std::max(iterations, 1)));
            if (iterations)
                TW_CUDA(cudaMemcpy(h.data(), cg->history, sizeof(double) * iterations,
                                   cudaMemcpyDeviceToHost));
            if (history_out) std::copy(h.begin(), h.begin() + iterations, history_out);
            if (x_out)
                copy_d2h(ctx, x_out, cg->x, sizeof(double) * static_cast<size_t>(cg->n),
                         ctx->compute);
            if (converged) // CgResult::converged (cg.cpp:392-393)
                *converged = cg->opt.tol > 0 && iterations > 0 && h[iterations - 1] < cg->opt.tol;
        } catch (...) {
            free_cg(cg);
            ctx->solve_cache.erase(A);
            throw;
        }
    });
}

} // extern "C"

