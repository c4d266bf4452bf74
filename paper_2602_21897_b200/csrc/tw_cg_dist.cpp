// Multi-rank CG transports of libtw_hpccg: the phases of
// one rank's distributed monolithic iteration over a z-slab -- NCCL (halo
// send/recv group + allgathers on the comm stream) and the NVLink peer
// transport (halo and scalar partials stored into the other ranks' memory
// by the kernels, flag waits fused into their consumers; tw_peer.cu) -- the
// CUDA-IPC setup of the peer transport, and the emulated rank group that
// runs P ranks on one device (host-sequenced, or as one cooperative kernel).
#include <algorithm>
#include <cstring>
#include <string>

#include "tw_cg_state.h"

namespace tw {
namespace cgi {

// Every NCCL call of the communicator is issued on the one comm stream, so
// the halo and the scalar allgathers are strictly ordered there; the caller's
// stream is joined in and out with events.
void allgather1(tw_cg* cg, const double* send, double* recv, cudaStream_t s) {
    cudaStream_t c = cg->ctx->comm;
    TW_CUDA(cudaEventRecord(cg->ag_in_ev, s));
    TW_CUDA(cudaStreamWaitEvent(c, cg->ag_in_ev, 0));
    TW_NCCL(nccl().AllGather(send, recv, 1, ncclDouble, cg->ctx->nccl_comm, c));
    TW_CUDA(cudaEventRecord(cg->ag_out_ev, c));
    TW_CUDA(cudaStreamWaitEvent(s, cg->ag_out_ev, 0));
}

// p_local: the buffer the next K1 reads (the pair buffer in the second
// iteration of an x-update pair), by default p_local
void halo_exchange(tw_cg* cg, cudaStream_t s, double* p_local) {
    const auto& api = nccl();
    const size_t pl = static_cast<size_t>(cg->plane);
    const int rank = cg->ctx->rank;
    const tw_slab_t& sp = cg->slab;
    double* p = p_local ? p_local : cg->p_local;
    TW_NCCL(api.GroupStart());
    if (sp.ghost_lo) {
        TW_NCCL(api.Recv(p + sp.recv_lo, pl, ncclDouble, rank - 1, cg->ctx->nccl_comm, s));
        TW_NCCL(api.Send(p + sp.send_lo, pl, ncclDouble, rank - 1, cg->ctx->nccl_comm, s));
    }
    if (sp.ghost_hi) {
        TW_NCCL(api.Recv(p + sp.recv_hi, pl, ncclDouble, rank + 1, cg->ctx->nccl_comm, s));
        TW_NCCL(api.Send(p + sp.send_hi, pl, ncclDouble, rank + 1, cg->ctx->nccl_comm, s));
    }
    TW_NCCL(api.GroupEnd());
}

// Phases of one rank's distributed monolithic iteration.  The NCCL path
// interleaves them with the halo and the allgathers (enqueue_mono); the
// emulated rank group (tw_cg_group_iterate) runs them rank by rank with
// loopback copies in place of NCCL.
// On an x-staged slab both launches are the staged K1 (the peer transport's
// one-launch form walks the same two index spaces, so the sums agree to the bit).
void dist_spmv_interior(tw_cg* cg, cudaStream_t s, const double* p_local) { // rows that read no ghost plane
    const double* p = p_local ? p_local : cg->p_local;
    const RowRange ri{cg->slab.interior_r0, cg->slab.interior_r1};
    if (launch_spmv_staged(cg->view(), p, cg->Ap, ri, cg->slot(0),
                           Fin{FIN_STORE, cg->pm, nullptr, nullptr}, s))
        return;
    launch_spmv(cg->view(), p, cg->Ap, RowRange{cg->slab.interior_r0, cg->slab.interior_r1},
                RowRange{0, 0}, true, cg->slot(0), Fin{FIN_STORE, cg->pm, nullptr, nullptr},
                launch_blocks(cg, true), s);
}

void dist_spmv_boundary(tw_cg* cg, cudaStream_t s, const double* p_local) { // the ghost-reading planes, then p.Ap
    const double* p = p_local ? p_local : cg->p_local;
    if (!launch_spmv_staged(cg->view(), p, cg->Ap, RowRange{0, cg->slab.interior_r0},
                            RowRange{cg->slab.interior_r1, cg->n}, RowRange{0, 0}, false,
                            cg->slot(0), Fin{FIN_STORE, cg->pm + 1, nullptr, nullptr}, s))
        launch_spmv(cg->view(), p, cg->Ap, RowRange{0, cg->slab.interior_r0},
                RowRange{cg->slab.interior_r1, cg->n}, true, cg->slot(0),
                    Fin{FIN_STORE, cg->pm + 1, nullptr, nullptr}, launch_blocks(cg, true), s);
    launch_combine(cg->pm, 2, Fin{FIN_STORE, cg->send_a, nullptr, nullptr}, s);
}

void dist_update_xr(tw_cg* cg, cudaStream_t s) { // alpha from the rank partials, local r.r
    launch_update_xr(0, cg->n, x_in_k3(cg) ? nullptr : cg->x, cg->p_owned, cg->r, cg->Ap, cg->sc,
                     ScalarSrc{cg->recv_a, cg->P}, cg->slot(0),
                     Fin{FIN_STORE, cg->send_b, nullptr, nullptr}, launch_blocks(cg, false), s);
}

void dist_update_p(tw_cg* cg, cudaStream_t s, int xph) { // beta from the rank partials; commit
    const ScalarSrc bs{cg->recv_b, cg->P};
    const int bv = launch_blocks(cg, false);
    if (xph == XPH_DEFER) // p_k+1 into the pair buffer, x left alone
        launch_update_p(0, cg->n, cg->r, cg->p2_owned, cg->sc, bs, cg->slot(0), cg->history, bv,
                        s, nullptr, cg->p_owned, false, nullptr);
    else if (xph == XPH_PAIR) // both x updates; p_k+2 back into p_owned
        launch_update_p(0, cg->n, cg->r, cg->p_owned, cg->sc, bs, cg->slot(0), cg->history, bv,
                        s, nullptr, cg->p2_owned, false, cg->x, cg->p_owned);
    else
        launch_update_p(0, cg->n, cg->r, cg->p_owned, cg->sc, bs, cg->slot(0), cg->history, bv,
                        s, nullptr, nullptr, false, x_in_k3(cg) ? cg->x : nullptr);
}

// Phases of the peer transport (NVLink stores + flags, fused into the
// kernels): 4 launches per iteration and no collective call.
// Whether the peer K1 runs as one launch (launch_spmv_split's conditions).
bool peer_k1_fused(const tw_cg* cg) {
    const EllView A = cg->view();
    if (A.max_width <= 0 || A.tma_blocks <= 0) return false;
    if ((A.cols16 ? spmv_staged_smem_bytes(A.max_width) : spmv_tma_smem_bytes(A.max_width)) + 2048 >
        227 * 1024)
        return false;
    auto slices = [](int64_t r0, int64_t r1) { return r1 > r0 ? ((r1 + 31) >> 5) - (r0 >> 5) : 0; };
    const int64_t full = static_cast<int64_t>(A.tma_blocks) * spmv_tma_warps();
    return slices(cg->slab.interior_r0, cg->slab.interior_r1) >= full &&
           slices(0, cg->slab.interior_r0) + slices(cg->slab.interior_r1, cg->n) >= full;
}

void peer_spmv(tw_cg* cg, cudaStream_t s, int xph) {
    // p of this iteration (and its ghost planes): the pair buffer in the
    // second iteration of an x-update pair
    const double* pl = xph == XPH_PAIR ? cg->p2_local : cg->p_local;
    const int ng = cg->slab.ghost_lo + cg->slab.ghost_hi;
    const unsigned long long* gf = cg->slab.ghost_lo ? &cg->win->flag_ghost_lo : &cg->win->flag_ghost_hi;
    const Fin fin{FIN_PUBLISH_A, cg->pm + 1, cg->sc, nullptr, cg->d_links, cg->pm};
    const RowRange ri{cg->slab.interior_r0, cg->slab.interior_r1}, b0{0, cg->slab.interior_r0},
        b1{cg->slab.interior_r1, cg->n};
    if (cg->view().cols16) { // x-staged slab: the same two forms with staged x runs
        if (launch_spmv_staged(cg->view(), pl, cg->Ap, ri, b0, b1, true, cg->slot(0), fin,
                               s, ng ? gf : nullptr, ng))
            return;
        dist_spmv_interior(cg, s, pl);
        if (!launch_spmv_staged(cg->view(), pl, cg->Ap, b0, b1, RowRange{0, 0}, false,
                                cg->slot(0), fin, s, ng ? gf : nullptr, ng))
            throw Error(TW_ERR_CUDA, "staged boundary SpMV did not launch after the interior did");
        return;
    }
    // one launch: interior rows first (they read no ghost plane, so they
    // overlap the neighbours' K3 tails), then the boundary rows
    if (launch_spmv_split(cg->view(), pl, cg->Ap,
                          RowRange{cg->slab.interior_r0, cg->slab.interior_r1},
                          RowRange{0, cg->slab.interior_r0}, RowRange{cg->slab.interior_r1, cg->n},
                          cg->slot(0), Fin{FIN_PUBLISH_A, cg->pm + 1, cg->sc, nullptr, cg->d_links, cg->pm},
                          s, ng ? gf : nullptr, ng))
        return;
    dist_spmv_interior(cg, s, pl);
    launch_spmv(cg->view(), pl, cg->Ap, RowRange{0, cg->slab.interior_r0},
                RowRange{cg->slab.interior_r1, cg->n}, true, cg->slot(0),
                Fin{FIN_PUBLISH_A, cg->pm + 1, cg->sc, nullptr, cg->d_links, cg->pm},
                launch_blocks(cg, true), s, ng ? gf : nullptr, ng);
}

void peer_update_xr(tw_cg* cg, cudaStream_t s) {
    launch_update_xr(0, cg->n, x_in_k3(cg) ? nullptr : cg->x, cg->p_owned, cg->r, cg->Ap, cg->sc,
                     ScalarSrc{cg->win->recv_a, cg->P, cg->win->flag_a}, cg->slot(0),
                     Fin{FIN_PUBLISH_B, cg->send_b, cg->sc, nullptr, cg->d_links, nullptr},
                     launch_blocks(cg, false), s);
}

void peer_update_p(tw_cg* cg, cudaStream_t s, int xph) {
    const ScalarSrc bs{cg->win->recv_b, cg->P, cg->win->flag_b};
    const int bv = launch_blocks(cg, false);
    if (xph == XPH_DEFER) // p_k+1 into the pair buffer and the neighbours' pair-buffer ghosts
        launch_update_p(0, cg->n, cg->r, cg->p2_owned, cg->sc, bs, cg->slot(0), cg->history, bv,
                        s, cg->d_links2, cg->p_owned, false, nullptr);
    else if (xph == XPH_PAIR) // both x updates; p_k+2 back into p_owned and its ghosts
        launch_update_p(0, cg->n, cg->r, cg->p_owned, cg->sc, bs, cg->slot(0), cg->history, bv,
                        s, cg->d_links, cg->p2_owned, false, cg->x, cg->p_owned);
    else
        launch_update_p(0, cg->n, cg->r, cg->p_owned, cg->sc, bs, cg->slot(0), cg->history, bv,
                        s, cg->d_links, nullptr, false, x_in_k3(cg) ? cg->x : nullptr);
}

void alloc_window(tw_cg* cg) {
    if (!cg->dist) contract_error("the peer transport needs a multi-rank context");
    if (cg->opt.variant != TW_CG_MONOLITHIC && cg->opt.dispatch != TW_DISPATCH_PERSISTENT)
        config_error("the peer transport runs the monolithic variant or the persistent dispatcher");
    if (cg->P > kMaxRanks) config_error("more ranks than the peer window holds");
    if (!cg->win) {
        TW_CUDA(cudaMalloc(&cg->win, sizeof(PeerWindow)));
        TW_CUDA(cudaMemset(cg->win, 0, sizeof(PeerWindow)));
    }
}

// (the caller set links' windows, flags and ghost targets, and links2's
// ghost targets when the x updates are paired)
void finish_links(tw_cg* cg) {
    cg->links.rank = cg->ctx->rank;
    cg->links.nranks = cg->P;
    cg->links.plane = cg->plane;
    if (!cg->d_links) TW_CUDA(cudaMalloc(&cg->d_links, sizeof(PeerLinks)));
    TW_CUDA(cudaMemcpy(cg->d_links, &cg->links, sizeof(PeerLinks), cudaMemcpyHostToDevice));
    if (cg->x_pairs) {
        PeerLinks L2 = cg->links;
        L2.ghost_lo_dst = cg->links2.ghost_lo_dst;
        L2.ghost_hi_dst = cg->links2.ghost_hi_dst;
        if ((L2.ghost_lo_dst == nullptr) != (cg->links.ghost_lo_dst == nullptr) ||
            (L2.ghost_hi_dst == nullptr) != (cg->links.ghost_hi_dst == nullptr))
            contract_error("a neighbour's pair buffer is missing (all ranks pair their x updates or none)");
        cg->links2 = L2;
        if (!cg->d_links2) TW_CUDA(cudaMalloc(&cg->d_links2, sizeof(PeerLinks)));
        TW_CUDA(cudaMemcpy(cg->d_links2, &cg->links2, sizeof(PeerLinks), cudaMemcpyHostToDevice));
    }
    cg->peer = true;
    if (cg->graph) { // graphs captured before the switch used the NCCL path
        cudaGraphExecDestroy(cg->graph);
        cg->graph = nullptr;
    }
    for (auto& kv : cg->timed_graphs) cudaGraphExecDestroy(kv.second);
    cg->timed_graphs.clear();
    for (auto& kv : cg->chunk_graphs) cudaGraphExecDestroy(kv.second);
    cg->chunk_graphs.clear();
}

// ------------------------------------------------ emulated rank group
//
// P contexts on ONE device, each owning a z-slab, driven phase by phase on a
// single stream.  The NCCL transport is replaced by loopback device copies
// (halo planes into the neighbours' ghost planes, every rank's partial into
// every rank's receive slots); everything else -- slab geometry, ghost
// layout, interior/boundary split, rank-ordered scalar sums -- is the code
// the NCCL path runs.  No kernel ever waits on another: the host sequences
// the phases, so this is safe on one GPU (B200_PROFILING.md).

void group_check(tw_cg** g, int P) {
    if (!g || P < 1) contract_error("empty rank group");
    for (int r = 0; r < P; ++r) {
        if (!g[r]) contract_error("null solver in rank group");
        const tw_ctx* c = g[r]->ctx;
        if (!c->emulated || c->rank != r || c->nranks != P)
            contract_error("rank group entry " + std::to_string(r) +
                           " is not emulated rank r of P (tw_ctx_init_emulated_rank)");
        if (c->device != g[0]->ctx->device) contract_error("emulated ranks share one device");
        if (g[r]->opt.variant != g[0]->opt.variant || g[r]->T != g[0]->T)
            config_error("the ranks of a group run the same variant and tile count");
        if (g[r]->opt.dispatch != g[0]->opt.dispatch)
            config_error("the ranks of a group use the same dispatch");
        if (g[r]->x_pairs != g[0]->x_pairs)
            config_error("the ranks of a group pair their x updates alike");
    }
}

void loopback_allgather(tw_cg** g, int P, double* tw_cg::*send, double* tw_cg::*recv,
                        cudaStream_t s) {
    for (int r = 0; r < P; ++r)
        for (int q = 0; q < P; ++q)
            TW_CUDA(cudaMemcpyAsync(g[r]->*recv + q, g[q]->*send, sizeof(double),
                                    cudaMemcpyDeviceToDevice, s));
}

void loopback_halo(tw_cg** g, int P, cudaStream_t s, int xph) {
    // the buffer this iteration's K1 reads: the pair buffer in the second
    // iteration of an x-update pair
    auto buf = [&](int r) { return xph == XPH_PAIR ? g[r]->p2_local : g[r]->p_local; };
    for (int r = 0; r < P; ++r) {
        const tw_slab_t& sp = g[r]->slab;
        const size_t bytes = sizeof(double) * static_cast<size_t>(sp.plane);
        if (sp.ghost_lo) // my lower ghost <- rank r-1's last owned plane
            TW_CUDA(cudaMemcpyAsync(buf(r) + sp.recv_lo, buf(r - 1) + g[r - 1]->slab.send_hi,
                                    bytes, cudaMemcpyDeviceToDevice, s));
        if (sp.ghost_hi) // my upper ghost <- rank r+1's first owned plane
            TW_CUDA(cudaMemcpyAsync(buf(r) + sp.recv_hi, buf(r + 1) + g[r + 1]->slab.send_lo,
                                    bytes, cudaMemcpyDeviceToDevice, s));
    }
}

// Every rank's compute stream continues after the group's work on s.
void group_join(tw_cg** g, int P, cudaStream_t s) {
    TW_CUDA(cudaEventRecord(g[0]->fork_ev, s));
    for (int r = 1; r < P; ++r) TW_CUDA(cudaStreamWaitEvent(g[r]->ctx->compute, g[0]->fork_ev, 0));
}

// Peer transport inside the emulated group: the "peer" pointers are the
// other ranks' buffers on the same device.
void group_enable_peer(tw_cg** g, int P) {
    group_check(g, P);
    if (g[0]->opt.variant != TW_CG_MONOLITHIC && g[0]->opt.dispatch != TW_DISPATCH_PERSISTENT)
        config_error("the peer transport runs the monolithic variant or the persistent dispatcher");
    for (int r = 0; r < P; ++r)
        if (g[r]->peer) contract_error("the peer transport is already connected");
    TW_CUDA(cudaSetDevice(g[0]->ctx->device));
    for (int r = 0; r < P; ++r) alloc_window(g[r]);
    for (int r = 0; r < P; ++r) {
        PeerLinks& L = g[r]->links;
        L = PeerLinks{};
        for (int q = 0; q < P; ++q) L.win[q] = g[q]->win;
        PeerLinks& L2 = g[r]->links2; // (its ghost targets: the pair buffers)
        L2 = PeerLinks{};
        if (r > 0) {
            L.ghost_lo_dst = g[r - 1]->p_local + g[r - 1]->slab.recv_hi;
            L.ghost_lo_flag = &g[r - 1]->win->flag_ghost_hi;
            if (g[r - 1]->p2_local) L2.ghost_lo_dst = g[r - 1]->p2_local + g[r - 1]->slab.recv_hi;
        }
        if (r + 1 < P) {
            L.ghost_hi_dst = g[r + 1]->p_local + g[r + 1]->slab.recv_lo;
            L.ghost_hi_flag = &g[r + 1]->win->flag_ghost_lo;
            if (g[r + 1]->p2_local) L2.ghost_hi_dst = g[r + 1]->p2_local + g[r + 1]->slab.recv_lo;
        }
        finish_links(g[r]);
    }
}

void group_set_rhs(tw_cg** g, int P, const double* const* b, bool on_device) {
    group_check(g, P);
    TW_CUDA(cudaSetDevice(g[0]->ctx->device));
    for (int r = 0; r < P; ++r) TW_CUDA(cudaStreamSynchronize(g[r]->ctx->compute));
    cudaStream_t s = g[0]->ctx->compute;
    for (int r = 0; r < P; ++r) set_rhs_prefix(g[r], b[r], on_device, s);
    loopback_allgather(g, P, &tw_cg::send_r, &tw_cg::recv_r, s);
    for (int r = 0; r < P; ++r)
        launch_combine(g[r]->recv_r, P, Fin{FIN_RTRANS, nullptr, g[r]->sc, nullptr}, s);
    if (g[0]->peer)
        for (int r = 0; r < P; ++r)
            launch_peer_push(g[r]->p_owned, g[r]->n, g[r]->plane, g[r]->links, g[r]->sc,
                             g[r]->tickets, s);
    TW_CUDA(cudaStreamSynchronize(s));
    for (int r = 0; r < P; ++r) reset_solve_state(g[r]);
}

// One block-task iteration of every rank (cg_tasks' DAG with the halo task,
// spawn_iteration, cg.cpp:166-334): the ranks' physical nodes phase by phase
// -- halo (loopback), the SpMV tiles, alpha (tile-order combine, the
// allgather, the rank-order combine), the x/r tiles, beta_res likewise, the
// p tiles -- with the very kernels and partial orders of the NCCL tasks path
// (launch_node), so its numbers are the multi-GPU executor's.
static void group_tasks_iteration(tw_cg** g, int P, cudaStream_t s, int xph) {
    auto nodes_of = [&](int kind) {
        for (int r = 0; r < P; ++r)
            for (const PNode& nd : g[r]->nodes)
                if (nd.kind == kind) launch_node(g[r], nd, s, xph);
    };
    auto reduce = [&](double* tw_cg::*tile_parts, double* tw_cg::*send, double* tw_cg::*recv,
                      int fin_mode) {
        for (int r = 0; r < P; ++r)
            launch_combine(g[r]->*tile_parts, g[r]->T, Fin{FIN_STORE, g[r]->*send, nullptr, nullptr}, s);
        loopback_allgather(g, P, send, recv, s);
        for (int r = 0; r < P; ++r)
            launch_combine(g[r]->*recv, P, Fin{fin_mode, nullptr, g[r]->sc, g[r]->history}, s);
    };
    loopback_halo(g, P, s, xph);
    nodes_of(PK_SPMV);
    reduce(&tw_cg::pa, &tw_cg::send_a, &tw_cg::recv_a, FIN_ALPHA);
    nodes_of(PK_UPD);
    reduce(&tw_cg::rrp, &tw_cg::send_b, &tw_cg::recv_b, FIN_BETA);
    nodes_of(PK_UPDP);
}

void group_iterate(tw_cg** g, int P, int k) {
    group_check(g, P);
    if (k < 0) config_error("negative iteration count");
    for (int r = 0; r < P; ++r)
        if (g[r]->enqueued + k > g[r]->max_iters) contract_error("iterations beyond max_iterations");
    TW_CUDA(cudaSetDevice(g[0]->ctx->device));
    cudaStream_t s = g[0]->ctx->compute;
    for (int r = 1; r < P; ++r) { // order after anything queued on the other ranks' streams
        TW_CUDA(cudaEventRecord(g[r]->fork_ev, g[r]->ctx->compute));
        TW_CUDA(cudaStreamWaitEvent(s, g[r]->fork_ev, 0));
    }
    const bool tasks = g[0]->opt.variant == TW_CG_TASKS;
    const bool persistent = g[0]->opt.dispatch == TW_DISPATCH_PERSISTENT;
    if (persistent && !g[0]->peer)
        contract_error("the multi-rank dispatcher runs over the peer transport (tw_cg_group_enable_peer)");
    // the block-task DAG of every rank in ONE persistent kernel: the ranks'
    // cross edges are the peer protocol's flag waits, so all ranks run at
    // once in one launch (never as separate launches waiting on each other)
    if (persistent && k > 0) enqueue_persistent(g, P, k);
    for (int it = 0; it < k && tasks && !persistent; ++it)
        group_tasks_iteration(g, P, s, x_phase(g[0], it, k));
    for (int it = 0; it < k && !tasks && g[0]->peer; ++it) { // peer transport: stores + flags
        const int xph = x_phase(g[0], it, k);
        for (int r = 0; r < P; ++r) peer_spmv(g[r], s, xph);
        for (int r = 0; r < P; ++r) peer_update_xr(g[r], s);
        for (int r = 0; r < P; ++r) peer_update_p(g[r], s, xph);
    }
    for (int it = 0; it < k && !tasks && !g[0]->peer; ++it) {
        const int xph = x_phase(g[0], it, k);
        loopback_halo(g, P, s, xph);
        for (int r = 0; r < P; ++r) {
            const double* pl = xph == XPH_PAIR ? g[r]->p2_local : g[r]->p_local;
            dist_spmv_interior(g[r], s, pl);
            dist_spmv_boundary(g[r], s, pl);
        }
        loopback_allgather(g, P, &tw_cg::send_a, &tw_cg::recv_a, s);
        for (int r = 0; r < P; ++r) dist_update_xr(g[r], s);
        loopback_allgather(g, P, &tw_cg::send_b, &tw_cg::recv_b, s);
        for (int r = 0; r < P; ++r) dist_update_p(g[r], s, xph);
    }
    group_join(g, P, s);
    for (int r = 0; r < P; ++r) g[r]->enqueued += k;
}

// The peer-transport group as ONE cooperative kernel (rank_group_kernel):
// the ranks run concurrently and really wait on one another's flags.
void group_iterate_concurrent(tw_cg** g, int P, int k, int jitter) {
    group_check(g, P);
    if (!g[0]->peer) contract_error("the concurrent group runs the peer transport (tw_cg_group_enable_peer)");
    if (k < 0) config_error("negative iteration count");
    for (int r = 0; r < P; ++r)
        if (g[r]->enqueued + k > g[r]->max_iters) contract_error("iterations beyond max_iterations");
    if (k == 0) return;
    TW_CUDA(cudaSetDevice(g[0]->ctx->device));
    cudaStream_t s = g[0]->ctx->compute;
    for (int r = 1; r < P; ++r) {
        TW_CUDA(cudaEventRecord(g[r]->fork_ev, g[r]->ctx->compute));
        TW_CUDA(cudaStreamWaitEvent(s, g[r]->fork_ev, 0));
    }
    // x-staged slabs run the staged K1: kThreads / 32 warp stages per block
    int wmax = 0;
    bool staged = false;
    for (int r = 0; r < P; ++r) {
        staged = staged || g[r]->view().cols16 != nullptr;
        wmax = std::max(wmax, static_cast<int>(g[r]->A->info.max_width));
    }
    int vb = 0, cb = 0;
    const int stage = staged ? staged_stage_bytes(wmax, &vb, &cb) : 0;
    const int smem = staged ? stage * (kGroupThreads / 32) : 0;
    int B = rank_group_blocks_per_rank(P, smem);
    for (int r = 0; r < P; ++r) B = std::min(B, staged ? g[r]->maxg / 2 : g[r]->maxg);
    if (B < 1) config_error("more ranks than co-resident blocks");
    std::vector<GroupRank> h(static_cast<size_t>(P));
    GroupRank* d = nullptr;
    unsigned* bars = nullptr;
    TW_CUDA(cudaMalloc(&d, sizeof(GroupRank) * P));
    TW_CUDA(cudaMalloc(&bars, sizeof(unsigned) * 2 * P));
    TW_CUDA(cudaMemsetAsync(bars, 0, sizeof(unsigned) * 2 * P, s));
    for (int r = 0; r < P; ++r) {
        tw_cg* c = g[r];
        GroupRank& R = h[static_cast<size_t>(r)];
        R.A = c->view();
        R.x = c->x; R.r = c->r; R.p_local = c->p_local; R.p_owned = c->p_owned; R.Ap = c->Ap;
        R.pm = c->pm; R.send_b = c->send_b; R.history = c->history;
        R.sc = c->sc;
        R.rs = c->slot(0);
        R.win = c->win;
        R.links = c->d_links;
        R.n_ghost = c->slab.ghost_lo + c->slab.ghost_hi;
        R.ghost_flags = c->slab.ghost_lo ? &c->win->flag_ghost_lo : &c->win->flag_ghost_hi;
        R.P = P;
        R.n = c->n; R.int_r0 = c->slab.interior_r0; R.int_r1 = c->slab.interior_r1;
        R.bar = bars + 2 * r;
        R.stage_bytes = stage;
        R.val_bytes = vb;
        R.c16_bytes = cb;
    }
    TW_CUDA(cudaMemcpyAsync(d, h.data(), sizeof(GroupRank) * P, cudaMemcpyHostToDevice, s));
    launch_rank_group(d, P, B, k, jitter, smem, s);
    TW_CUDA(cudaStreamSynchronize(s));
    cudaFree(d);
    cudaFree(bars);
    group_join(g, P, s);
    for (int r = 0; r < P; ++r) g[r]->enqueued += k;
}

} // namespace cgi
} // namespace tw

using namespace tw::cgi;

extern "C" {

int tw_cg_group_set_rhs(tw_cg** cgs, int nranks, const double* const* b, int b_is_device) {
    return guarded([&] {
        if (!b) contract_error("null rhs list");
        group_set_rhs(cgs, nranks, b, b_is_device != 0);
    });
}

int tw_cg_group_iterate(tw_cg** cgs, int nranks, int iterations) {
    return guarded([&] { group_iterate(cgs, nranks, iterations); });
}

int tw_cg_group_iterate_concurrent(tw_cg** cgs, int nranks, int iterations, int jitter) {
    return guarded([&] { group_iterate_concurrent(cgs, nranks, iterations, jitter); });
}

int tw_cg_group_enable_peer(tw_cg** cgs, int nranks) {
    return guarded([&] { group_enable_peer(cgs, nranks); });
}

// Transport check of a connected peer transport (collective in two steps:
// every rank sends, then every rank checks -- so on one device, too, no
// kernel ever waits for a kernel that has not been launched).
int tw_cg_peer_ping_send(tw_cg* cg) {
    return guarded([&] {
        if (!cg || !cg->peer) contract_error("the peer transport is not connected");
        TW_CUDA(cudaSetDevice(cg->ctx->device));
        ++cg->ping_seq;
        const unsigned long long token = 0x5057000000000000ull | cg->ping_seq; // 'PW' + round
        launch_peer_ping_send(cg->links, token, cg->ctx->compute);
        TW_CUDA(cudaStreamSynchronize(cg->ctx->compute));
    });
}

int tw_cg_peer_ping_check(tw_cg* cg, int timeout_ms, int* ok) {
    return guarded([&] {
        if (!cg || !cg->peer || !ok) contract_error("the peer transport is not connected");
        if (timeout_ms < 0) config_error("negative timeout");
        TW_CUDA(cudaSetDevice(cg->ctx->device));
        const unsigned long long token = 0x5057000000000000ull | cg->ping_seq;
        int* d_ok = nullptr;
        TW_CUDA(cudaMalloc(&d_ok, sizeof(int)));
        launch_peer_ping_check(cg->win, cg->P, token, static_cast<long long>(timeout_ms) * 1000000LL,
                               d_ok, cg->ctx->compute);
        int h = 0;
        const cudaError_t e = cudaMemcpyAsync(&h, d_ok, sizeof(int), cudaMemcpyDeviceToHost,
                                              cg->ctx->compute);
        const cudaError_t e2 = cudaStreamSynchronize(cg->ctx->compute);
        cudaFree(d_ok);
        TW_CUDA(e);
        TW_CUDA(e2);
        *ok = h;
    });
}

// blob: [0,64) window IPC handle, [64,128) p_base IPC handle, [128,136)
// byte offset of the lower ghost plane in p_base, [136,144) of the upper,
// [144,148) rank, [148,152) rank count, [152,160) plane size (checked on
// connect: a neighbour's ghost planes must match this rank's planes),
// [160,168) byte offset of the pair buffer in p_base (0 without paired x
// updates; all ranks must agree).
int tw_cg_peer_export(tw_cg* cg, unsigned char* blob) {
    return guarded([&] {
        if (!cg || !blob) contract_error("null solver or blob");
        TW_CUDA(cudaSetDevice(cg->ctx->device));
        alloc_window(cg);
        std::memset(blob, 0, TW_PEER_BLOB_BYTES);
        cudaIpcMemHandle_t hw, hp;
        TW_CUDA(cudaIpcGetMemHandle(&hw, cg->win));
        TW_CUDA(cudaIpcGetMemHandle(&hp, cg->p_base));
        std::memcpy(blob, &hw, sizeof(hw));
        std::memcpy(blob + 64, &hp, sizeof(hp));
        const int64_t lo = (cg->p_local + cg->slab.recv_lo - cg->p_base) * static_cast<int64_t>(sizeof(double));
        const int64_t hi = (cg->p_local + cg->slab.recv_hi - cg->p_base) * static_cast<int64_t>(sizeof(double));
        std::memcpy(blob + 128, &lo, 8);
        std::memcpy(blob + 136, &hi, 8);
        const int rank = cg->ctx->rank, nranks = cg->P;
        std::memcpy(blob + 144, &rank, 4);
        std::memcpy(blob + 148, &nranks, 4);
        const int64_t plane = cg->plane;
        std::memcpy(blob + 152, &plane, 8); // a neighbour's ghost planes must be this size
        // paired x updates: the pair buffer's byte offset from p_base (0: none)
        const int64_t p2 = cg->p2_base ? (cg->p2_base - cg->p_base) * static_cast<int64_t>(sizeof(double)) : 0;
        std::memcpy(blob + 160, &p2, 8);
    });
}

int tw_cg_peer_connect(tw_cg* cg, const unsigned char* blobs) {
    return guarded([&] {
        if (!cg || !blobs) contract_error("null solver or blobs");
        if (cg->peer) contract_error("the peer transport is already connected");
        TW_CUDA(cudaSetDevice(cg->ctx->device));
        alloc_window(cg);
        const int P = cg->P, me = cg->ctx->rank;
        PeerLinks& L = cg->links;
        L = PeerLinks{};
        cg->links2 = PeerLinks{};
        auto open = [&](const unsigned char* h) {
            cudaIpcMemHandle_t mh;
            std::memcpy(&mh, h, sizeof(mh));
            void* p = nullptr;
            TW_CUDA(cudaIpcOpenMemHandle(&p, mh, cudaIpcMemLazyEnablePeerAccess));
            cg->ipc_mapped.push_back(p);
            return static_cast<unsigned char*>(p);
        };
        for (int q = 0; q < P; ++q) { // validate every blob before mapping any
            const unsigned char* b = blobs + static_cast<size_t>(q) * TW_PEER_BLOB_BYTES;
            int rq = -1, pq = -1;
            int64_t plane_q = -1;
            std::memcpy(&rq, b + 144, 4);
            std::memcpy(&pq, b + 148, 4);
            std::memcpy(&plane_q, b + 152, 8);
            if (rq != q) contract_error("peer blobs must be in rank order");
            if (pq != P) contract_error("peer blob of a different rank count");
            if (plane_q != cg->plane) contract_error("peer blob of a different plane size (nx * ny)");
            int64_t p2_q = 0;
            std::memcpy(&p2_q, b + 160, 8);
            if ((p2_q != 0) != cg->x_pairs)
                contract_error("peer blob of a rank that pairs its x updates differently");
        }
        for (int q = 0; q < P; ++q) {
            const unsigned char* b = blobs + static_cast<size_t>(q) * TW_PEER_BLOB_BYTES;
            if (q == me) {
                L.win[q] = cg->win;
                continue;
            }
            auto* w = reinterpret_cast<PeerWindow*>(open(b));
            L.win[q] = w;
            if (q == me - 1 || q == me + 1) {
                unsigned char* pb = open(b + 64);
                int64_t lo = 0, hi = 0, p2 = 0;
                std::memcpy(&lo, b + 128, 8);
                std::memcpy(&hi, b + 136, 8);
                std::memcpy(&p2, b + 160, 8);
                if (q == me - 1) { // my first plane -> its upper ghost
                    L.ghost_lo_dst = reinterpret_cast<double*>(pb + hi);
                    L.ghost_lo_flag = &w->flag_ghost_hi;
                    if (p2) cg->links2.ghost_lo_dst = reinterpret_cast<double*>(pb + p2 + hi);
                } else {           // my last plane -> its lower ghost
                    L.ghost_hi_dst = reinterpret_cast<double*>(pb + lo);
                    L.ghost_hi_flag = &w->flag_ghost_lo;
                    if (p2) cg->links2.ghost_hi_dst = reinterpret_cast<double*>(pb + p2 + lo);
                }
            }
        }
        finish_links(cg);
    });
}

} // extern "C"
