// Host-side block-task DAG inference (see tw_dag_host.h).
#include "tw_dag_host.h"

#include <algorithm>
#include <cstring>
#include <sstream>

#include "tw_objects.h"

namespace tw {

namespace {

// Synthetic byte addresses for the dependency rule: one 2^40-byte window per array,
// element i of array k at (k << 40) + 8 i.  Only overlap matters for edges.
enum Arr : uint64_t { A_X = 1, A_R, A_P, A_AP, A_PA, A_RR, A_RTRANS, A_ALPHA, A_BETA };
Acc reg(Arr a, int64_t i0, int64_t i1, int mode) {
    return Acc{(static_cast<uint64_t>(a) << 40) + 8u * static_cast<uint64_t>(i0),
               (static_cast<uint64_t>(a) << 40) + 8u * static_cast<uint64_t>(i1), mode};
}

// spawn_iteration (cg.cpp:166-334): same tasks, labels and access regions;
// plus, across GPUs, a halo task that refreshes p's ghost planes.  p is
// addressed in local x coordinates (ghost planes included).
} // namespace

void build_logical(const DagSpec& d, int iter, std::vector<LTask>& out,
                   std::vector<PNode>* nodes) {
    const int T = d.T;
    const int64_t ds = d.ds;
    auto tag = [iter](const char* fam, int t) {
        return std::string(fam) + ":" + std::to_string(iter) + ":" + std::to_string(t);
    };
    out.clear();
    const bool halo = d.halo;
    const int off_spmv = halo ? 1 : 0, off_alpha = off_spmv + T, off_upd = off_alpha + 1,
              off_beta = off_upd + T, off_updp = off_beta + 1;
    if (nodes) {
        nodes->clear();
        if (halo) nodes->push_back(PNode{PK_HALO, 0, {}, {}, {}});
        for (int t = 0; t < T; ++t) nodes->push_back(PNode{PK_SPMV, t, {}, {}, {}});
        nodes->push_back(PNode{PK_ALPHA, 0, {}, {}, {}});
        for (int t = 0; t < T; ++t) nodes->push_back(PNode{PK_UPD, t, {}, {}, {}});
        nodes->push_back(PNode{PK_BETA, 0, {}, {}, {}});
        for (int t = 0; t < T; ++t) nodes->push_back(PNode{PK_UPDP, t, {}, {}, {}});
    }
    if (halo) {
        std::vector<Acc> acc;
        const int64_t n = d.n, pl = d.plane;
        if (d.glo) {
            acc.push_back(reg(A_P, ds, ds + pl, ACC_R));
            acc.push_back(reg(A_P, 0, pl, ACC_W));
        }
        if (d.ghi) {
            acc.push_back(reg(A_P, ds + n - pl, ds + n, ACC_R));
            acc.push_back(reg(A_P, ds + n, ds + n + pl, ACC_W));
        }
        out.push_back(LTask{tag("halo", 0), acc, 0});
    }
    for (int t = 0; t < T; ++t)
        out.push_back(LTask{tag("spmv", t),
                            {reg(A_P, d.lo[t], d.hi[t] + 1, ACC_R),
                             reg(A_AP, d.r0[t], d.r1[t], ACC_W)},
                            off_spmv + t});
    for (int t = 0; t < T; ++t)
        out.push_back(LTask{tag("dot_pAp", t),
                            {reg(A_P, ds + d.r0[t], ds + d.r1[t], ACC_R),
                             reg(A_AP, d.r0[t], d.r1[t], ACC_R), reg(A_PA, t, t + 1, ACC_W)},
                            off_spmv + t});
    out.push_back(LTask{tag("alpha", 0),
                        {reg(A_PA, 0, T, ACC_R), reg(A_RTRANS, 0, 1, ACC_R),
                         reg(A_ALPHA, 0, 1, ACC_W)},
                        off_alpha});
    for (int t = 0; t < T; ++t)
        out.push_back(LTask{tag("x_up", t),
                            {reg(A_ALPHA, 0, 1, ACC_R),
                             reg(A_P, ds + d.r0[t], ds + d.r1[t], ACC_R),
                             reg(A_X, d.r0[t], d.r1[t], ACC_RW)},
                            off_upd + t});
    for (int t = 0; t < T; ++t)
        out.push_back(LTask{tag("r_up", t),
                            {reg(A_ALPHA, 0, 1, ACC_R), reg(A_AP, d.r0[t], d.r1[t], ACC_R),
                             reg(A_R, d.r0[t], d.r1[t], ACC_RW)},
                            off_upd + t});
    for (int t = 0; t < T; ++t)
        out.push_back(LTask{tag("dot_rr", t),
                            {reg(A_R, d.r0[t], d.r1[t], ACC_R), reg(A_RR, t, t + 1, ACC_W)},
                            off_upd + t});
    out.push_back(LTask{tag("beta_res", 0),
                        {reg(A_RR, 0, T, ACC_R), reg(A_RTRANS, 0, 1, ACC_RW),
                         reg(A_BETA, 0, 1, ACC_W)},
                        off_beta});
    for (int t = 0; t < T; ++t)
        out.push_back(LTask{tag("p_up", t),
                            {reg(A_BETA, 0, 1, ACC_R), reg(A_R, d.r0[t], d.r1[t], ACC_R),
                             reg(A_P, ds + d.r0[t], ds + d.r1[t], ACC_RW)},
                            off_updp + t});
}

// Runs the dependency rule over `iters` iterations; returns logical edges (global
// task ids = iter * tasks_per_iter + k) and, optionally, the label list.
void logical_edges(const DagSpec& d, int iters, std::vector<std::pair<int, int>>& edges,
                   std::vector<std::string>* labels, std::vector<int>* phys_of) {
    AccessLog log;
    std::vector<LTask> it_tasks;
    int base = 0;
    for (int it = 0; it < iters; ++it) {
        build_logical(d, it, it_tasks, nullptr);
        for (size_t k = 0; k < it_tasks.size(); ++k) {
            const int id = base + static_cast<int>(k);
            std::vector<int> pr;
            for (const Acc& a : it_tasks[k].acc) log.depends(a, pr);
            std::sort(pr.begin(), pr.end());
            pr.erase(std::unique(pr.begin(), pr.end()), pr.end());
            for (int p : pr)
                if (p != id) edges.emplace_back(p, id);
            for (const Acc& a : it_tasks[k].acc) log.add(a, id);
            if (labels) labels->push_back(it_tasks[k].label);
            if (phys_of) phys_of->push_back(it_tasks[k].phys);
        }
        base += static_cast<int>(it_tasks.size());
    }
    std::sort(edges.begin(), edges.end());
}

std::string edges_text(const DagSpec& d, int iters) {
    std::vector<std::pair<int, int>> edges;
    std::vector<std::string> labels;
    logical_edges(d, iters, edges, &labels, nullptr);
    std::ostringstream os;
    for (auto [a, b] : edges) os << labels[static_cast<size_t>(a)] << ' ' << labels[static_cast<size_t>(b)] << '\n';
    return os.str();
}

} // namespace tw

using namespace tw;

extern "C" int tw_task_dag_edges(int64_t n_rows, int tiles, const int64_t* r0, const int64_t* r1,
                      const int64_t* band_lo, const int64_t* band_hi, int64_t diag_shift,
                      int64_t plane, int ghost_lo, int ghost_hi, int iterations, char* buf,
                      int64_t cap, int64_t* needed) {
    return guarded([&] {
        if (tiles < 1 || n_rows < tiles) config_error("tile plan needs 1 <= tiles <= rows");
        if (iterations < 1) config_error("iterations must be positive");
        DagSpec d;
        d.T = tiles;
        d.n = n_rows;
        d.ds = diag_shift;
        d.plane = plane;
        d.glo = ghost_lo != 0;
        d.ghi = ghost_hi != 0;
        d.halo = d.glo || d.ghi;
        d.r0.assign(r0, r0 + tiles);
        d.r1.assign(r1, r1 + tiles);
        d.lo.assign(band_lo, band_lo + tiles);
        d.hi.assign(band_hi, band_hi + tiles);
        const std::string s = edges_text(d, iterations);
        if (needed) *needed = static_cast<int64_t>(s.size()) + 1;
        if (buf && cap > 0) {
            const int64_t k = std::min<int64_t>(cap - 1, static_cast<int64_t>(s.size()));
            std::memcpy(buf, s.data(), static_cast<size_t>(k));
            buf[k] = '\0';
        }
    });
}

