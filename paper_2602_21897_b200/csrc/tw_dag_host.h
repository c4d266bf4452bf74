// Host-side inference of the cg_tasks block-task DAG: the reference's
// spawn_iteration tasks and access regions (cg.cpp:166-334) and the
// RAW/WAR/WAW rule of its depsys (dep_system.cpp:22-65),
// plus the fused physical nodes the CUDA executors launch.  No device code.
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <string>
#include <utility>
#include <vector>

namespace tw {

// ------------------------------------------------------ dependency rule
//
// The depsys semantics the reference's tests pin (region_ledger.hpp:11-27,
// dep_system.cpp:22-65), stated per byte: a read depends on the byte's last
// writer; a write or readwrite depends on the last writer and on every read
// since that write.  AccessLog applies the rule directly: it keeps the
// accesses in issue order and, for a new one, walks them newest first while
// some of its bytes still lack their last writer.  A write found there is
// the last writer of the bytes it covers (they close); a read found there
// happened after those bytes' last write, so a new write depends on it
// (the bytes stay open).  Empty intervals take no part.

enum AccMode { ACC_R = 0, ACC_W = 1, ACC_RW = 2 };
struct Acc {
    uint64_t lo, hi; // [lo, hi)
    int mode;
};

class AccessLog {
public:
    // Tasks the access `a` depends on (appended to out, unsorted).
    void depends(const Acc& a, std::vector<int>& out) const {
        if (a.hi <= a.lo) return;
        std::vector<std::pair<uint64_t, uint64_t>> open{{a.lo, a.hi}}, next;
        for (auto it = log_.rbegin(); it != log_.rend() && !open.empty(); ++it) {
            const Acc& e = it->a;
            const bool writes = e.mode != ACC_R;
            if (!writes && a.mode == ACC_R) continue; // read after read
            bool hit = false;
            next.clear();
            for (const auto& [lo, hi] : open) {
                const uint64_t l = std::max(lo, e.lo), h = std::min(hi, e.hi);
                if (l >= h || !writes) {
                    hit = hit || l < h;
                    next.emplace_back(lo, hi);
                    continue;
                }
                hit = true;
                if (lo < l) next.emplace_back(lo, l);
                if (h < hi) next.emplace_back(h, hi);
            }
            if (hit) out.push_back(it->task);
            open.swap(next);
        }
    }
    void add(const Acc& a, int task) {
        if (a.hi > a.lo) log_.push_back(Rec{a, task});
    }

private:
    struct Rec {
        Acc a;
        int task;
    };
    std::vector<Rec> log_;
};

enum PhysKind { PK_HALO, PK_SPMV, PK_ALPHA, PK_UPD, PK_BETA, PK_UPDP };

struct LTask {
    std::string label;
    std::vector<Acc> acc;
    int phys; // physical node index within the iteration
};

// Everything the logical DAG depends on: tile rows, the p band each tile's
// SpMV reads (local x coordinates, inclusive, as make_tile_plan's band), and
// across ranks the ghost-plane geometry.
struct DagSpec {
    int T = 1;
    bool halo = false, glo = false, ghi = false;
    int64_t n = 0, ds = 0, plane = 0;
    std::vector<int64_t> r0, r1, lo, hi;
};

struct PNode {
    PhysKind kind;
    int tile;
    std::vector<int> preds_first; // iteration right after a fork point
    std::vector<int> preds_intra; // same-iteration predecessors (steady state)
    std::vector<int> preds_cross; // previous-iteration predecessors
};


// spawn_iteration's logical tasks of iteration `iter` (and, optionally, the
// physical nodes of one iteration).
void build_logical(const DagSpec& d, int iter, std::vector<LTask>& out,
                   std::vector<PNode>* nodes);
// The dependency rule over `iters` iterations: logical edges (ids = iter * tasks_per_iter
// + k), optional labels and physical node of every logical task.
void logical_edges(const DagSpec& d, int iters, std::vector<std::pair<int, int>>& edges,
                   std::vector<std::string>* labels, std::vector<int>* phys_of);
// "pred succ\n" label lines of logical_edges.
std::string edges_text(const DagSpec& d, int iters);

} // namespace tw
