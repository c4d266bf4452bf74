// Host-side inference of the cg_tasks block-task DAG: the reference's
// spawn_iteration tasks and access regions (cg.cpp:166-334) and the
// RAW/WAR/WAW rules of its depsys (region_ledger.cpp, dep_system.cpp:22-65),
// plus the fused physical nodes the CUDA executors launch.  No device code.
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <string>
#include <utility>
#include <vector>

namespace tw {

// --------------------------------------------------------------- ledger
//
// Byte-interval dependency inference with the reference's rules
// (region_ledger.hpp:11-27): a read conflicts with the last writer; a write
// or readwrite conflicts with the last writer and every reader since.

enum AccMode { ACC_R = 0, ACC_W = 1, ACC_RW = 2 };
struct Acc {
    uint64_t lo, hi; // [lo, hi)
    int mode;
};

class Ledger {
public:
    void conflicts(const Acc& a, std::vector<int>& out) const {
        auto it = seg_.upper_bound(a.lo);
        if (it != seg_.begin()) --it;
        for (; it != seg_.end() && it->first < a.hi; ++it) {
            const Seg& s = it->second;
            if (s.hi <= a.lo) continue;
            if (s.writer >= 0) out.push_back(s.writer);
            if (a.mode != ACC_R) out.insert(out.end(), s.readers.begin(), s.readers.end());
        }
    }
    void record(const Acc& a, int task) {
        split(a.lo);
        split(a.hi);
        if (a.mode != ACC_R) {
            seg_.erase(seg_.lower_bound(a.lo), seg_.lower_bound(a.hi));
            seg_[a.lo] = Seg{a.hi, task, {}};
            return;
        }
        uint64_t pos = a.lo;
        auto it = seg_.lower_bound(a.lo);
        while (pos < a.hi) {
            if (it == seg_.end() || it->first >= a.hi) {
                seg_[pos] = Seg{a.hi, -1, {task}};
                break;
            }
            if (it->first > pos) {
                seg_[pos] = Seg{it->first, -1, {task}};
                pos = it->first;
                continue;
            }
            auto& rd = it->second.readers;
            if (std::find(rd.begin(), rd.end(), task) == rd.end()) rd.push_back(task);
            pos = it->second.hi;
            ++it;
        }
    }

private:
    struct Seg {
        uint64_t hi;
        int writer;
        std::vector<int> readers;
    };
    void split(uint64_t x) {
        auto it = seg_.upper_bound(x);
        if (it == seg_.begin()) return;
        --it;
        if (it->first == x || it->second.hi <= x) return;
        Seg right = it->second;
        it->second.hi = x;
        seg_[x] = std::move(right);
    }
    std::map<uint64_t, Seg> seg_;
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
// Ledger over `iters` iterations: logical edges (ids = iter * tasks_per_iter
// + k), optional labels and physical node of every logical task.
void logical_edges(const DagSpec& d, int iters, std::vector<std::pair<int, int>>& edges,
                   std::vector<std::string>* labels, std::vector<int>* phys_of);
// "pred succ\n" label lines of logical_edges.
std::string edges_text(const DagSpec& d, int iters);

} // namespace tw
