"""Kernel timeline probe (tuning tool): needs the -DTW_TIMELINE build
(`bash scripts/build_variants.sh tl="-DTW_TIMELINE"`, then
TW_HPCCG_LIB=.../libtw_hpccg_tl.so).  Every CTA of K1 / K2 / K3 / the
combine kernel records its SM, first row and entry / exit globaltimer; this
groups them into launches and prints, per executor, the mean span of each
phase and the gaps between phases over the timed iterations.

    python scripts/timeline.py [nx] [iters]
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_21897_b200 as P  # noqa: E402
from paper_2602_21897_b200 import _native as N  # noqa: E402

TAGS = {1: "K1", 2: "K2", 3: "K3", 4: "comb"}
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 128
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
lib = N.load()
lib.tw_timeline_fetch.argtypes = [ctypes.c_void_p, ctypes.c_int]
rt = P.Runtime(0)
A = P.gen_stencil_matrix(nx, nx, nx, rt=rt)
b = P.rhs_xorshift(rt, A.n, 7)
buf = np.zeros((1 << 20, 4), dtype=np.uint64)


def launches(rec):
    """CTA records -> launches: per (tag, first row), split where a CTA
    starts after every earlier CTA of that key has ended (the next
    iteration's instance of the same tile kernel)."""
    out = []
    key = (rec[:, 0] & 0xFF) * (1 << 40) + rec[:, 1]
    for k in np.unique(key):
        r = rec[key == k]
        r = r[np.argsort(r[:, 2])]
        s0, e0, n = r[0, 2], r[0, 3], 1
        for t0, t1 in r[1:, 2:4]:
            if t0 > e0:
                out.append((int(k >> 40), s0, e0, n))
                s0, e0, n = t0, t1, 1
            else:
                e0, n = max(e0, t1), n + 1
        out.append((int(k >> 40), s0, e0, n))
    out.sort(key=lambda x: x[1])
    return out


def probe(name, variant, **kw):
    S = P.CgSolver(rt, A, K + 10, P.CgOptions(iteration_marks=False, **kw), variant=variant)
    S.set_rhs(b)
    S.iterate(6)
    S.wait()
    lib.tw_timeline_reset()
    torch.cuda.synchronize()
    S.iterate(K)
    S.wait()
    n = lib.tw_timeline_fetch(buf.ctypes.data, buf.shape[0])
    S.close()
    rec = buf[:n].astype(np.int64)
    L = launches(rec)
    t_first = L[0][1]
    # phases: consecutive launches of one tag form a phase
    phases = []
    for tag, s, e, nb in L:
        if phases and phases[-1][0] == tag and s < phases[-1][2] + 500:
            ph = phases[-1]
            phases[-1] = (tag, min(ph[1], s), max(ph[2], e), ph[3] + 1)
        else:
            phases.append((tag, s, e, 1))
    span = (phases[-1][2] - phases[0][1]) / 1e3
    k1 = [p for p in phases if p[0] == 1]
    per_it = span / max(len(k1), 1)
    print(f"{name}: {len(L)} launches, {len(phases)} phases, {per_it:.1f} us per iteration "
          f"(first K1 to last kernel end over {len(k1)} iterations)")
    stats = {}
    for i in range(1, len(phases)):
        a, c = phases[i - 1], phases[i]
        g = (c[1] - a[2]) / 1e3
        stats.setdefault(f"gap {TAGS[a[0]]}->{TAGS[c[0]]}", []).append(g)
    for p in phases:
        stats.setdefault(f"span {TAGS[p[0]]} ({p[3]} launches)", []).append((p[2] - p[1]) / 1e3)
    for k, v in sorted(stats.items()):
        print(f"   {k:28s} mean {np.mean(v):7.2f} us  min {np.min(v):7.2f}  max {np.max(v):7.2f}  n={len(v)}")
    # per-launch detail of one middle iteration
    mid = k1[len(k1) // 2][1]
    nxt = [p for p in k1 if p[1] > mid]
    end = nxt[0][1] if nxt else L[-1][2]
    print("   one iteration (us from its first K1 start):")
    for tag, s, e, nb in L:
        if mid <= s < end:
            print(f"     {TAGS[tag]:4s} {(s - mid) / 1e3:8.2f} -> {(e - mid) / 1e3:8.2f}  ({nb} CTAs)")
    del t_first


probe("mono graph", 0, tiles=1, use_graph=True)
probe("T4 graphK", 1, tiles=4, use_graph=True)
probe("T4 streams", 1, tiles=4)
probe("T4 chain graphK", 1, tiles=4, use_graph=True, chain=True)
