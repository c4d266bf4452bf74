"""Stress of the multi-rank persistent dispatcher (one GPU, every rank's task
table in one launch, cross-rank edges as peer-protocol flag waits): random
grids, rank and tile counts, call splits and re-solves, every history
compared with the single-domain oracle and every rank's with rank 0's.
Usage: python scripts/stress_dispatcher.py [cases] [seed]"""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2602_21897_b200 as P  # noqa: E402
from conftest import check_history, rel_gap  # noqa: E402
from oracle import Oracle  # noqa: E402

ncases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
o = Oracle()
fails = solves = spread = 0


def ref_spread(m, b, iters, want_h, want_x):
    """Per iteration, the largest relative gap between the reference's
    cg_reference history and its tiled cg_tasks histories (the oracle's
    tile-order restatement, pinned bitwise to the reference), and the
    largest elementwise gap of their final x."""
    sp, sx = np.zeros(iters), 1e-10
    for t in (2, 4, 8, 16, 32, 64, 128):
        if t <= m.n:
            h, x, _ = o.cg(m, b, iters, tiles=t)
            sp = np.maximum(sp, rel_gap(h, want_h))
            sx = max(sx, float(rel_gap(x, want_x).max()))
    return sp, sx


for c in range(ncases):
    ranks = rng.choice([2, 3, 4, 5, 8])
    nz = ranks * rng.choice([1, 2, 3, 5, 8])
    nx = rng.choice([8, 13, 30, 32, 48, 64])
    ny = rng.choice([4, 9, 16, 24])
    rows_per_rank = nx * ny * (nz // ranks)
    T = rng.choice([t for t in (1, 2, 4, 7, 16, 32) if t <= rows_per_rank])
    iters = rng.choice([15, 30])
    m = o.stencil(nx, ny, nz)
    try:
        G = P.EmulatedRankGroup(nx, ny, nz, ranks, iters, variant=1, transport="peer",
                                options=P.CgOptions(tiles=T, persistent=True,
                                                    iteration_marks=False))
    except P.ConfigError as e:  # e.g. a slab too thin for its tiles
        print("skip", (nx, ny, nz), ranks, T, str(e)[:80])
        continue
    for rd in range(2):
        b = o.rhs_xorshift(m.n, 3 + rd + c)
        want_h, want_x, _ = o.cg(m, b, iters)
        G.set_rhs(b)
        k = rng.randint(1, iters - 1)
        G.iterate(k)
        G.iterate(iters - k)
        hs = G.history(iters)
        x = G.solution()
        solves += 1
        try:
            assert all(np.array_equal(h, hs[0]) for h in hs)
            check_history(hs[0], want_h)
            assert np.all(rel_gap(x, want_x) <= 1e-10)
        except AssertionError as e:
            # near exact convergence of a tiny system (res_k / res_0 ~ 1e-15,
            # the window's edge) the reference's own tiled cg_tasks leaves
            # the rule too: such a case counts when the GPU's gap exceeds
            # twice the largest gap of the reference's tile orders there
            sp, sx = ref_spread(m, b, iters, want_h, want_x)
            g = rel_gap(hs[0], want_h)
            res0 = abs(want_h[0])
            inside = np.abs(want_h) >= 1e-15 * res0
            # the iterations that break the rule: inside the window a
            # relative gap > 1e-10, after it an absolute one > 1e-10 res_0
            bad = np.where(inside, g > 1e-10, np.abs(hs[0] - want_h) > 1e-10 * res0)
            same = all(np.array_equal(h, hs[0]) for h in hs)
            if same and bad.any() and np.all(g[bad] <= 2 * sp[bad]) and \
                    np.all(rel_gap(x, want_x) <= 2 * sx):
                spread += 1
                k = int(np.argmax(np.where(bad, g, 0)))
                print("SPREAD", (nx, ny, nz), ranks, T, rd, f"it {k} gap {g[k]:.2e} ref spread {sp[k]:.2e} "
                      f"res/res0 {abs(want_h[k]) / res0:.1e}", flush=True)
                continue
            fails += 1
            print("FAIL", (nx, ny, nz), ranks, T, rd, str(e)[:200], flush=True)
    G.close()
    print("done", (nx, ny, nz), "ranks", ranks, "tiles", T, flush=True)
print(f"stress: {solves} solves, {fails} failures, {spread} within the reference's own tile-order spread")
sys.exit(1 if fails else 0)
