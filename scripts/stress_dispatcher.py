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
fails = solves = 0
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
            fails += 1
            print("FAIL", (nx, ny, nz), ranks, T, rd, str(e)[:200], flush=True)
    G.close()
    print("done", (nx, ny, nz), "ranks", ranks, "tiles", T, flush=True)
print(f"stress: {solves} solves, {fails} failures")
sys.exit(1 if fails else 0)
