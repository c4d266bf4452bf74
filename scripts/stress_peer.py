"""Stress of the peer protocol under real concurrency (one GPU, all ranks in
one cooperative kernel): many solves with rank-dependent delays, every
history compared with the single-domain oracle.  Usage: python
scripts/stress_peer.py [rounds]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2602_21897_b200 as P  # noqa: E402
from conftest import check_history  # noqa: E402
from oracle import Oracle  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 10
o = Oracle()
# nx % 32 == 0 cases run the x-staged one-launch K1 (ghost runs staged after
# each warp's flag acquire); the others the gather K1
cases = [((24, 20, 16), 8), ((32, 32, 32), 4), ((40, 24, 30), 3), ((64, 64, 48), 6), ((16, 16, 8), 8),
         ((64, 24, 40), 4), ((32, 8, 32), 8), ((96, 40, 24), 3)]
fails = 0
for dims, ranks in cases:
    m = o.stencil(*dims)
    G = P.EmulatedRankGroup(*dims, ranks, 40, transport="peer")
    for rd in range(rounds):
        b = o.rhs_xorshift(m.n, 1 + rd)
        want_h, _, _ = o.cg(m, b, 40)
        G.set_rhs(b)
        G.iterate_concurrent(40, jitter=bool(rd % 2))
        hs = G.history(40)
        try:
            assert all(np.array_equal(h, hs[0]) for h in hs)
            check_history(hs[0], want_h)
        except AssertionError as e:
            fails += 1
            print("FAIL", dims, ranks, rd, str(e)[:200])
    G.close()
    print("done", dims, ranks, flush=True)
print("stress fails:", fails)
sys.exit(1 if fails else 0)
