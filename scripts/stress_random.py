"""Randomised sweep of every executor against the oracle (one GPU): random
grids (x-staged closed-form and run-table, thin and ragged), variants,
tile counts, dispatch modes, graphs, x placement and L2 policy, host CSR
matrices, and emulated rank groups over every transport.  Each solve is
compared with the oracle under the SURVEY 8(c) rule.
Usage: python scripts/stress_random.py [cases] [seed]"""
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

ncases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
o = Oracle()
rt = P.Runtime(0)
fails = solves = 0


def dims_pick():
    nx = rng.choice([1, 2, 3, 7, 13, 30, 32, 33, 48, 64, 96])
    ny = rng.choice([1, 2, 5, 9, 16, 24])
    nz = rng.choice([1, 2, 3, 6, 8, 12, 17])
    return nx, ny, nz


def check(tag, h, x, m, b, iters):
    global fails, solves
    solves += 1
    want_h, want_x, _ = o.cg(m, b, iters)
    try:
        # a tiny system converges exactly and then breaks down (0 / 0) in the
        # reference too: the breakdown must come at the same iteration, and
        # the finite prefix must match
        fin = np.isfinite(want_h)
        if not np.array_equal(np.isfinite(h), fin):
            # the reference's own tile orders (cg_tasks) may break down at
            # another iteration than cg_reference as well: a GPU breakdown
            # point one of them shares is their spread, not a failure
            for t in (2, 4, 8, 16):
                if t <= m.n:
                    ht = o.cg(m, b, iters, tiles=t)[0]
                    if np.array_equal(np.isfinite(ht), np.isfinite(h)):
                        print("SPREAD", tag, f"breakdown as the reference's {t}-tile order", flush=True)
                        return
            raise AssertionError("breakdown at another iteration")
        k = int(np.argmin(fin)) if not fin.all() else len(fin)
        if k:
            check_history(h[:k], want_h[:k])
        if fin.all():
            assert np.all(rel_gap(x, want_x) <= 1e-10), "x"
    except AssertionError as e:
        fails += 1
        print("FAIL", tag, str(e)[:160], flush=True)


for c in range(ncases):
    kind = rng.choice(["single", "single", "csr", "group", "group"])
    iters = rng.choice([5, 12, 25])
    if kind == "single":
        dims = dims_pick()
        m = o.stencil(*dims)
        b = o.rhs_xorshift(m.n, c + 1)
        A = P.gen_stencil_matrix(*dims, rt=rt)
        if rng.random() < 0.2:
            A.set_x_staged(False)
        variant = rng.choice([0, 1])
        T = 1 if variant == 0 else rng.choice([t for t in (1, 2, 3, 4, 8, 16, 64) if t <= m.n])
        persistent = variant == 1 and rng.random() < 0.5
        opt = P.CgOptions(tiles=T, use_graph=not persistent and rng.random() < 0.5,
                          iteration_marks=rng.random() < 0.5, persistent=persistent,
                          x_update=rng.choice([None, "k2", "k3", "k3_pairs"]),
                          l2_keep=rng.choice([None, True, False]))
        tag = (kind, dims, variant, T, persistent, opt.use_graph, opt.x_update, opt.l2_keep)
        try:
            S = P.CgSolver(rt, A, iters, opt, variant=variant)
        except P.ConfigError as e:
            print("skip", tag, str(e)[:80])
            continue
        S.set_rhs(b)
        k = rng.randint(0, iters)
        S.iterate(k)
        S.iterate(iters - k)
        check(tag, S.history(iters), S.solution(), m, b, iters)
        S.close()
    elif kind == "csr":
        n = rng.choice([100, 1000, 5000])
        band = rng.choice([3, 20, 40, 200])
        rows, cols = [], []
        for i in range(n):
            cc = np.unique(np.clip(i + np.array([rng.randint(-band, band) for _ in range(7)]), 0, n - 1))
            cc = np.union1d(cc, [i])
            rows.append(len(cc))
            cols.append(cc)
        rp = np.concatenate([[0], np.cumsum(rows)]).astype(np.int64)
        ci = np.concatenate(cols).astype(np.int64)
        va = np.where(ci == np.repeat(np.arange(n), rows), 2.0 * band + 10, -1.0)
        from oracle import Csr
        m = Csr(n, rp, ci, va)
        b = o.rhs_splitmix(n, c)
        A = P.ell_from_csr(rp, ci, va, rt=rt)
        res = P.cg_solve(rt, A, b, iters, P.CgOptions(tiles=1, iteration_marks=False))
        check((kind, n, band, A.x_staged), res.residual_history, res.x, m, b, iters)
    else:
        ranks = rng.choice([2, 3, 4, 8])
        nx, ny = rng.choice([13, 30, 32, 48, 64]), rng.choice([4, 9, 16])
        nz = ranks * rng.choice([1, 2, 3])
        m = o.stencil(nx, ny, nz)
        b = o.rhs_xorshift(m.n, c + 3)
        how = rng.choice(["loopback", "peer", "peer_concurrent", "tasks", "tasks_persistent"])
        rows = nx * ny * (nz // ranks)
        T = rng.choice([t for t in (1, 2, 4, 8) if t <= rows])
        if how in ("tasks", "tasks_persistent"):
            opt = P.CgOptions(tiles=T, persistent=how == "tasks_persistent", iteration_marks=False)
            G = P.EmulatedRankGroup(nx, ny, nz, ranks, iters, variant=1, options=opt,
                                    transport="peer" if how == "tasks_persistent" else "loopback")
        else:
            G = P.EmulatedRankGroup(nx, ny, nz, ranks, iters,
                                    transport="loopback" if how == "loopback" else "peer")
        G.set_rhs(b)
        k = rng.randint(1, iters - 1)
        if how == "peer_concurrent":
            G.iterate_concurrent(k, jitter=True)
            G.iterate_concurrent(iters - k)
        else:
            G.iterate(k)
            G.iterate(iters - k)
        hs = G.history(iters)
        tag = (kind, (nx, ny, nz), ranks, how, T)
        if not all(np.array_equal(h, hs[0]) for h in hs):
            fails += 1
            print("FAIL ranks disagree", tag, flush=True)
        check(tag, hs[0], G.solution(), m, b, iters)
        G.close()
print(f"stress: {solves} solves, {fails} failures")
sys.exit(1 if fails else 0)
