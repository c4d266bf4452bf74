"""Randomised sweep of the standalone operators and builders against the
oracle (one GPU): K0 on random grids and z-slabs (structure bit-exact in
both column forms), CSR round trips of random matrices (empty rows, ragged
widths), SpMV / waxpby bit-exact and dots within 1e-12 over random row
ranges (aliasing included), the fused K2 / K3 operators, tile plans.
Usage: python scripts/stress_ops.py [cases] [seed]"""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_21897_b200 as P  # noqa: E402
from oracle import Csr, Oracle  # noqa: E402

ncases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
o = Oracle()
rt = P.Runtime(0)
fails = checks = 0


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()


def expect(cond, tag):
    global fails, checks
    checks += 1
    if not cond:
        fails += 1
        print("FAIL", tag, flush=True)


for c in range(ncases):
    kind = rng.choice(["k0", "k0", "csr", "ops", "tiles"])
    if kind in ("k0", "tiles", "ops"):
        nx, ny, nz = rng.choice([1, 2, 5, 31, 32, 33, 64]), rng.choice([1, 3, 8, 17]), rng.choice([1, 2, 4, 9])
        m = o.stencil(nx, ny, nz)
    if kind == "k0":
        zb = rng.randint(0, nz - 1)
        ze = rng.randint(zb + 1, nz)
        A = P.gen_stencil_matrix(nx, ny, nz, rt=rt, z_begin=zb, z_end=ze)
        r0g = A.info.row_offset
        n = A.n
        want = o.stencil_rows(nx, ny, nz, r0g, r0g + n)
        for staged in ((False, True) if A.x_staged else (False,)):
            a0 = 32 * rng.randint(0, max(0, (n - 1) // 32))
            a1 = rng.randint(a0, n)
            rp, ci, va = A.to_csr_rows(a0, a1, staged=staged)
            k0, k1 = want.row_ptr[a0], want.row_ptr[a1]
            expect(np.array_equal(rp, want.row_ptr[a0:a1 + 1] - k0) and
                   np.array_equal(ci, want.col_idx[k0:k1]) and np.array_equal(va, want.values[k0:k1]),
                   ("k0", (nx, ny, nz, zb, ze), staged, a0, a1))
    elif kind == "csr":
        n = rng.choice([1, 5, 40, 300, 2000])
        lens = [rng.choice([0, 0, 1, 3, 9, 27, 40]) for _ in range(n)]
        cols = [np.unique(np.array([rng.randrange(n) for _ in range(L)], np.int64)) for L in lens]
        rp = np.concatenate([[0], np.cumsum([len(x) for x in cols])]).astype(np.int64)
        ci = np.concatenate(cols).astype(np.int64) if rp[-1] else np.zeros(0, np.int64)
        va = np.array([rng.uniform(-2, 2) for _ in range(len(ci))])
        A = P.ell_from_csr(rp, ci, va, rt=rt)
        r2, c2, v2 = A.to_csr()
        expect(np.array_equal(r2, rp) and np.array_equal(c2, ci) and np.array_equal(v2, va), ("csr", n))
        x = np.array([rng.uniform(-1, 1) for _ in range(n)])
        y = torch.full((n,), -7.0, dtype=torch.float64, device="cuda")
        a0 = rng.randint(0, n)
        a1 = rng.randint(a0, n)
        P.spmv_range(A, dev(x), y, a0, a1)
        want = o.spmv(Csr(n, rp, ci, va), x, a0, a1, np.full(n, -7.0))
        expect(np.array_equal(y.cpu().numpy(), want), ("csr spmv", n, a0, a1))
    elif kind == "ops":
        A = P.gen_stencil_matrix(nx, ny, nz, rt=rt)
        n = A.n
        x = o.rhs_splitmix(n, c)
        a0 = rng.randint(0, n)
        a1 = rng.randint(a0, n)
        y = torch.zeros(n, dtype=torch.float64, device="cuda")
        d = P.spmv_dot(A, dev(x), y, a0, a1)
        want = o.spmv(m, x, a0, a1, np.zeros(n))
        expect(np.array_equal(y.cpu().numpy(), want), ("spmv_dot", (nx, ny, nz), a0, a1))
        wd = o.dot(x, want, a0, a1)
        expect(abs(d - wd) <= 1e-12 * max(1e-300, float(np.abs(x[a0:a1] * want[a0:a1]).sum())),
               ("spmv_dot dot", (nx, ny, nz), a0, a1))
        al, be = rng.uniform(-2, 2), rng.uniform(-2, 2)
        xs, ys = dev(x), dev(want)
        alias = rng.choice(["none", "x", "y"])
        w = xs if alias == "x" else ys if alias == "y" else torch.zeros(n, dtype=torch.float64, device="cuda")
        P.waxpby_range(al, xs, be, ys, w, a0, a1, rt=rt)
        wref = o.waxpby(al, x, be, want, None if alias == "none" else (x.copy() if alias == "x" else want.copy()), a0, a1)
        got = w.cpu().numpy()
        expect(np.array_equal(got[a0:a1], wref[a0:a1]), ("waxpby", alias, a0, a1))
        # fused K2 / K3
        xx, pp, rr, aa = (o.rhs_splitmix(n, c + k) for k in (11, 12, 13, 14))
        X, Pp, R, Ap = dev(xx), dev(pp), dev(rr), dev(aa)
        g = P.update_xr_rr(al, X, Pp, R, Ap, a0, a1, rt=rt)
        xw = o.waxpby(1.0, xx, al, pp, xx.copy(), a0, a1)
        rw = o.waxpby(1.0, rr, -al, aa, rr.copy(), a0, a1)
        expect(np.array_equal(X.cpu().numpy(), xw) and np.array_equal(R.cpu().numpy(), rw),
               ("update_xr", a0, a1))
        expect(abs(g - o.dot(rw, rw, a0, a1)) <= 1e-12 * max(1e-300, o.dot(rw, rw, a0, a1)), ("update_xr rr", a0, a1))
        P.update_p(be, R, Pp, a0, a1, rt=rt)
        pw = o.waxpby(1.0, rw, be, pp, pp.copy(), a0, a1)
        expect(np.array_equal(Pp.cpu().numpy(), pw), ("update_p", a0, a1))
    else:  # tiles
        A = P.gen_stencil_matrix(nx, ny, nz, rt=rt)
        T = rng.randint(1, min(A.n, 70))
        got = P.make_tile_plan(A, T)
        want = o.tile_plan(m, T)
        expect(all(g.r0 == want[0][i] and g.r1 == want[1][i] and g.band_lo == want[2][i] and
                   g.band_hi == want[3][i] for i, g in enumerate(got)), ("tiles", (nx, ny, nz), T))
    rt.synchronize()
print(f"stress ops: {checks} checks, {fails} failures")
sys.exit(1 if fails else 0)
