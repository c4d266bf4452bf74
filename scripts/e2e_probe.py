import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2602_21897_b200 as P
from paper_2602_21897_b200 import _native as N
rt = P.Runtime(0)
A = P.gen_stencil_matrix(256, 256, 256, rt=rt)
rp, ci, va = A.to_csr()
Ac = P.ell_from_csr(rp, ci, va, rt=rt)
del rp, ci, va
b = np.random.default_rng(0).random(A.n)
bp = torch.from_numpy(b.copy()).pin_memory().numpy()
xp = torch.empty(A.n, dtype=torch.float64).pin_memory().numpy()
opt = P.CgOptions(tiles=1, iteration_marks=False)
for K in (1, 100):
    for name, bb, xx in (("pageable", b, None), ("pinned", bp, xp)):
        ts = []
        for _ in range(4):
            t0 = time.perf_counter(); P.cg_solve(rt, Ac, bb, K, opt, 0, x_out=xx); ts.append(time.perf_counter() - t0)
        print(f"K={K} {name}: {1e3*min(ts):.2f} ms", flush=True)
