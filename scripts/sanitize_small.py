"""Small end-to-end exercise of every kernel, for compute-sanitizer runs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_21897_b200 as P  # noqa: E402

rt = P.Runtime(0)
for dims in [(20, 18, 17), (3, 1, 7), (33, 5, 2)]:
    A = P.gen_stencil_matrix(*dims, rt=rt)
    n = A.n
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    P.spmv_range(A, x, y, 0, n)
    P.spmv_dot(A, x, y, 0, n)
    P.dot_range(x, y, 3, n, rt=rt)
    P.waxpby_range(1.0, x, 0.5, y, y, 1, n, rt=rt)
    b = np.random.default_rng(0).random(n)
    for run, T, g in [(P.cg_monolithic, 1, False), (P.cg_monolithic, 1, True),
                      (P.cg_tasks, 3, False), (P.cg_tasks, 5, True)]:
        run(rt, A, b, 12, P.CgOptions(tiles=T, use_graph=g))
    P.make_tile_plan(A, 4)
Z = P.gen_stencil_matrix(6, 5, 8, rt=rt, z_begin=2, z_end=5)
rng = np.random.default_rng(1)
lens = rng.integers(0, 40, 100)
rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
ci = np.concatenate([np.sort(rng.choice(100, l, replace=False)) for l in lens]).astype(np.int64)
G = P.ell_from_csr(rp, ci, rng.standard_normal(len(ci)), rt=rt)
xg = torch.rand(100, dtype=torch.float64, device="cuda")
yg = torch.zeros(100, dtype=torch.float64, device="cuda")
P.spmv_range(G, xg, yg, 0, 100)
P.rhs_xorshift(rt, 5000, 7, 123)
P.rhs_splitmix(rt, 5000, 7, 123)
torch.cuda.synchronize()
print("sanitize workload ok")
