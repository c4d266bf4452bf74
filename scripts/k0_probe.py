"""Host wall clock of gen_stencil_matrix at 256^3 in the situations bench.py
meets it (fresh, after solves through tw_cg_solve, after freeing a matrix)."""
import gc
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_21897_b200 as P  # noqa: E402

rt = P.Runtime(0)


def gen(tag):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    A = P.gen_stencil_matrix(256, 256, 256, rt=rt)
    print(f"{tag}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    return A


A = gen("first")
B = gen("second")
del B
gc.collect()
C = gen("after del")
b = np.ones(A.n)
P.cg_solve(rt, A, b, 10, P.CgOptions(tiles=1), 0)
D = gen("after cg_solve")
del C, D
gc.collect()
E = gen("after del x2")
S = P.CgSolver(rt, A, 10, P.CgOptions(tiles=1), variant=0)
F = gen("with a solver open")
S.close()
G = gen("after solver close")
