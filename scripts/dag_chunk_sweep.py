"""Persistent-dispatcher chunk sizes (CgOptions.dag_spmv_slices /
dag_vec_rows) at 128^3 (4/16/64 tiles) and 256^3 (16/64 tiles): us per iteration, best of two
passes.  0 = the library's choice.  `big256`: larger SpMV / update chunks at
256^3 (8 / 16 / 64 tiles)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_21897_b200 as P  # noqa: E402

rt = P.Runtime(0)
s = torch.cuda.ExternalStream(rt.compute_stream)
CASES = ((128, 300, (4, 16, 64), (0, 54, 72, 90, 108), (0, 8192)),
         (256, 60, (16, 64), (0, 180, 216), (0,)))
if sys.argv[1:] == ["big256"]:  # SpMV chunks above 12 slices per warp at 256^3
    CASES = ((256, 60, (8, 16, 64), (0, 288, 432, 648, 864), (0, 65536)),)
if sys.argv[1:] == ["small256"]:  # ... and below
    CASES = ((256, 60, (8, 16, 64), (0, 72, 108, 144, 180), (0, 16384)),)
for nx, K, tiles, slices, vecs in CASES:
    A = P.gen_stencil_matrix(nx, nx, nx, rt=rt)
    b = P.rhs_xorshift(rt, A.n, 7)
    for T in tiles:
        for sl in slices:
            row = []
            for vr in vecs:
                S = P.CgSolver(rt, A, K + 5, P.CgOptions(tiles=T, persistent=True,
                                                         iteration_marks=False,
                                                         dag_spmv_slices=sl, dag_vec_rows=vr))
                best = 1e9
                for _ in range(2):
                    S.set_rhs(b)
                    S.iterate(5)
                    S.wait()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    S.iterate(K)
                    e1.record(s)
                    torch.cuda.synchronize()
                    best = min(best, e0.elapsed_time(e1) / K * 1e3)
                S.close()
                row.append(f"{vr}:{best:.1f}")
            print(f"{nx}^3 T={T} slices={sl} " + " ".join(row), flush=True)
    del A
