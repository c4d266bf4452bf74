"""x-update placement in the block-task DAG at 128^3 (tuning tool): x in the
x/r-update tiles (k2) or in the p-update tiles / dispatcher chunks (k3), per
executor, alternating over two rounds; us per iteration, best of two passes."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_21897_b200 as P  # noqa: E402

rt = P.Runtime(0)
stream = torch.cuda.ExternalStream(rt.compute_stream)


def rate(A, b, K, **kw):
    S = P.CgSolver(rt, A, K + 5, P.CgOptions(**kw), variant=1)
    best = 1e9
    for _ in range(2):
        S.set_rhs(b)
        S.iterate(5)
        S.wait()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        S.iterate(K)
        e1.record(stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / K)
    S.close()
    return 1e3 * best


ROWS = (("T4 streams", dict(tiles=4, iteration_marks=False)),
        ("T4 graphK", dict(tiles=4, use_graph=True, iteration_marks=False)),
        ("T16 graphK", dict(tiles=16, use_graph=True, iteration_marks=False)),
        ("T16 persistent", dict(tiles=16, persistent=True, iteration_marks=False)),
        ("T64 persistent", dict(tiles=64, persistent=True, iteration_marks=False)))
for nx, K in ((128, 400), (96, 600)):
    A = P.gen_stencil_matrix(nx, nx, nx, rt=rt)
    b = P.rhs_xorshift(rt, A.n, 7)
    for rnd in range(2):
        for name, kw in ROWS:
            r = [f"{xu} {rate(A, b, K, x_update=xu, **kw):.1f}" for xu in ("k2", "k3")]
            print(f"{nx}^3 round {rnd} {name}: " + " | ".join(r), flush=True)
    del A
