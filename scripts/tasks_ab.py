"""C2 / C5 executor timings for A/Bs (tuning tool): 128^3 monolithic vs the
block-task DAG on streams, one-iteration graphs (marks on), chunked graphs
(marks off) and the persistent dispatcher; 256^3 with 8-64 tiles.  Works
with the round-1 tree as well (only CgSolver / CgOptions basics)."""
import os
import sys

import torch

HERE = os.environ.get("TW_TREE") or os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)
import paper_2602_21897_b200 as P  # noqa: E402

tag = os.environ.get("TW_TAG", "new")
rt = P.Runtime(0)
stream = torch.cuda.ExternalStream(rt.compute_stream)


def rate(A, b, K, variant, **kw):
    S = P.CgSolver(rt, A, K + 5, P.CgOptions(**kw), variant=variant)
    best = 1e9
    for _ in range(2):
        S.set_rhs(b)
        S.iterate(5)
        S.wait()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        S.iterate(K)
        e1.record(stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / K)
    S.close()
    return best


for nx, K, rows in ((128, 400, [("mono graph", 0, dict(tiles=1, use_graph=True, iteration_marks=False)),
                                ("mono graph1", 0, dict(tiles=1, use_graph=True, iteration_marks=True)),
                                ("T4 streams", 1, dict(tiles=4, iteration_marks=False)),
                                ("T4 graph1", 1, dict(tiles=4, use_graph=True, iteration_marks=True)),
                                ("T4 graphK", 1, dict(tiles=4, use_graph=True, iteration_marks=False)),
                                ("T16 persistent", 1, dict(tiles=16, persistent=True, iteration_marks=False)),
                                ("T16 streams", 1, dict(tiles=16, iteration_marks=False)),
                                ("T16 graph1", 1, dict(tiles=16, use_graph=True, iteration_marks=True)),
                                ("T16 graphK", 1, dict(tiles=16, use_graph=True, iteration_marks=False)),
                                ("T64 graph1", 1, dict(tiles=64, use_graph=True, iteration_marks=True)),
                                ("T64 graphK", 1, dict(tiles=64, use_graph=True, iteration_marks=False))]),
                    (256, 60, [("mono graph", 0, dict(tiles=1, use_graph=True, iteration_marks=False)),
                               ("T4 streams", 1, dict(tiles=4, iteration_marks=False)),
                               ("T8 persistent", 1, dict(tiles=8, persistent=True, iteration_marks=False)),
                               ("T64 persistent", 1, dict(tiles=64, persistent=True, iteration_marks=False))])):
    A = P.gen_stencil_matrix(nx, nx, nx, rt=rt)
    b = P.rhs_xorshift(rt, A.n, 7)
    out = []
    for name, v, kw in rows:
        out.append(f"{name} {1e3 * rate(A, b, K, v, **kw):.1f}")
    print(f"{tag} {nx}^3: " + " | ".join(out), flush=True)
    del A
