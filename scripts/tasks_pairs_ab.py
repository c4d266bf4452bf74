"""Paired x updates in the block-task DAG on streams / graphs (tuning tool):
x_update = k3 vs k3_pairs per executor at 256^3 and 128^3, alternating over
two rounds; us per iteration, best of two passes."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_21897_b200 as P  # noqa: E402

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
        e0.record(stream)
        S.iterate(K)
        e1.record(stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / K)
    S.close()
    return 1e3 * best


ROWS = (("mono graphK", 0, dict(tiles=1, use_graph=True, iteration_marks=False)),
        ("T2 streams", 1, dict(tiles=2, iteration_marks=False)),
        ("T4 streams", 1, dict(tiles=4, iteration_marks=False)),
        ("T4 graphK", 1, dict(tiles=4, use_graph=True, iteration_marks=False)),
        ("T16 graphK", 1, dict(tiles=16, use_graph=True, iteration_marks=False)),
        ("T8 persistent", 1, dict(tiles=8, persistent=True, iteration_marks=False)),
        ("T16 persistent", 1, dict(tiles=16, persistent=True, iteration_marks=False)),
        ("T64 persistent", 1, dict(tiles=64, persistent=True, iteration_marks=False)))
ROWS = tuple(r for r in ROWS if os.environ.get("ONLY", "") in r[0])
for nx, K in ((256, 60), (128, 400)):
    A = P.gen_stencil_matrix(nx, nx, nx, rt=rt)
    b = P.rhs_xorshift(rt, A.n, 7)
    for rnd in range(2):
        for name, v, kw in ROWS:
            r = [f"{xu} {rate(A, b, K, v, x_update=xu, **kw):.1f}" for xu in ("k3", "k3_pairs")]
            print(f"{nx}^3 round {rnd} {name}: " + " | ".join(r), flush=True)
    del A
