"""The tasks variant's programmatic chain (CgOptions.chain, TW_DISPATCH_CHAIN)
against the other executors (tuning tool): us per iteration, best of two
passes, two rounds alternating.  128^3: 2 / 4 / 8 / 16 tiles; 256^3 (C5's
per-GPU share): 2 / 4 / 8 / 16 / 32 / 64 tiles; `small`: 64^3 and 96^3 at
2 / 4 / 8 tiles."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_21897_b200 as P  # noqa: E402

rt = P.Runtime(0)
stream = torch.cuda.ExternalStream(rt.compute_stream)


def rate(A, b, K, variant, **kw):
    S = P.CgSolver(rt, A, K + 5, P.CgOptions(iteration_marks=False, **kw), variant=variant)
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
    return 1e3 * best


CASES = ((128, 400, (2, 4, 8, 16)), (256, 60, (2, 4, 8, 16, 32, 64)))
if sys.argv[1:] == ["small"]:  # the lower end of the chain's range
    CASES = ((64, 1500, (2, 4, 8)), (96, 800, (2, 4, 8)))
tag = os.path.basename(os.environ.get("TW_HPCCG_LIB", "default"))
for nx, K, tiles in CASES:
    A = P.gen_stencil_matrix(nx, nx, nx, rt=rt)
    b = P.rhs_xorshift(rt, A.n, 7)
    for rnd in range(2):
        out = [f"mono {rate(A, b, K, 0, tiles=1, use_graph=True):.1f}"]
        for T in tiles:
            if os.environ.get("CHAIN_ONLY"):  # library A/Bs of the chain itself
                out.append(f"T{T}: chain {rate(A, b, K, 1, tiles=T, chain=True):.1f}")
                continue
            row = [f"chain {rate(A, b, K, 1, tiles=T, chain=True):.1f}",
                   f"chainK {rate(A, b, K, 1, tiles=T, chain=True, use_graph=True):.1f}",
                   f"graphK {rate(A, b, K, 1, tiles=T, use_graph=True):.1f}" if T <= 16 else "",
                   f"streams {rate(A, b, K, 1, tiles=T):.1f}" if T <= 8 else "",
                   f"persistent {rate(A, b, K, 1, tiles=T, persistent=True):.1f}" if T >= 4 else ""]
            out.append(f"T{T}: " + " ".join(x for x in row if x))
        print(f"{tag} {nx}^3 round {rnd}: " + " | ".join(out), flush=True)
    del A
