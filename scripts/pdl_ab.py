"""Monolithic CG per-iteration time, streams vs CUDA graph, no timing events
in the loop (scripts/gpu_pdl.sh runs it with TW_PDL=1 / 0)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2602_21897_b200 as P  # noqa: E402

rt = P.Runtime(0)
for nx, K in ((256, 200), (128, 600)):
    A = P.gen_stencil_matrix(nx, nx, nx, rt=rt)
    b = P.rhs_xorshift(rt, A.n, 7)
    s = torch.cuda.ExternalStream(rt.compute_stream)
    for graph in (False, True):
        S = P.CgSolver(rt, A, 2 * K + 10, P.CgOptions(use_graph=graph, iteration_marks=False), variant=0)
        S.set_rhs(b)
        S.iterate(K)  # warm (and graph build)
        S.set_rhs(b)
        S.iterate(5)
        S.wait()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        S.iterate(K)
        e1.record(s)
        torch.cuda.synchronize()
        print(f"pdl={os.environ.get('TW_PDL', '1')} {nx}^3 {'graph' if graph else 'streams'} "
              f"{e0.elapsed_time(e1) / K:.4f} ms/iter", flush=True)
        S.close()
