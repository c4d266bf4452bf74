"""The auto-dispatch rule at 256^3 (tuning tool): 4 / 8 / 16 tiles on streams,
chunked graphs and the persistent dispatcher with the library's default
options (x updates paired where it pairs them), us per iteration, best of two."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_21897_b200 as P  # noqa: E402

rt = P.Runtime(0)
stream = torch.cuda.ExternalStream(rt.compute_stream)


def rate(A, b, K, **kw):
    S = P.CgSolver(rt, A, K + 5, P.CgOptions(iteration_marks=False, **kw), variant=1)
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
    m = S.mode()
    S.close()
    return 1e3 * best, m["x_in_k3"]


A = P.gen_stencil_matrix(256, 256, 256, rt=rt)
b = P.rhs_xorshift(rt, A.n, 7)
for T in (4, 8, 16):
    out = []
    for name, kw in (("streams", {}), ("graphK", dict(use_graph=True)),
                     ("persistent", dict(persistent=True)), ("auto", dict(auto_dispatch=True))):
        us, xk = rate(A, b, 60, tiles=T, **kw)
        out.append(f"{name} {us:.1f} (x {xk})")
    print(f"256^3 T={T}: " + " | ".join(out), flush=True)
