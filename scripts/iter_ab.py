"""Monolithic CG A/B timing (tuning tool): per grid, the event-timed
iteration of the headline path (one-iteration CUDA graph replayed, no events
inside) and the event-timed K1 / K2 / K3 of a separate pass (per-kernel events
on the launch stream).  The library is the default build or TW_HPCCG_LIB
(a variant from scripts/build_variants.sh); one line per grid."""
import hashlib
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_21897_b200 as P  # noqa: E402

lib = os.path.basename(os.environ.get("TW_HPCCG_LIB", "default"))
rt = P.Runtime(0)
stream = torch.cuda.ExternalStream(rt.compute_stream)
for nx, K in ((256, 200), (128, 800)):
    A = P.gen_stencil_matrix(nx, nx, nx, rt=rt)
    b = P.rhs_xorshift(rt, A.n, 7)
    S = P.CgSolver(rt, A, K + 10, P.CgOptions(tiles=1, use_graph=True, iteration_marks=False),
                   variant=0)
    best = 1e9
    for _ in range(3):
        S.set_rhs(b)
        S.iterate(10)
        S.wait()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        S.iterate(K)
        e1.record(stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / K)
    # result fingerprint: variants that change no bit print the same digest
    S.set_rhs(b)
    S.iterate(50)
    hd = hashlib.sha256(S.history(50).tobytes()).hexdigest()[:12]
    S.close()
    T = P.CgSolver(rt, A, K + 10, P.CgOptions(tiles=1, use_graph=False, iteration_marks=False),
                   variant=0)
    T.set_rhs(b)
    T.iterate(10)
    T.wait()
    T.enable_kernel_timing(True)
    T.iterate(K)
    T.wait()
    k1, k2, k3, nt = T.kernel_times()
    T.close()
    print(f"{lib} {nx}^3 iter {1e3 * best:.1f} us | K1 {1e3 * k1 / nt:.1f} K2 {1e3 * k2 / nt:.1f} "
          f"K3 {1e3 * k3 / nt:.1f} us | history {hd}", flush=True)
    del A
