"""x-update placement A/B (tuning tool): the headline monolithic path
(chunked CUDA graphs, no events inside) with CgOptions.x_update = k3 (x in
every K3), k3_pairs (x once per pair of iterations) and k2, alternating over
rounds on one box; then the event-timed K1 / K2 / K3 of a separate pass (K3
averaged over the launches).  One line per grid, placement and round."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_21897_b200 as P  # noqa: E402

rt = P.Runtime(0)
stream = torch.cuda.ExternalStream(rt.compute_stream)
PLACES = tuple(os.environ.get("PLACES", "k3,k3_pairs,k2").split(","))
lib = os.path.basename(os.environ.get("TW_HPCCG_LIB", "default"))
GRIDS = {256: 200, 128: 800, 96: 1000, 64: 1500, 32: 3000}
for nx in map(int, os.environ.get("GRIDS", "256,128").split(",")):
    K = GRIDS[nx]
    A = P.gen_stencil_matrix(nx, nx, nx, rt=rt)
    b = P.rhs_xorshift(rt, A.n, 7)
    S = {xu: P.CgSolver(rt, A, K + 10, P.CgOptions(tiles=1, use_graph=True, iteration_marks=False,
                                                   x_update=xu), variant=0) for xu in PLACES}
    for rnd in range(3):
        for xu in PLACES:
            s = S[xu]
            s.set_rhs(b)
            s.iterate(10)
            s.wait()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            s.iterate(K)
            e1.record(stream)
            torch.cuda.synchronize()
            print(f"{lib} {nx}^3 round {rnd} {xu:9s} iter {1e3 * e0.elapsed_time(e1) / K:.1f} us",
                  flush=True)
    for xu in PLACES:
        S[xu].close()
        T = P.CgSolver(rt, A, K + 10, P.CgOptions(tiles=1, use_graph=False, iteration_marks=False,
                                                  x_update=xu), variant=0)
        T.set_rhs(b)
        T.iterate(10)
        T.wait()
        T.enable_kernel_timing(True)
        T.iterate(K)
        T.wait()
        k1, k2, k3, nt = T.kernel_times()
        T.close()
        print(f"{lib} {nx}^3 {xu:9s} K1 {1e3 * k1 / nt:.1f} K2 {1e3 * k2 / nt:.1f} "
              f"K3 {1e3 * k3 / nt:.1f} us", flush=True)
    del A
