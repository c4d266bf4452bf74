"""Event-timed K1 / K2 / K3 of the monolithic CG (graph off, per-kernel
events on the launch stream): one line per grid, us per launch, for the x
update in K3 and in K2 (CgOptions.x_update)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_21897_b200 as P  # noqa: E402

rt = P.Runtime(0)
for nx, K in ((256, 200), (128, 600)):
    A = P.gen_stencil_matrix(nx, nx, nx, rt=rt)
    b = P.rhs_xorshift(rt, A.n, 7)
    for xu in ("k3", "k2"):
        S = P.CgSolver(rt, A, 2 * K + 10, P.CgOptions(use_graph=False, iteration_marks=False,
                                                      x_update=xu), variant=0)
        S.set_rhs(b)
        S.iterate(10)
        S.wait()
        S.enable_kernel_timing(True)
        S.iterate(K)
        S.wait()
        k1, k2, k3, nt = S.kernel_times()
        print(f"x_update={xu} {nx}^3 K1 {1e3 * k1 / nt:.1f} K2 {1e3 * k2 / nt:.1f} "
              f"K3 {1e3 * k3 / nt:.1f} K2+K3 {1e3 * (k2 + k3) / nt:.1f} us", flush=True)
        S.close()
