"""Short 256^3 monolithic runs per x-update placement for an ncu launch list
(scripts/gpu: ncu -k regex:update_p ... python scripts/xupd_probe.py)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_21897_b200 as P  # noqa: E402

rt = P.Runtime(0)
A = P.gen_stencil_matrix(256, 256, 256, rt=rt)
b = P.rhs_xorshift(rt, A.n, 7)
for xu in sys.argv[1:] or ("k3", "k3_pairs"):
    S = P.CgSolver(rt, A, 12, P.CgOptions(tiles=1, use_graph=False, iteration_marks=False,
                                          x_update=xu), variant=0)
    S.set_rhs(b)
    S.iterate(6)
    S.wait()
    S.close()
    print(xu, "done", flush=True)
