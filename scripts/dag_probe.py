"""Time the persistent dispatcher (128^3 and 256^3; 4, 16 and 64 tiles) under whatever library
TW_HPCCG_LIB names -- used with the TW_DAG_PROBE_SKIP_* timing-probe builds
to split the dispatcher's iteration into its SpMV and update shares."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2602_21897_b200 as P  # noqa: E402

rt = P.Runtime(0)
s = torch.cuda.ExternalStream(rt.compute_stream)
for nx, K in ((128, 300), (256, 60)):
    A = P.gen_stencil_matrix(nx, nx, nx, rt=rt)
    b = P.rhs_xorshift(rt, A.n, 7)
    for T in (4, 16, 64):
        S = P.CgSolver(rt, A, 2 * K + 10, P.CgOptions(tiles=T, persistent=True,
                                                      iteration_marks=False))
        for rep in range(2):
            S.set_rhs(b)
            S.iterate(5)
            S.wait()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            S.iterate(K)
            e1.record(s)
            torch.cuda.synchronize()
        print(f"{os.path.basename(os.environ.get('TW_HPCCG_LIB', 'default'))} {nx}^3 T={T} "
              f"{e0.elapsed_time(e1) / K * 1e3:.1f} us/iter", flush=True)
        S.close()
    del A
