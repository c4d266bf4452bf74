"""K1/K2/K3 micro-benchmark at 256^3 (CUDA events on the launch stream).
Usage: TW_HPCCG_LIB=<variant.so> python scripts/kbench.py [nx] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_21897_b200 as P  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rt = P.Runtime(0)
A = P.gen_stencil_matrix(nx, nx, nx, rt=rt)
n, nnz = A.n, A.nnz()
s = torch.cuda.ExternalStream(rt.compute_stream)
S = P.CgSolver(rt, A, reps + 5, P.CgOptions(iteration_marks=False), variant=0)
S.set_rhs(P.rhs_xorshift(rt, n, 7))
S.iterate(3)
S.wait()
S.enable_kernel_timing(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
S.iterate(reps)
e1.record(s)
torch.cuda.synchronize()
k1, k2, k3, it = S.kernel_times()
tot = e0.elapsed_time(e1) / reps
lib = os.path.basename(os.environ.get("TW_HPCCG_LIB", "default"))
print(f"{lib:28s} n={n} K1 {k1/it*1e3:8.1f} us {(12*nnz+16*n)/(k1/it/1e3)/1e9:7.0f} GB/s | "
      f"K2 {k2/it*1e3:6.1f} us {48*n/(k2/it/1e3)/1e9:6.0f} GB/s | K3 {k3/it*1e3:6.1f} us "
      f"{24*n/(k3/it/1e3)/1e9:6.0f} GB/s | iter {tot*1e3:7.1f} us "
      f"{(12*nnz+88*n)/(tot/1e3)/1e9:6.0f} GB/s {(2*nnz+10*n)/(tot/1e3)/1e9:6.0f} GFLOP/s",
      flush=True)
