"""K0 (gen_stencil_matrix on the device) at 256^3, twice: run under
`ncu --metrics gpu__time_duration.sum -k regex:stencil` for the fill kernel's
per-launch time (profiles/r02_final/k0_launches.csv)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2602_21897_b200 import hpccg as P

rt = P.Runtime(0)
for i in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    A = P.gen_stencil_matrix(256, 256, 256, rt=rt)
    torch.cuda.synchronize()
    print(f"gen_stencil_matrix 256^3 pass {i}: {1e3 * (time.perf_counter() - t):.2f} ms (host wall)")
    del A
