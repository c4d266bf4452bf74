"""Generate tests/golden/hpccg_golden_256.npz from the REFERENCE itself at the
headline size (BASELINE configs[2]: 256^3 per GPU, b = xorshift64 seed 7).

Run in the build container (where /root/reference exists; needs ~16 GB RAM
and about two minutes):
    make -C oracle && python tests/golden/make_golden_256.py

Contents (small enough to commit; the full CSR is 7.3 GB):
  * csr_256_plane_digests: uint8[256, 3, 32] -- SHA-256 of each z-plane's
    slice of the reference's gen_stencil_matrix (csr.cpp:29-59) output:
    row_ptr (relative to the plane's first row, int64), col_idx (int64) and
    values (f64), in that order.  The GPU test exports the device matrix a
    plane range at a time and compares digests (bit-exact structure).
  * csr_256_nnz: the reference's nnz.
  * cg_256_xorshift7_history: cg_reference (cg.cpp:372-395) residual history,
    60 iterations.
  * cg_256_xorshift7_x_idx / _x_val: the final x at every 4093rd row plus the
    first and last rows (the 134 MB vector itself is not committed).
  * cg_256_xorshift7_x_fsum: math.fsum of the final x (exactly rounded).
"""
import hashlib
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import Oracle, Reference  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "hpccg_golden_256.npz")
D = 256
ITERS = 60


def plane_digests(rp, ci, va, nx, ny, nz):
    plane = nx * ny
    dg = np.zeros((nz, 3, 32), np.uint8)
    for z in range(nz):
        r0, r1 = z * plane, (z + 1) * plane
        k0, k1 = int(rp[r0]), int(rp[r1])
        for j, arr in enumerate((rp[r0:r1 + 1] - rp[r0], ci[k0:k1], va[k0:k1])):
            dg[z, j] = np.frombuffer(hashlib.sha256(np.ascontiguousarray(arr).tobytes()).digest(),
                                     np.uint8)
    return dg


def x_sample_idx(n):
    return np.unique(np.concatenate([np.arange(0, n, 4093), [n - 1]])).astype(np.int64)


def main():
    R = Reference()
    o = Oracle()
    t = time.time()
    M = R.stencil(D, D, D)
    print(f"reference gen_stencil_matrix {D}^3: {time.time() - t:.1f} s", flush=True)
    out = {}
    m = M.export()
    out["csr_256_nnz"] = np.array([m.nnz], np.int64)
    out["csr_256_plane_digests"] = plane_digests(m.row_ptr, m.col_idx, m.values, D, D, D)
    del m
    b = o.rhs_xorshift(D ** 3, 7)
    t = time.time()
    h, x, _ = R.cg_reference(M, b, ITERS)
    print(f"reference cg_reference x{ITERS}: {time.time() - t:.1f} s", flush=True)
    idx = x_sample_idx(D ** 3)
    out["cg_256_xorshift7_history"] = h
    out["cg_256_xorshift7_x_idx"] = idx
    out["cg_256_xorshift7_x_val"] = x[idx]
    out["cg_256_xorshift7_x_fsum"] = np.array([math.fsum(x)])
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, "res[0] =", repr(h[0]))


if __name__ == "__main__":
    main()
