"""CPU tests: the oracle restatement (oracle/hpccg_oracle.c) against the
reference's own outputs -- the committed golden vectors (tests/golden, made by
running the reference build) and, where oracle/_ref is built, the reference
library itself.  Mirrors proj/tests/test_bench.cpp's hot-path cases."""
import numpy as np
import pytest

from conftest import check_history, rel_gap

# SURVEY.md 8(c) probe table (reference code, g++ -O2): residual history of
# cg_reference on 32^3 with b = xorshift seed 7 / SplitMix seed 7.
SURVEY_XORSHIFT = {0: 312.10258754890583, 9: 8.4228643982508551, 49: 4.9743586177269403e-08,
                   149: 6.671486394281344e-30}
SURVEY_SPLITMIX = {0: 134.226481108976, 9: 4.6225678414464992, 49: 3.9219341048792209e-08,
                   149: 5.2143498151126253e-30}


@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 2, 2), (4, 3, 5), (5, 5, 5), (6, 5, 4)])
def test_stencil_structure_matches_golden(orc, golden, dims):
    m = orc.stencil(*dims)
    key = "csr_%dx%dx%d" % dims
    assert np.array_equal(m.row_ptr, golden[key + "_row_ptr"])
    assert np.array_equal(m.col_idx, golden[key + "_col_idx"])
    assert np.array_equal(m.values, golden[key + "_values"])
    assert orc.validate(m)
    assert m.nnz == orc.stencil_nnz(*dims)


def test_single_cell_and_2x2x2(orc):
    m = orc.stencil(1, 1, 1)  # test_bench.cpp:54-61
    assert m.n == 1 and m.nnz == 1 and m.col_idx[0] == 0 and m.values[0] == 27.0
    m = orc.stencil(2, 2, 2)  # test_bench.cpp:63-75
    assert m.n == 8 and m.nnz == 64
    for i in range(8):
        assert m.row_ptr[i + 1] - m.row_ptr[i] == 8
        assert m.values[m.row_ptr[i]:m.row_ptr[i + 1]].sum() == 20.0


def test_row_sums_interior_one(orc):
    d = 5  # test_bench.cpp:97-115
    m = orc.stencil(d, d, d)
    sums = np.add.reduceat(m.values, m.row_ptr[:-1])
    idx = np.arange(m.n)
    x, y, z = idx % d, (idx // d) % d, idx // (d * d)
    interior = (x > 0) & (x < d - 1) & (y > 0) & (y < d - 1) & (z > 0) & (z < d - 1)
    assert np.all(sums[interior] == 1.0) and np.all(sums[~interior] > 1.0)


def test_bad_dims_rejected(orc):
    from oracle import OracleError
    with pytest.raises(OracleError):
        orc.stencil(0, 1, 1)  # test_bench.cpp:144


@pytest.mark.parametrize("nnz_dims", [(32, 32, 32, 830584), (128, 128, 128, 55742968),
                                      (256, 256, 256, 449455096), (512, 512, 512, 3609741304)])
def test_nnz_closed_form(orc, nnz_dims):
    nx, ny, nz, want = nnz_dims  # SURVEY.md 8 header
    assert orc.stencil_nnz(nx, ny, nz) == want


def test_spmv_matches_golden_bitwise(orc, golden):
    m = orc.stencil(6, 5, 4)
    x = golden["spmv_6x5x4_x"]
    assert np.array_equal(x, orc.rhs_xorshift(m.n, 3))
    y = orc.spmv(m, x)
    assert np.array_equal(y, golden["spmv_6x5x4_y"])
    # tiled spmv reproduces the full call bit for bit (test_bench.cpp:177-186)
    r0, r1, _, _ = orc.tile_plan(m, 7)
    yt = np.zeros(m.n)
    for a, b in zip(r0, r1):
        orc.spmv(m, x, int(a), int(b), y=yt)
    assert np.array_equal(yt, y)
    # matrix-free restatement is bit-identical
    assert np.array_equal(orc.stencil_spmv(6, 5, 4, x), y)


def test_spmv_identity_and_hand_matrix(orc):
    from oracle import Csr
    ident = Csr(5, np.arange(6, dtype=np.int64), np.arange(5, dtype=np.int64), np.ones(5))
    x = orc.rhs_xorshift(5, 11)
    assert np.array_equal(orc.spmv(ident, x), x)  # test_bench.cpp:147-158
    m = Csr(3, np.array([0, 2, 3, 6], np.int64), np.array([0, 2, 1, 0, 1, 2], np.int64),
            np.array([2, 1, 3, 4, 5, 6], np.float64))
    y = orc.spmv(m, np.array([1.0, -2.0, 3.0]))
    assert np.array_equal(y, np.array([5.0, -6.0, 12.0]))  # test_bench.cpp:160-175


def test_dot_and_waxpby_identities(orc):
    n = 1000  # test_bench.cpp:188-222
    ones = np.ones(n)
    assert orc.dot(ones, ones) == float(n)
    a, b = orc.rhs_xorshift(n, 5), orc.rhs_xorshift(n, 9)
    plain = 0.0
    for i in range(n):
        plain += a[i] * b[i]
    assert orc.dot(a, b) == plain
    parts = sum(orc.dot(a, b, n * t // 8, n * (t + 1) // 8) for t in range(8))
    assert rel_gap(parts, plain) < 1e-12
    n = 257
    x, y = orc.rhs_xorshift(n, 21), orc.rhs_xorshift(n, 22)
    assert np.array_equal(orc.waxpby(1.0, x, 0.0, y), x)
    assert np.array_equal(orc.waxpby(0.0, x, 1.0, y), y)
    assert np.array_equal(orc.waxpby(2.0, x, 3.0, y), 2.0 * x + 3.0 * y)


@pytest.mark.parametrize("T", [1, 3, 7])
def test_tile_plan_matches_golden(orc, golden, T):
    m = orc.stencil(5, 4, 3)
    got = np.stack(orc.tile_plan(m, T))
    assert np.array_equal(got, golden["tiles_5x4x3_T%d" % T])


def test_tile_plan_rejects(orc):
    from oracle import OracleError
    m = orc.stencil(5, 4, 3)
    with pytest.raises(OracleError):
        orc.tile_plan(m, 0)
    with pytest.raises(OracleError):
        orc.tile_plan(m, m.n + 1)


@pytest.mark.parametrize("name,dims,gen,seed,iters", [
    ("cg_32_xorshift7", (32, 32, 32), "xorshift", 7, 150),
    ("cg_32_splitmix7", (32, 32, 32), "splitmix", 7, 150),
    ("cg_8_xorshift7", (8, 8, 8), "xorshift", 7, 10),
    ("cg_6_xorshift17", (6, 6, 6), "xorshift", 17, 8),
])
def test_cg_reference_bitwise_vs_golden(orc, golden, name, dims, gen, seed, iters):
    m = orc.stencil(*dims)
    b = orc.rhs_xorshift(m.n, seed) if gen == "xorshift" else orc.rhs_splitmix(m.n, seed)
    if name + "_b" in golden:
        assert np.array_equal(b, golden[name + "_b"])
    h, x, _ = orc.cg(m, b, iters)
    assert np.array_equal(h, golden[name + "_history"])
    assert np.array_equal(x, golden[name + "_x"])


def test_cg_survey_probe_values(orc):
    m = orc.stencil(32, 32, 32)
    for gen, want in (("xorshift", SURVEY_XORSHIFT), ("splitmix", SURVEY_SPLITMIX)):
        b = orc.rhs_xorshift(m.n, 7) if gen == "xorshift" else orc.rhs_splitmix(m.n, 7)
        h, _, _ = orc.cg(m, b, 150)
        for k, v in want.items():
            assert h[k] == v, (gen, k)


@pytest.mark.parametrize("T", [4, 16, 64])
def test_cg_tasks_tile_order_bitwise(orc, golden, T):
    m = orc.stencil(32, 32, 32)
    b = orc.rhs_xorshift(m.n, 7)
    h, x, _ = orc.cg(m, b, 50, tiles=T)
    assert np.array_equal(h, golden["cgtasks_32_T%d_history" % T])
    if "cgtasks_32_T%d_x" % T in golden:
        assert np.array_equal(x, golden["cgtasks_32_T%d_x" % T])
    # and the reference's own tasks variant is within the stated rule of cg_reference
    check_history(h, golden["cg_32_xorshift7_history"][:50])


def test_cg_identity_one_iteration(orc, golden):
    from oracle import Csr
    ident = Csr(6, np.arange(7, dtype=np.int64), np.arange(6, dtype=np.int64), np.ones(6))
    b = golden["cg_identity_b"]
    h, x, conv = orc.cg(ident, b, 1, tol=1e-12)
    assert conv and h[0] == golden["cg_identity_history"][0]
    assert np.array_equal(x, golden["cg_identity_x"])


def test_residual_monotone(orc):
    m = orc.stencil(8, 8, 8)  # test_bench.cpp:297-305
    h, _, _ = orc.cg(m, orc.rhs_xorshift(m.n, 13), 25)
    assert np.all(h[1:] <= h[:-1] * (1 + 1e-12))


def test_matrix_free_cg_bitwise(orc, golden):
    b = orc.rhs_xorshift(32 ** 3, 7)
    h, x = orc.cg_stencil(32, 32, 32, b, 150)
    assert np.array_equal(h, golden["cg_32_xorshift7_history"])
    assert np.array_equal(x, golden["cg_32_xorshift7_x"])


# ---- against the live reference build (oracle/_ref), when present ----------

@pytest.mark.parametrize("dims", [(3, 4, 5), (7, 1, 3), (16, 16, 16)])
def test_oracle_vs_reference_library(orc, ref, dims):
    m = orc.stencil(*dims)
    M = ref.stencil(*dims)
    rm = M.export()
    assert np.array_equal(m.row_ptr, rm.row_ptr) and np.array_equal(m.col_idx, rm.col_idx)
    assert np.array_equal(m.values, rm.values)
    x = orc.rhs_splitmix(m.n, 3)
    assert np.array_equal(orc.spmv(m, x), ref.spmv(M, x))
    h, xs, _ = orc.cg(m, x, 20)
    hr, xr, _ = ref.cg_reference(M, x, 20)
    assert np.array_equal(h, hr) and np.array_equal(xs, xr)


def test_reference_task_path_runs_on_threads(orc, ref):
    M = ref.stencil(16, 16, 16)
    b = orc.rhs_xorshift(M.n, 7)
    h, x, secs = ref.cg_tasks(M, b, 10, tiles=8, workers=4, real_threads=True)
    ho, xo, _ = orc.cg(orc.stencil(16, 16, 16), b, 10, tiles=8)
    assert np.array_equal(h, ho) and np.array_equal(x, xo) and secs > 0


# ---- the headline size (256^3, BASELINE configs[2]) against the reference --

def test_matrix_free_cg_threaded_bitwise(orc, golden):
    """orc_cg_stencil_mt splits only row-independent work over threads: the
    32^3 x 150 reference history and x to the bit for any thread / tile count."""
    b = orc.rhs_xorshift(32 ** 3, 7)
    for threads in (1, 3, 8):
        h, x = orc.cg_stencil_mt(32, 32, 32, b, 150, threads=threads)
        assert np.array_equal(h, golden["cg_32_xorshift7_history"])
        assert np.array_equal(x, golden["cg_32_xorshift7_x"])
    h4, x4 = orc.cg_stencil(32, 32, 32, b, 50, tiles=4)
    h4t, x4t = orc.cg_stencil_mt(32, 32, 32, b, 50, tiles=4, threads=5)
    assert np.array_equal(h4, h4t) and np.array_equal(x4, x4t)


@pytest.mark.parametrize("dims,ranges", [((5, 4, 3), [(0, 60), (7, 33), (20, 20)]),
                                         ((17, 9, 13), [(0, 153), (153, 1989), (1000, 1001)])])
def test_stencil_rows_is_the_full_matrix_sliced(orc, dims, ranges):
    m = orc.stencil(*dims)
    for r0, r1 in ranges:
        c = orc.stencil_rows(*dims, r0, r1)
        k0, k1 = m.row_ptr[r0], m.row_ptr[r1]
        assert np.array_equal(c.row_ptr, m.row_ptr[r0:r1 + 1] - k0)
        assert np.array_equal(c.col_idx, m.col_idx[k0:k1])
        assert np.array_equal(c.values, m.values[k0:k1])


def test_oracle_256_structure_vs_reference_digests(orc, golden256):
    """The oracle's gen_stencil_matrix restatement at 256^3 against the
    reference's own matrix: per-plane SHA-256 of row_ptr / col_idx / values
    for the boundary and a few interior planes (all 256 are compared with
    the device matrix in tests/test_gpu_headline.py)."""
    from conftest import csr_digests
    D = 256
    plane = D * D
    assert orc.stencil_nnz(D, D, D) == int(golden256["csr_256_nnz"][0])
    for z in (0, 1, 128, 254, 255):
        c = orc.stencil_rows(D, D, D, z * plane, (z + 1) * plane)
        assert np.array_equal(csr_digests(c.row_ptr, c.col_idx, c.values),
                              golden256["csr_256_plane_digests"][z]), z


def test_oracle_256_cg_vs_reference(orc, golden256):
    """The threaded matrix-free oracle at the headline size reproduces the
    reference's cg_reference (cg.cpp:372-395) history bit for bit (first 12
    of the 60 committed iterations; the GPU test checks all 60)."""
    D = 256
    b = orc.rhs_xorshift(D ** 3, 7)
    h, _ = orc.cg_stencil_mt(D, D, D, b, 12)
    assert np.array_equal(h, golden256["cg_256_xorshift7_history"][:12])
    assert h[0] == 9518.4498236045511  # SURVEY.md 8(c) probe value
