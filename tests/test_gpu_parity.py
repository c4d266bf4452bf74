"""GPU parity tests: the CUDA path (libtw_hpccg.so through the C ABI) against
the oracle and the reference's golden vectors.

Bar: matrix structure and values bit-exact; SpMV and waxpby
bit-exact; dots within reassociation error; CG residual histories within
1e-10 relative inside the window res_k >= 1e-15 res_0 (|d| <= 1e-10 res_0
after it); final x within 1e-10 relative elementwise."""
import numpy as np
import pytest

from conftest import check_history, rel_gap

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_2602_21897_b200")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0")


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


# ------------------------------------------------------------------- K0

@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 2, 2), (4, 3, 5), (5, 5, 5), (6, 5, 4)])
def test_structure_bit_exact_vs_golden(rt, golden, dims):
    A = P.gen_stencil_matrix(*dims, rt=rt)
    rp, ci, va = A.to_csr()
    key = "csr_%dx%dx%d" % dims
    assert np.array_equal(rp, golden[key + "_row_ptr"])
    assert np.array_equal(ci, golden[key + "_col_idx"])
    assert np.array_equal(va, golden[key + "_values"])
    A.validate()


@pytest.mark.parametrize("dims", [(3, 1, 7), (1, 9, 2), (33, 17, 5), (32, 32, 32), (64, 48, 40),
                                  (128, 128, 128)])
def test_structure_bit_exact_vs_oracle(rt, orc, dims):
    A = P.gen_stencil_matrix(*dims, rt=rt)
    m = orc.stencil(*dims)
    rp, ci, va = A.to_csr()
    assert A.nnz() == m.nnz
    assert np.array_equal(rp, m.row_ptr)
    assert np.array_equal(ci, m.col_idx)
    assert np.array_equal(va, m.values)
    assert A.info.max_width == (27 if min(dims) >= 3 else A.info.max_width)


@pytest.mark.parametrize("dims,zb,ze", [((8, 6, 10), 0, 3), ((8, 6, 10), 3, 7), ((8, 6, 10), 7, 10),
                                        ((5, 7, 4), 1, 2)])
def test_slab_structure_is_a_row_block(rt, orc, dims, zb, ze):
    nx, ny, nz = dims
    A = P.gen_stencil_matrix(nx, ny, nz, rt=rt, z_begin=zb, z_end=ze)
    m = orc.stencil(*dims)
    r0, r1 = zb * nx * ny, ze * nx * ny
    rp, ci, va = A.to_csr()
    assert np.array_equal(rp, m.row_ptr[r0:r1 + 1] - m.row_ptr[r0])
    assert np.array_equal(ci, m.col_idx[m.row_ptr[r0]:m.row_ptr[r1]])
    assert np.array_equal(va, m.values[m.row_ptr[r0]:m.row_ptr[r1]])
    assert A.info.row_offset == r0
    assert A.info.col_offset == max(zb - 1, 0) * nx * ny


def test_bad_dims_config_error(rt):
    with pytest.raises(P.ConfigError):
        P.gen_stencil_matrix(0, 1, 1, rt=rt)  # csr.cpp:30-31
    with pytest.raises(P.ConfigError):
        P.gen_stencil_matrix(1 << 40, 1 << 20, 1, rt=rt)  # csr.cpp:32-34
    with pytest.raises(P.ContractViolation):
        P.gen_stencil_matrix(4, 4, 4, rt=rt, z_begin=3, z_end=2)


def test_from_csr_roundtrip_and_validation(rt, orc):
    m = orc.stencil(7, 5, 3)
    vals = m.values.copy()
    vals[5] = 0.1 + 1.0 / 3.0  # full-precision-hostile value (test_bench.cpp:117-130)
    A = P.ell_from_csr(m.row_ptr, m.col_idx, vals, rt=rt)
    rp, ci, va = A.to_csr()
    assert np.array_equal(rp, m.row_ptr) and np.array_equal(ci, m.col_idx)
    assert np.array_equal(va, vals)
    bad = m.col_idx.copy()
    bad[0] = 99999
    with pytest.raises(P.ConfigError):
        P.ell_from_csr(m.row_ptr, bad, m.values, rt=rt)  # test_bench.cpp:132-135
    rpb = m.row_ptr.copy()
    rpb[1] = rpb[2] + 1
    with pytest.raises(P.ConfigError):
        P.ell_from_csr(rpb, m.col_idx, m.values, rt=rt)


# ------------------------------------------------------------------- K1

@pytest.mark.parametrize("dims", [(6, 5, 4), (32, 32, 32), (37, 29, 23), (128, 128, 128)])
def test_spmv_bit_exact(rt, orc, golden, dims):
    A = P.gen_stencil_matrix(*dims, rt=rt)
    m = orc.stencil(*dims)
    x = orc.rhs_xorshift(m.n, 3) if dims == (6, 5, 4) else orc.rhs_splitmix(m.n, 11) - 0.5
    xd, yd = dev(x), torch.zeros(m.n, dtype=torch.float64, device="cuda:0")
    P.spmv_range(A, xd, yd, 0, m.n)
    y = host(yd)
    want = golden["spmv_6x5x4_y"] if dims == (6, 5, 4) else orc.spmv(m, x)
    assert np.array_equal(y, want)
    # fused K1: same Ap bits, p.Ap within reassociation error
    y2 = torch.zeros_like(yd)
    d = P.spmv_dot(A, xd, y2, 0, m.n)
    assert np.array_equal(host(y2), want)
    assert rel_gap(d, orc.dot(x, want)) < 1e-12


def test_spmv_tiled_equals_full(rt, orc):
    m = orc.stencil(6, 5, 4)  # test_bench.cpp:177-186
    A = P.gen_stencil_matrix(6, 5, 4, rt=rt)
    x = dev(orc.rhs_xorshift(m.n, 3))
    full = torch.zeros(m.n, dtype=torch.float64, device="cuda:0")
    tiled = torch.zeros_like(full)
    P.spmv_range(A, x, full, 0, m.n)
    for t in P.make_tile_plan(A, 7):
        P.spmv_range(A, x, tiled, t.r0, t.r1)
    assert torch.equal(full, tiled)


def test_spmv_identity_hand_matrix_and_padding(rt, orc):
    ident = P.ell_from_csr(np.arange(6), np.arange(5), np.ones(5), rt=rt)
    x = orc.rhs_xorshift(5, 11)
    y = torch.zeros(5, dtype=torch.float64, device="cuda:0")
    P.spmv_range(ident, dev(x), y, 0, 5)
    assert np.array_equal(host(y), x)
    H = P.ell_from_csr([0, 2, 3, 6], [0, 2, 1, 0, 1, 2], [2, 1, 3, 4, 5, 6], rt=rt)
    y = torch.zeros(3, dtype=torch.float64, device="cuda:0")
    P.spmv_range(H, dev(np.array([1.0, -2.0, 3.0])), y, 0, 3)
    assert np.array_equal(host(y), [5.0, -6.0, 12.0])
    # ragged rows of a general matrix (padding masked, -0.0 preserved)
    rng = np.random.default_rng(5)
    n = 300
    lens = rng.integers(0, 40, n)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int64)
    va = rng.standard_normal(len(ci))
    from oracle import Csr
    G = P.ell_from_csr(rp, ci, va, rt=rt)
    xv = rng.standard_normal(n)
    y = torch.zeros(n, dtype=torch.float64, device="cuda:0")
    P.spmv_range(G, dev(xv), y, 0, n)
    assert np.array_equal(host(y), orc.spmv(Csr(n, rp, ci, va), xv))


# ------------------------------------------------------------------- K2-K4

def test_waxpby_bit_exact_and_aliasing(rt, orc):
    n = 257  # test_bench.cpp:207-222
    x, y = orc.rhs_xorshift(n, 21), orc.rhs_xorshift(n, 22)
    xd, yd, wd = dev(x), dev(y), torch.zeros(n, dtype=torch.float64, device="cuda:0")
    P.waxpby_range(1.0, xd, 0.0, yd, wd, 0, n, rt=rt)
    assert np.array_equal(host(wd), x)
    P.waxpby_range(0.0, xd, 1.0, yd, wd, 0, n, rt=rt)
    assert np.array_equal(host(wd), y)
    P.waxpby_range(2.0, xd, 3.0, yd, wd, 0, n, rt=rt)
    assert np.array_equal(host(wd), orc.waxpby(2.0, x, 3.0, y))
    P.waxpby_range(1.0, xd, -0.37, yd, xd, 3, 200, rt=rt)  # w aliases x
    want = x.copy()
    want[3:200] = orc.waxpby(1.0, x, -0.37, y)[3:200]
    assert np.array_equal(host(xd), want)


def test_standalone_fused_updates_bit_exact(rt, orc):
    """tw_update_xr_rr / tw_update_p (K2 / K3 as operators) against the
    reference's waxpby_range and dot_range on ragged ranges."""
    n = 100_003
    x, p, r, ap = (orc.rhs_splitmix(n, s) for s in (1, 2, 3, 4))
    alpha, beta = 0.3712345678901, -1.25e-3
    for i0, i1 in ((0, n), (1, n - 1), (7, 8), (5, 5)):
        xd, pd, rd, ad = dev(x), dev(p), dev(r), dev(ap)
        rr = P.update_xr_rr(alpha, xd, pd, rd, ad, i0, i1, rt=rt)
        wx, wr = x.copy(), r.copy()
        wx[i0:i1] = orc.waxpby(1.0, x, alpha, p)[i0:i1]
        wr[i0:i1] = orc.waxpby(1.0, r, -alpha, ap)[i0:i1]
        assert np.array_equal(host(xd), wx) and np.array_equal(host(rd), wr)
        want = orc.dot(wr, wr, i0, i1) if i1 > i0 else 0.0
        assert (rr == want == 0.0) or rel_gap(rr, want) < 1e-12
        P.update_p(beta, rd, pd, i0, i1, rt=rt)
        wp = p.copy()
        wp[i0:i1] = orc.waxpby(1.0, wr, beta, p)[i0:i1]
        assert np.array_equal(host(pd), wp)


def test_dot_identities(rt, orc):
    n = 1000  # test_bench.cpp:188-205
    ones = dev(np.ones(n))
    assert P.dot_range(ones, ones, 0, n, rt=rt) == float(n)
    a, b = orc.rhs_xorshift(n, 5), orc.rhs_xorshift(n, 9)
    assert rel_gap(P.dot_range(dev(a), dev(b), 0, n, rt=rt), orc.dot(a, b)) < 1e-12
    big = orc.rhs_splitmix(3_000_001, 2)
    bd = dev(big)
    assert rel_gap(P.dot_range(bd, bd, 17, 3_000_001, rt=rt), orc.dot(big, big, 17)) < 1e-12
    assert P.dot_range(bd, bd, 5, 5, rt=rt) == 0.0


def test_standalone_reductions_on_concurrent_streams(rt, orc):
    """tw_dot_range / tw_spmv_dot called on several streams at once (the
    reference's kernels may run from any worker, kernels.hpp:7-9): each
    stream has its own reduction scratch, so every result is the one the
    same call gives alone."""
    import ctypes
    from paper_2602_21897_b200 import _native as N
    lib = N.load()
    n = 4_000_003
    vecs = [dev(orc.rhs_splitmix(n, s)) for s in range(4)]
    want = [P.dot_range(v, v, 0, n, rt=rt) for v in vecs]
    A = P.gen_stencil_matrix(64, 64, 64, rt=rt)
    p = dev(orc.rhs_xorshift(A.n, 3))
    Ap = torch.empty(A.n, dtype=torch.float64, device="cuda:0")
    want_pap = P.spmv_dot(A, p, Ap, 0, A.n)
    streams = [torch.cuda.Stream() for _ in range(4)]
    outs = torch.zeros(8, dtype=torch.float64, device="cuda:0")
    aps = [torch.empty(A.n, dtype=torch.float64, device="cuda:0") for _ in range(4)]
    torch.cuda.synchronize()
    for rep in range(5):
        for i, st in enumerate(streams):
            N.check(lib.tw_dot_range(rt.h, ctypes.c_void_p(vecs[i].data_ptr()),
                                     ctypes.c_void_p(vecs[i].data_ptr()), 0, n,
                                     ctypes.c_void_p(outs.data_ptr() + 8 * i),
                                     ctypes.c_void_p(st.cuda_stream)))
            N.check(lib.tw_spmv_dot(A.h, ctypes.c_void_p(p.data_ptr()),
                                    ctypes.c_void_p(aps[i].data_ptr()), 0, A.n,
                                    ctypes.c_void_p(outs.data_ptr() + 8 * (4 + i)),
                                    ctypes.c_void_p(st.cuda_stream)))
        got = host(outs)
        assert list(got[:4]) == want and all(g == want_pap for g in got[4:])


def test_rhs_generators_bit_exact(rt, orc):
    for first, count in [(0, 1000), (12345, 70000)]:
        b = host(torch.zeros(count, dtype=torch.float64, device="cuda:0"))
        xs = torch.zeros(count, dtype=torch.float64, device="cuda:0")
        P.rhs_xorshift(rt, count, 7, first, out=xs)
        assert np.array_equal(host(xs), orc.rhs_xorshift(first + count, 7)[first:])
        sm = torch.zeros(count, dtype=torch.float64, device="cuda:0")
        P.rhs_splitmix(rt, count, 7, first, out=sm)
        assert np.array_equal(host(sm), orc.rhs_splitmix(first + count, 7)[first:])
        del b


@pytest.mark.parametrize("T", [1, 3, 7])
def test_tile_plan_vs_golden(rt, golden, T):
    A = P.gen_stencil_matrix(5, 4, 3, rt=rt)
    got = np.array([[t.r0, t.r1, t.band_lo, t.band_hi] for t in P.make_tile_plan(A, T)]).T
    assert np.array_equal(got, golden["tiles_5x4x3_T%d" % T])
    with pytest.raises(P.ConfigError):
        P.make_tile_plan(A, 0)
    with pytest.raises(P.ConfigError):
        P.make_tile_plan(A, A.n + 1)


# ------------------------------------------------------------------- CG

@pytest.mark.parametrize("variant,T,graph", [("mono", 1, False), ("mono", 1, True),
                                             ("tasks", 4, False), ("tasks", 16, True),
                                             ("tasks", 64, False)])
def test_cg_32cubed_vs_reference(rt, orc, golden, variant, T, graph):
    """Acceptance criterion 5 input (acceptance.cpp:298-349) at 150 iterations."""
    A = P.gen_stencil_matrix(32, 32, 32, rt=rt)
    b = orc.rhs_xorshift(A.n, 7)
    opt = P.CgOptions(tiles=T, use_graph=graph)
    run = P.cg_monolithic if variant == "mono" else P.cg_tasks
    res = run(rt, A, b, 150, opt)
    check_history(res.residual_history, golden["cg_32_xorshift7_history"])
    assert np.all(rel_gap(res.x, golden["cg_32_xorshift7_x"]) <= 1e-10)
    h = res.residual_history[:50]
    assert np.all(h[1:] <= h[:-1] * (1 + 1e-12))
    if variant == "tasks":
        check_history(res.residual_history[:50], golden["cgtasks_32_T%d_history" % T]
                      if "cgtasks_32_T%d_history" % T in golden else h)


def test_cg_splitmix_and_small_cases(rt, orc, golden):
    A = P.gen_stencil_matrix(32, 32, 32, rt=rt)
    res = P.cg_monolithic(rt, A, orc.rhs_splitmix(A.n, 7), 150)
    check_history(res.residual_history, golden["cg_32_splitmix7_history"])
    A8 = P.gen_stencil_matrix(8, 8, 8, rt=rt)  # test_bench.cpp:275-295
    b8 = golden["cg_8_xorshift7_b"]
    for T in (1, 4, 16):
        r = P.cg_tasks(rt, A8, b8, 10, P.CgOptions(tiles=T))
        check_history(r.residual_history, golden["cg_8_xorshift7_history"])
    A6 = P.gen_stencil_matrix(6, 6, 6, rt=rt)  # test_bench.cpp:307-334
    r = P.cg_tasks(rt, A6, golden["cg_6_xorshift17_b"], 8, P.CgOptions(tiles=8))
    check_history(r.residual_history, golden["cg_6_device_ta_T8_history"])


def test_cg_identity_converges(rt, golden):
    ident = P.ell_from_csr(np.arange(7), np.arange(6), np.ones(6), rt=rt)
    r = P.cg_monolithic(rt, ident, golden["cg_identity_b"], 1, P.CgOptions(tol=1e-12))
    assert r.converged and abs(r.residual_history[0]) < 1e-14
    assert np.allclose(r.x, golden["cg_identity_b"], rtol=1e-14)


def test_cg_deterministic_and_marks(rt, orc):
    A = P.gen_stencil_matrix(48, 40, 36, rt=rt)
    b = orc.rhs_xorshift(A.n, 7)
    r1 = P.cg_tasks(rt, A, b, 30, P.CgOptions(tiles=8))
    r2 = P.cg_tasks(rt, A, b, 30, P.CgOptions(tiles=8, use_graph=True))
    assert np.array_equal(r1.residual_history, r2.residual_history)
    assert np.array_equal(r1.x, r2.x)
    assert np.all(r1.iteration_marks > 0) and np.all(np.diff(r1.iteration_marks) >= 0)
    m = orc.stencil(48, 40, 36)
    h, x, _ = orc.cg(m, b, 30, tiles=8)
    check_history(r1.residual_history, h)
    assert np.all(rel_gap(r1.x, x) <= 1e-10)


def test_cg_task_dag_edges_match_reference(rt, orc, golden):
    A = P.gen_stencil_matrix(4, 4, 4, rt=rt)
    s = P.CgSolver(rt, A, 2, P.CgOptions(tiles=4))
    s.set_rhs(orc.rhs_xorshift(64, 7))
    s.iterate(2)
    s.wait()
    got = sorted(" ".join(e) for e in s.task_edges())
    want = sorted(str(e) for e in golden["dag_4x4x4_T4_it2_edges"])
    assert got == want
    s.close()


def test_cg_iterate_in_pieces_equals_one_shot(rt, orc):
    A = P.gen_stencil_matrix(20, 20, 20, rt=rt)
    b = orc.rhs_splitmix(A.n, 3)
    for variant in (0, 1):
        s = P.CgSolver(rt, A, 40, P.CgOptions(tiles=5), variant=variant)
        s.set_rhs(b)
        s.iterate(13)
        s.iterate(27)
        h = s.history(40)
        x = s.solution()
        s.set_rhs(dev(b))
        s.iterate(40)
        assert np.array_equal(h, s.history(40)) and np.array_equal(x, s.solution())
        with pytest.raises(P.ContractViolation):
            s.iterate(1)
        s.close()


def test_cg_256_properties(rt):
    """Full-size (256^3) properties the domain offers: residual non-increasing,
    deterministic replay, and r = b - A x consistency of the recurrence."""
    A = P.gen_stencil_matrix(256, 256, 256, rt=rt)
    assert A.nnz() == 449455096 and A.info.max_width == 27
    n = A.n
    b = P.rhs_xorshift(rt, n, 7)
    s = P.CgSolver(rt, A, 20, P.CgOptions(iteration_marks=False), variant=0)
    s.set_rhs(b)
    s.iterate(20)
    h = s.history(20)
    assert np.all(h[1:] <= h[:-1] * (1 + 1e-12))
    x, r, p, Ap = s.vectors()
    # true residual ||b - A x|| tracks the recurrence residual (CG, 20 its)
    xt = torch.zeros(n, dtype=torch.float64, device="cuda:0")
    bt = torch.zeros(n, dtype=torch.float64, device="cuda:0")
    import ctypes
    ctypes.memmove  # noqa
    from paper_2602_21897_b200 import _native as N
    N.check(N.load().tw_memcpy(rt.h, ctypes.c_void_p(xt.data_ptr()), ctypes.c_void_p(x), 8 * n, None))
    N.check(N.load().tw_memcpy(rt.h, ctypes.c_void_p(bt.data_ptr()), ctypes.c_void_p(b.ptr), 8 * n, None))
    rt.synchronize()
    ax = torch.zeros_like(xt)
    P.spmv_range(A, xt, ax, 0, n)
    rt.synchronize()
    true_res = torch.linalg.norm(bt - ax).item()
    assert abs(true_res - h[-1]) / h[-1] < 1e-6
    s.set_rhs(b)
    s.iterate(20)
    assert np.array_equal(h, s.history(20))
    s.close()


# ------------------------------------------------------------ interop (f)

def test_load_csr_to_device_round_trip(rt, golden):
    text = str(golden["csr_text_3x3x3"][0])
    A = P.load_csr(text, rt=rt)
    assert P.dump_csr(A) == text
    with pytest.raises(P.ConfigError):
        P.load_csr("# taskweave csr v1\n2 2\n0 1 2\n0 1\n26\n", rt=rt)


def test_scenario_run_point_csv(rt, orc, golden):
    from paper_2602_21897_b200 import scenario as S
    c = S.ScenarioConfig(nx=32, ny=32, nz=32, iterations=20, warmup=5, repetitions=2,
                         tiles=[1, 4, 16], variant="tasks")
    pts = S.run_sweep(c, rt=rt)  # 16 tiles: the persistent dispatcher (automatic dispatch)
    assert [p.tile for p in pts] == [1, 4, 16]
    # automatic dispatch: 1 tile streams (3 launches per iteration: alpha and
    # beta_res fold into the tile kernels on one rank); small
    # tiles of an x-staged matrix the persistent dispatcher (one launch)
    assert pts[0].rows[0].tasks_executed == 3 * 20
    assert pts[1].rows[0].tasks_executed == 1 and pts[2].rows[0].tasks_executed == 1
    for p in pts:
        assert len(p.rows) == 40
        assert all(r.warmup for r in p.rows[:20])            # repetition 0 is warm-up
        assert [r.warmup for r in p.rows[20:]] == [True] * 5 + [False] * 15
        assert all(r.iter_time > 0 for r in p.rows) and p.steady_iter_time > 0
        check_history(p.residual_history, golden["cg_32_splitmix7_history"][:20])
    text = S.metrics_to_csv(pts)
    assert S.parse_metrics_csv(text) == [r for p in pts for r in p.rows]


# ------------------------------------------------ persistent DAG dispatcher

@pytest.mark.parametrize("T", [1, 4, 16, 64])
def test_persistent_dispatcher_vs_reference(rt, orc, golden, T):
    A = P.gen_stencil_matrix(32, 32, 32, rt=rt)
    b = orc.rhs_xorshift(A.n, 7)
    r1 = P.cg_tasks(rt, A, b, 150, P.CgOptions(tiles=T, persistent=True))
    check_history(r1.residual_history, golden["cg_32_xorshift7_history"])
    assert np.all(rel_gap(r1.x, golden["cg_32_xorshift7_x"]) <= 1e-10)
    if "cgtasks_32_T%d_history" % T in golden:
        check_history(r1.residual_history[:50], golden["cgtasks_32_T%d_history" % T])
    r2 = P.cg_tasks(rt, A, b, 150, P.CgOptions(tiles=T, persistent=True))
    assert np.array_equal(r1.residual_history, r2.residual_history)  # deterministic
    assert np.array_equal(r1.x, r2.x)


def test_persistent_dispatcher_pieces_times_and_rejects(rt, orc):
    A = P.gen_stencil_matrix(40, 36, 30, rt=rt)
    b = orc.rhs_splitmix(A.n, 5)
    s = P.CgSolver(rt, A, 30, P.CgOptions(tiles=6, persistent=True))
    s.set_rhs(b)
    s.iterate(7)
    s.iterate(23)
    h, x = s.history(30), s.solution()
    t = s.iteration_times(30)
    assert np.all(t > 0) and np.all(t < 1.0)
    s.set_rhs(b)
    s.iterate(30)
    assert np.array_equal(h, s.history(30)) and np.array_equal(x, s.solution())
    s.close()
    m = orc.stencil(40, 36, 30)
    want, _, _ = orc.cg(m, b, 30, tiles=6)
    check_history(h, want)
    with pytest.raises(P.ConfigError):
        P.CgSolver(rt, A, 5, P.CgOptions(tiles=1, persistent=True), variant=0)
    with pytest.raises(P.ConfigError):
        P.CgSolver(rt, A, 5, P.CgOptions(tiles=4, persistent=True, use_graph=True))


# ------------------------------------------------ distributed code path (1 rank)

def test_distributed_code_path_on_one_rank(orc, golden):
    """A real 1-rank NCCL communicator drives the multi-GPU code path on the
    one available B200: NCCL loading and comm init, the halo group on the comm
    stream, the interior/boundary SpMV split, allgathers of the rank partials
    (joined through the comm stream), rank-ordered scalar sums inside K2/K3 and
    K3's last-block commit of rtrans/history."""
    rt2 = P.Runtime(0)
    rt2.init_comm(0, 1, P.Runtime.comm_unique_id())
    assert (rt2.rank, rt2.nranks) == (0, 1)
    A = P.gen_stencil_matrix(32, 32, 32, rt=rt2)
    b = orc.rhs_xorshift(A.n, 7)
    for run, T, graph in [(P.cg_monolithic, 1, False), (P.cg_tasks, 4, False),
                          (P.cg_monolithic, 1, True)]:
        res = run(rt2, A, b, 150, P.CgOptions(tiles=T, use_graph=graph))
        check_history(res.residual_history, golden["cg_32_xorshift7_history"])
        assert np.all(rel_gap(res.x, golden["cg_32_xorshift7_x"]) <= 1e-10)
    s = P.CgSolver(rt2, A, 4, P.CgOptions(), variant=0)
    assert s.launches_per_iteration() == (5, 3)
    s.close()
    # exchange_externals on the 1-rank communicator: no neighbour, a no-op
    xv = dev(b)
    P.halo_exchange(A, xv)
    assert np.array_equal(host(xv), b)
    # the persistent dispatcher on the 1-rank communicator (no halo task,
    # alpha / beta_res local) and over its peer transport (publication and
    # gather through the one rank's window, flags stamped per iteration)
    for peer in (False, True):
        s = P.CgSolver(rt2, A, 150, P.CgOptions(tiles=4, persistent=True, iteration_marks=False),
                       variant=1)
        if peer:
            s.peer_connect([s.peer_export()])
        s.set_rhs(b)
        s.iterate(60)
        s.iterate(90)
        check_history(s.history(150), golden["cg_32_xorshift7_history"])
        assert np.all(rel_gap(s.solution(), golden["cg_32_xorshift7_x"]) <= 1e-10)
        s.close()
    # the NVLink peer transport on the same 1-rank communicator: export /
    # connect (own window, no IPC mapping), fused publish / wait kernels
    for graph in (False, True):
        s = P.CgSolver(rt2, A, 150, P.CgOptions(use_graph=graph), variant=0)
        with pytest.raises(P.ContractViolation):
            s.peer_ping_send()  # not connected yet
        blob = s.peer_export()
        bad = bytearray(blob)
        bad[152] ^= 1  # a different plane size
        with pytest.raises(P.ContractViolation):
            s.peer_connect([bytes(bad)])
        s.peer_connect([blob])
        s.peer_ping_send()
        assert s.peer_ping_check(1000)
        with pytest.raises(P.ContractViolation):
            s.peer_connect([s.peer_export()])  # connected once per solver
        assert s.launches_per_iteration() == (4, 0)
        s.set_rhs(b)
        s.iterate(70)
        s.iterate(80)
        check_history(s.history(150), golden["cg_32_xorshift7_history"])
        assert np.all(rel_gap(s.solution(), golden["cg_32_xorshift7_x"]) <= 1e-10)
        s.close()
    rt2.close()


def test_timed_graph_kernel_times(rt, orc):
    A = P.gen_stencil_matrix(48, 48, 48, rt=rt)
    b = orc.rhs_xorshift(A.n, 7)
    S = P.CgSolver(rt, A, 30, P.CgOptions(use_graph=True, iteration_marks=False), variant=0)
    S.set_rhs(b)
    S.enable_kernel_timing(True)
    S.iterate(20)
    k1, k2, k3, n = S.kernel_times()
    assert n == 20 and k1 > 0 and k2 > 0 and k3 > 0
    h = S.history(20)
    S.set_rhs(b)
    S.enable_kernel_timing(False)
    S.iterate(20)
    assert np.array_equal(h, S.history(20))
    S.close()


def test_general_matrix_with_empty_slices(rt, orc):
    """Rows 32..95 empty (two whole slices of width 0), long rows elsewhere:
    SpMV bit-exact, empty rows give +0.0, CG on an SPD general matrix."""
    from oracle import Csr
    rng = np.random.default_rng(9)
    n = 200
    lens = rng.integers(1, 60, n)
    lens[32:96] = 0
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int64)
    va = rng.standard_normal(len(ci))
    G = P.ell_from_csr(rp, ci, va, rt=rt)
    assert G.info.max_width == lens.max()
    x = rng.standard_normal(n)
    y = torch.full((n,), 7.0, dtype=torch.float64, device="cuda:0")
    P.spmv_range(G, dev(x), y, 0, n)
    want = orc.spmv(Csr(n, rp, ci, va), x)
    got = host(y)
    assert np.array_equal(got, want) and np.all(got[32:96] == 0.0)
    # SPD: diagonally dominant symmetric tridiagonal + identity rows
    m = 150
    rows = [[(i, 4.0)] + ([(i - 1, -1.0)] if i else []) + ([(i + 1, -1.0)] if i + 1 < m else [])
            for i in range(m)]
    rows = [sorted(r) for r in rows]
    rp2 = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    ci2 = np.array([c for r in rows for c, _ in r], np.int64)
    va2 = np.array([v for r in rows for _, v in r])
    T = P.ell_from_csr(rp2, ci2, va2, rt=rt)
    b = orc.rhs_xorshift(m, 3)
    for run in (P.cg_monolithic, P.cg_tasks):
        res = run(rt, T, b, 12, P.CgOptions(tiles=3))
        want_h, want_x, _ = orc.cg(Csr(m, rp2, ci2, va2), b, 12, tiles=1 if run is P.cg_monolithic else 3)
        check_history(res.residual_history, want_h)


def test_cg_128cubed_vs_oracle(rt, orc):
    """Mid-size parity (C2 grid): monolithic, 8-tile DAG and the dispatcher
    against the oracle's cg_reference / tile-order cg on 128^3, 25 iterations."""
    m = orc.stencil(128, 128, 128)
    b = orc.rhs_splitmix(m.n, 7)
    want_h, want_x, _ = orc.cg(m, b, 25)
    A = P.gen_stencil_matrix(128, 128, 128, rt=rt)
    for run, opt in [(P.cg_monolithic, P.CgOptions()),
                     (P.cg_tasks, P.CgOptions(tiles=8, use_graph=True)),
                     (P.cg_tasks, P.CgOptions(tiles=8, persistent=True))]:
        res = run(rt, A, b, 25, opt)
        check_history(res.residual_history, want_h)
        assert np.all(rel_gap(res.x, want_x) <= 1e-10)


# ------------------------------------------- emulated multi-rank group (1 GPU)

@pytest.mark.parametrize("transport", ["loopback", "peer"])
@pytest.mark.parametrize("dims,P_", [((32, 32, 32), 2), ((40, 24, 30), 3), ((32, 32, 32), 4),
                                     ((24, 20, 16), 8), ((16, 16, 2), 2)])
def test_emulated_rank_group_matches_single_domain(orc, golden, dims, P_, transport):
    """P z-slab ranks on the one B200 (tw_cg_group_*): slab matrices, ghost
    planes, interior/boundary SpMV split, rank-ordered scalar sums -- the
    multi-GPU code with loopback copies for the NCCL transport -- must
    reproduce the single-domain reference CG."""
    m = orc.stencil(*dims)
    b = orc.rhs_xorshift(m.n, 7)
    want_h, want_x, _ = orc.cg(m, b, 40)
    G = P.EmulatedRankGroup(*dims, P_, 40, transport=transport)
    G.set_rhs(b)
    G.iterate(15)
    G.iterate(25)
    hs = G.history(40)
    for h in hs:
        assert np.array_equal(h, hs[0])  # every rank holds the same scalars
    check_history(hs[0], want_h)
    assert np.all(rel_gap(G.solution(), want_x) <= 1e-10)
    G.close()
    if dims == (32, 32, 32):
        check_history(hs[0], golden["cg_32_xorshift7_history"][:40])


def test_peer_transport_resolve_new_epoch(orc):
    """A second solve on the peer transport: the flag stamps carry the solve
    epoch, so flags left by the first solve must not release the second."""
    dims = (24, 24, 24)
    m = orc.stencil(*dims)
    G = P.EmulatedRankGroup(*dims, 4, 30, transport="peer")
    assert G.peer_check() and G.peer_check()  # two rounds, fresh tokens
    # a rank that never sends: the others' check reports it (no trap, no hang)
    for s in G.solvers[1:]:
        s.peer_ping_send()
    assert not G.solvers[1].peer_ping_check(50)
    for seed in (3, 11, 3):
        b = orc.rhs_xorshift(m.n, seed)
        want_h, want_x, _ = orc.cg(m, b, 30)
        G.set_rhs(b)
        G.iterate(30)
        check_history(G.history(30)[0], want_h)
        assert np.all(rel_gap(G.solution(), want_x) <= 1e-10)
    G.close()


def test_peer_transport_contract_errors(rt):
    from paper_2602_21897_b200 import _native as N
    A = P.gen_stencil_matrix(8, 8, 8, rt=rt)
    with pytest.raises(P.ContractViolation):
        P.halo_exchange(A, dev(np.zeros(A.n)))  # no communicator
    s = P.CgSolver(rt, A, 5, variant=N.TW_CG_MONOLITHIC)
    with pytest.raises(P.ContractViolation):
        s.peer_export()  # single-rank context
    s.close()


def _read_dev(rt, ptr, n):
    import ctypes
    from paper_2602_21897_b200 import _native as N
    out = np.zeros(n, np.float64)
    N.check(N.load().tw_memcpy(rt.h, out.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(ptr),
                               8 * n, None))
    rt.synchronize()
    return out


@pytest.mark.parametrize("maxw", [9, 33, 34, 70])
def test_spmv_generic_widths_tma_and_register_paths(rt, orc, maxw):
    """Random general matrices whose slice widths are mostly outside the
    stencil's fixed set {8, 12, 18, 27}: the TMA-staged kernel's generic row
    body (max width <= 33 fits 18 warps' stages in shared memory) and the
    register-path fallback (34, 70) must both be bit-exact, including the
    fused p.Ap dot's inputs (spmv_dot) and ragged last slices."""
    from oracle import Csr
    rng = np.random.default_rng(maxw)
    n = 32 * 37 + 11
    lens = rng.integers(0, maxw + 1, n)
    lens[5] = maxw
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int64)
    va = rng.standard_normal(len(ci))
    G = P.ell_from_csr(rp, ci, va, rt=rt)
    assert G.info.max_width == maxw
    x = rng.standard_normal(n)
    want = orc.spmv(Csr(n, rp, ci, va), x)
    y = torch.zeros(n, dtype=torch.float64, device="cuda:0")
    P.spmv_range(G, dev(x), y, 0, n)
    assert np.array_equal(host(y), want)
    # sub-ranges with ragged ends
    y2 = torch.full((n,), -3.0, dtype=torch.float64, device="cuda:0")
    P.spmv_range(G, dev(x), y2, 45, n - 7)
    got = host(y2)
    assert np.array_equal(got[45:n - 7], want[45:n - 7])
    assert np.all(got[:45] == -3.0) and np.all(got[n - 7:] == -3.0)
    d = P.spmv_dot(G, dev(x), y, 0, n)
    assert abs(d - float(np.dot(x, want))) <= 1e-12 * np.abs(x * want).sum()


@pytest.mark.parametrize("dims,P_", [((32, 32, 32), 2), ((40, 24, 30), 3), ((32, 32, 32), 4),
                                     ((24, 20, 16), 8), ((23, 17, 12), 3), ((64, 24, 40), 4),
                                     ((32, 8, 32), 8)])
def test_peer_transport_under_concurrency(orc, golden, dims, P_):
    """The peer protocol with the ranks really running at the same time:
    tw_cg_group_iterate_concurrent runs all P ranks as one cooperative
    kernel whose rank groups spin on one another's flags (stamps, rank-order
    partial sums, fused halo stores), with and without rank-dependent
    delays, interleaved with host-sequenced iterations and a re-solve.
    Slabs with nx % 32 == 0 are x-staged: their K1 stages the ghost runs by
    TMA only after each warp's flag acquire and a proxy fence."""
    m = orc.stencil(*dims)
    G = P.EmulatedRankGroup(*dims, P_, 60, transport="peer")
    assert all(A.x_staged for A in G.mats)  # closed-form runs or a run table
    for seed in (7, 2):
        b = orc.rhs_xorshift(m.n, seed)
        want_h, want_x, _ = orc.cg(m, b, 60)
        G.set_rhs(b)
        G.iterate_concurrent(17)
        G.iterate(3)
        G.iterate_concurrent(40, jitter=True)
        hs = G.history(60)
        for h in hs:
            assert np.array_equal(h, hs[0])
        check_history(hs[0], want_h)
        assert np.all(rel_gap(G.solution(), want_x) <= 1e-10)
    G.close()


def test_streams_events_and_task_aware_binding():
    """The reference's QueuePool / Device / TaskAware layer over real CUDA
    objects (tw_stream_* / tw_event_*): FIFO pool exhaustion, a non-blocking
    query, a device-side edge and bind_event_async's release hook."""
    import threading
    rt = P.Runtime(0, stream_pool_capacity=2)
    s1, s2 = rt.acquire_stream(), rt.acquire_stream()
    assert s1 != s2
    got = []
    t = threading.Thread(target=lambda: got.append(rt.acquire_stream()))
    t.start()
    t.join(0.2)
    assert t.is_alive()  # pool exhausted: the third acquire waits (FIFO)
    rt.release_stream(s1)
    t.join(5)
    assert got == [s1]
    with pytest.raises(P.ContractViolation):
        rt.release_stream(12345)
    # a long kernel on s2, an event after it, an edge into s1 and a bound callback
    ts2 = torch.cuda.ExternalStream(s2)
    ev = P.Event()
    fired = threading.Event()
    with torch.cuda.stream(ts2):
        torch.cuda._sleep(200_000_000)  # ~0.1 s of GPU time
    ev.record(s2)
    ev.bind_async(rt, fired.set)
    assert not ev.query() and not fired.is_set()
    x = torch.zeros(1, device="cuda:0")
    ev.block_stream(s1)
    with torch.cuda.stream(torch.cuda.ExternalStream(s1)):
        x += 1  # ordered after the sleep through the event edge
    ev.wait(rt)
    assert ev.query()
    assert fired.wait(5)
    torch.cuda.synchronize()
    assert x.item() == 1.0
    rt.release_stream(s1)
    rt.release_stream(s2)
    with pytest.raises(P.ContractViolation):
        rt.release_stream(s2)  # double release (QueuePool::release, task_aware.cpp:150-153)
    s3 = rt.acquire_stream()
    rt.release_stream(s3)
    with pytest.raises(P.ContractViolation):
        rt.release_stream(s3)
    ev.close()
    rt.close()


def test_reference_binding_drop_in():
    """The INTEGRATION.md binding end to end: the reference's own CsrMatrix
    (its gen_stencil_matrix, compiled from its sources into oracle/_ref)
    through tw_cg_solve on the B200, checked against its own cg_reference."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "oracle", "_ref", "binding_demo")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/binding_demo not built (needs the reference tree at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "binding ok" in r.stdout


@pytest.mark.parametrize("dims,P_", [((32, 32, 32), 4), ((40, 24, 30), 3), ((24, 20, 16), 8),
                                     ((320, 288, 9), 3), ((320, 288, 12), 2), ((321, 287, 9), 3)])
def test_peer_transport_bit_identical_to_nccl_path(orc, dims, P_):
    """The peer transport sums the same partials in the same order as the
    NCCL path (whose emulation is the loopback group), so histories and x
    are identical to the bit -- the property bench.py's pre-timing
    validation relies on.  The 320x288 planes (>= one slice per warp in
    every range) run the peer path's one-launch K1 (launch_spmv_split)."""
    b = orc.rhs_xorshift(int(np.prod(dims)), 5)
    out = []
    for transport in ("loopback", "peer"):
        G = P.EmulatedRankGroup(*dims, P_, 40, transport=transport)
        if transport == "peer":  # one-launch K1 on the big planes
            assert G.solvers[0].launches_per_iteration() == ((3 if dims[0] >= 320 else 4), 0)
        G.set_rhs(b)
        G.iterate(40)
        out.append((G.history(40)[0], G.solution()))
        G.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
    if dims[0] >= 320:
        want_h, want_x, _ = orc.cg(orc.stencil(*dims), b, 40)
        check_history(out[1][0], want_h)
        assert np.all(rel_gap(out[1][1], want_x) <= 1e-10)


def test_auto_dispatch_and_persistent_marks(rt, orc):
    """TW_DISPATCH_AUTO (the C default): the persistent dispatcher for the
    tasks variant with small tiles (> 8 tiles on a gather matrix, < 400k
    rows per tile on an x-staged one), streams otherwise; the persistent path's
    per-iteration host marks are placed by the device clock before each
    call's polled mark (non-decreasing, each call's last one polled)."""
    A = P.gen_stencil_matrix(48, 40, 36, rt=rt)
    assert not A.set_x_staged(False)  # a gather matrix
    b = orc.rhs_xorshift(A.n, 3)
    want_h, want_x, _ = orc.cg(orc.stencil(48, 40, 36), b, 30)
    for T, want_k in ((16, 0), (4, 3 * 4)):
        s = P.CgSolver(rt, A, 30, P.CgOptions(tiles=T, auto_dispatch=True, iteration_marks=True))
        assert s.launches_per_iteration()[0] == want_k
        s.set_rhs(b)
        s.iterate(12)
        s.iterate(18)
        check_history(s.history(30), want_h)
        assert np.all(rel_gap(s.solution(), want_x) <= 1e-10)
        m = s.marks(30)  # polled marks share a poll's time stamp: non-decreasing
        assert np.all(m > 0) and np.all(np.diff(m) >= 0)
        t = s.iteration_times(30)
        assert np.all(t > 0)
        s.close()


def test_abi_misuse_is_reported_not_crashed(rt):
    """Misuse through the C ABI comes back as the reference's exception types
    (ConfigError / ContractViolation, types.hpp:23-33) with the context still
    usable afterwards: bad ranges, iterations beyond max_iterations, bad
    options, null scalars, slabs without a rank context."""
    import ctypes
    from paper_2602_21897_b200 import _native as N
    lib = N.load()
    A = P.gen_stencil_matrix(8, 8, 8, rt=rt)
    x = dev(np.ones(A.n))
    y = torch.zeros(A.n, dtype=torch.float64, device="cuda:0")
    with pytest.raises(P.ContractViolation):
        P.spmv_range(A, x, y, 0, A.n + 1)
    with pytest.raises(P.ContractViolation):
        P.spmv_range(A, x, y, 5, 4)
    with pytest.raises(P.ContractViolation):
        P.dot_range(x, x, 9, 3, rt=rt)
    with pytest.raises(P.ContractViolation):
        N.check(lib.tw_update_p(rt.h, None, ctypes.c_void_p(x.data_ptr()),
                                ctypes.c_void_p(y.data_ptr()), 0, 8, None))
    with pytest.raises(P.ConfigError):
        P.make_tile_plan(A, 0)
    with pytest.raises(P.ConfigError):
        P.make_tile_plan(A, A.n + 1)
    with pytest.raises(P.ConfigError):
        P.CgSolver(rt, A, 5, P.CgOptions(tiles=0))
    with pytest.raises(P.ConfigError):
        P.CgSolver(rt, A, 5, P.CgOptions(tiles=2), variant=7)
    with pytest.raises(P.ConfigError):
        P.CgSolver(rt, A, 5, P.CgOptions(tiles=2, persistent=True, use_graph=True))
    s = P.CgSolver(rt, A, 5, P.CgOptions(tiles=2))
    s.set_rhs(np.ones(A.n))
    with pytest.raises(P.ContractViolation):
        s.iterate(6)  # beyond max_iterations
    with pytest.raises(P.ContractViolation):
        s.set_rhs(np.ones(A.n + 1))
    s.iterate(5)
    assert np.all(np.isfinite(s.history(5)))
    s.close()
    slab = None
    with pytest.raises(P.ContractViolation):  # a partial slab needs a rank context
        slab = P.gen_stencil_matrix(8, 8, 8, rt=rt, z_begin=0, z_end=4)
        P.CgSolver(rt, slab, 5, P.CgOptions(), variant=N.TW_CG_MONOLITHIC)
    # the context is still fine
    P.spmv_range(A, x, y, 0, A.n)
    torch.cuda.synchronize()


@pytest.mark.parametrize("dims", [(32, 32, 32), (64, 32, 24), (96, 5, 7), (32, 1, 3), (30, 20, 18),
                                  (5, 7, 9)])
def test_x_staged_k1_bit_identical(rt, orc, dims):
    """Every stencil matrix carries 16-bit columns into per-slice staged runs
    of x (closed-form runs for nx % 32 == 0, a per-slice run table
    otherwise), and the CG's K1 reads its operands from shared memory.  Same
    per-row order and roundings, same reductions: histories and x
    bit-identical to the gather path (the staged form dropped), and within
    the rule of the oracle."""
    b = orc.rhs_xorshift(int(np.prod(dims)), 9)
    out = []
    for stage in (True, False):
        A = P.gen_stencil_matrix(*dims, rt=rt)
        assert A.x_staged
        if not stage:
            assert not A.set_x_staged(False)
        for graph in (False, True):
            res = P.cg_monolithic(rt, A, b, 40, P.CgOptions(use_graph=graph))
            out.append((res.residual_history, res.x))
        for T in (3, 16):  # tiles cut slices: partial slices at the tile edges
            res = P.cg_tasks(rt, A, b, 40, P.CgOptions(tiles=T))
            out.append((res.residual_history, res.x))
    # out: [mono, mono graph, tasks T=3, tasks T=16] staged, then the same gathered
    def same(i, j):
        return np.array_equal(out[i][0], out[j][0]) and np.array_equal(out[i][1], out[j][1])
    assert same(0, 1) and same(0, 4) and same(0, 5)   # monolithic
    assert same(2, 6) and same(3, 7)                  # tasks, per tile count
    want_h, want_x, _ = orc.cg(orc.stencil(*dims), b, 40)
    check_history(out[0][0], want_h)
    assert np.all(rel_gap(out[0][1], want_x) <= 1e-10)


@pytest.mark.parametrize("dims", [(32, 16, 8), (30, 20, 18), (7, 5, 3)])
def test_csr_drop_in_gets_the_staged_k1(rt, orc, dims):
    """A caller's CsrMatrix (the reference's gen_stencil_matrix output, here
    the oracle's bit-identical one) through tw_ell_from_csr gets the x-staged
    form as a per-slice run table; its CG is bit-identical to the device-
    generated stencil's, and its staged columns decode to the CSR exactly."""
    m = orc.stencil(*dims)
    A = P.ell_from_csr(m.row_ptr, m.col_idx, m.values, rt=rt)
    assert A.x_staged
    rp, ci, va = A.to_csr_rows(0, m.n, staged=True)
    assert np.array_equal(rp, m.row_ptr) and np.array_equal(ci, m.col_idx)
    assert np.array_equal(va, m.values)
    G = P.gen_stencil_matrix(*dims, rt=rt)
    b = orc.rhs_xorshift(m.n, 3)
    r1 = P.cg_monolithic(rt, A, b, 30, P.CgOptions())
    r2 = P.cg_monolithic(rt, G, b, 30, P.CgOptions())
    assert np.array_equal(r1.residual_history, r2.residual_history)
    assert np.array_equal(r1.x, r2.x)
    r3 = P.cg_tasks(rt, A, b, 30, P.CgOptions(tiles=8, persistent=True))
    want_h, want_x, _ = orc.cg(m, b, 30)
    for r in (r1, r3):
        check_history(r.residual_history, want_h)
        assert np.all(rel_gap(r.x, want_x) <= 1e-10)


@pytest.mark.parametrize("seed", [1, 2])
def test_csr_run_table_general_matrix(rt, orc, seed):
    """A random banded matrix (columns within +-40 of the diagonal, SPD by
    diagonal dominance): its slices fit 9 runs of 36, so it is staged through
    the run table; SpMV-driven CG bit-identical to the gather form, and the
    staged columns decode to the CSR.  A matrix with wide-spread columns
    stays unstaged (the gather K1)."""
    rng = np.random.default_rng(seed)
    n = 3000
    rows, cols = [], []
    for i in range(n):
        c = np.unique(np.clip(i + rng.integers(-40, 41, size=9), 0, n - 1))
        c = np.union1d(c, [i])
        rows.append(len(c))
        cols.append(c)
    rp = np.concatenate([[0], np.cumsum(rows)]).astype(np.int64)
    ci = np.concatenate(cols).astype(np.int64)
    va = np.where(ci == np.repeat(np.arange(n), rows), 20.0, -1.0)
    A = P.ell_from_csr(rp, ci, va, rt=rt)
    assert A.x_staged
    r0, c0, v0 = A.to_csr_rows(0, n, staged=True)
    assert np.array_equal(r0, rp) and np.array_equal(c0, ci) and np.array_equal(v0, va)
    b = orc.rhs_splitmix(n, seed)
    s1 = P.cg_monolithic(rt, A, b, 25, P.CgOptions())
    assert not A.set_x_staged(False)
    s2 = P.cg_monolithic(rt, A, b, 25, P.CgOptions())
    assert np.array_equal(s1.residual_history, s2.residual_history) and np.array_equal(s1.x, s2.x)
    from oracle import Csr
    want_h, _, _ = orc.cg(Csr(n, rp, ci, va), b, 25)
    check_history(s1.residual_history, want_h)
    # spread columns: row i also touches column (i * 7919) % n
    ci2 = [np.union1d(c, [(i * 7919) % n]) for i, c in enumerate(cols)]
    rp2 = np.concatenate([[0], np.cumsum([len(c) for c in ci2])]).astype(np.int64)
    ci2 = np.concatenate(ci2).astype(np.int64)
    va2 = np.where(ci2 == np.repeat(np.arange(n), np.diff(rp2)), 30.0, -1.0)
    B = P.ell_from_csr(rp2, ci2, va2, rt=rt)
    assert not B.x_staged


@pytest.mark.parametrize("dims,P_", [((64, 24, 40), 4), ((32, 8, 32), 8), ((32, 4, 4), 4),
                                     ((320, 288, 12), 2), ((30, 20, 18), 3)])
def test_x_staged_slabs_multi_rank(orc, dims, P_):
    """z-slab matrices with nx % 32 == 0 are x-staged too: their staged runs
    reach into the ghost planes (global line geometry, local columns).  The
    NCCL-path phases (loopback) and the peer transport -- whose boundary
    slices stage x only after the ghost-plane flags are acquired, in one
    launch on the 320x288 planes -- must agree to the bit, and both within
    the rule of the oracle; the gather slabs (staged form dropped) too."""
    b = orc.rhs_xorshift(int(np.prod(dims)), 4)
    want_h, want_x, _ = orc.cg(orc.stencil(*dims), b, 30)
    out = {}
    for stage in (True, False):
        for transport in ("loopback", "peer"):
            G = P.EmulatedRankGroup(*dims, P_, 30, transport=transport, x_staged=stage)
            assert all(A.x_staged == stage for A in G.mats)
            G.set_rhs(b)
            G.iterate(11)
            G.iterate(19)
            hs = G.history(30)
            for h in hs:
                assert np.array_equal(h, hs[0])
            out[stage, transport] = (hs[0], G.solution())
            G.close()
            check_history(hs[0], want_h)
            assert np.all(rel_gap(out[stage, transport][1], want_x) <= 1e-10)
    for stage in (True, False):
        (h0, x0), (h1, x1) = out[stage, "loopback"], out[stage, "peer"]
        assert np.array_equal(h0, h1) and np.array_equal(x0, x1)


@pytest.mark.parametrize("where", ["mono", "mono_graph", "loopback", "peer", "tasks",
                                   "tasks_graph", "persistent"])
def test_x_update_in_k3_bit_identical(rt, orc, where):
    """From 4M rows per rank the x update (x += alpha p_old) runs in K3, which
    reads p_old anyway, instead of K2 (in the tasks variant: in the p-update
    tile kernels / dispatcher chunks instead of the x/r ones).  x feeds
    nothing inside the iteration and keeps its roundings, so histories and x
    must be bit-identical to the K2 placement (CgOptions.x_update forces
    either), on every executor and both multi-rank transports."""
    dims = (64, 40, 36)
    b = orc.rhs_xorshift(int(np.prod(dims)), 6)
    out = []
    for xk3 in ("k3", "k2"):
        if where.startswith("mono"):
            A = P.gen_stencil_matrix(*dims, rt=rt)
            res = P.cg_monolithic(rt, A, b, 35, P.CgOptions(use_graph=where == "mono_graph",
                                                            x_update=xk3))
            out.append((res.residual_history, res.x))
        elif where.startswith("tasks") or where == "persistent":
            A = P.gen_stencil_matrix(*dims, rt=rt)
            opt = P.CgOptions(tiles=5, use_graph=where == "tasks_graph",
                              persistent=where == "persistent", x_update=xk3)
            res = P.cg_tasks(rt, A, b, 35, opt)
            out.append((res.residual_history, res.x))
        else:
            G = P.EmulatedRankGroup(*dims, 3, 35, transport=where,
                                    options=P.CgOptions(iteration_marks=False, x_update=xk3))
            G.set_rhs(b)
            G.iterate(20)
            G.iterate(15)
            out.append((G.history(35)[0], G.solution()))
            G.close()
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
    want_h, want_x, _ = orc.cg(orc.stencil(*dims), b, 35)
    check_history(out[0][0], want_h)
    assert np.all(rel_gap(out[0][1], want_x) <= 1e-10)




@pytest.mark.parametrize("P_", [2, 3, 4, 8])
@pytest.mark.parametrize("T", [1, 4, 16])
def test_multi_rank_block_task_dag(orc, P_, T):
    """The block-task DAG across z-slab ranks (cg_tasks with the halo task,
    cg.cpp:166-334): every rank's tile kernels, the loopback halo, tile-order
    then rank-order alpha / beta_res -- the kernels and partial orders of the
    NCCL tasks executor -- against the oracle under the SURVEY 8(c) rule;
    every rank holds the same history, and a re-solve repeats it bit for
    bit.  x-staged slabs (nx % 32 == 0) and run-table slabs (nx = 30)."""
    for dims in ((32, 16, 24), (30, 12, 16)):
        m = orc.stencil(*dims)
        b = orc.rhs_xorshift(m.n, 5)
        want_h, want_x, _ = orc.cg(m, b, 40)
        G = P.EmulatedRankGroup(*dims, P_, 40, variant=N_TASKS,
                                options=P.CgOptions(tiles=T, iteration_marks=False))
        assert all(s.mode()["variant"] == N_TASKS and s.mode()["tiles"] == T for s in G.solvers)
        runs = []
        for _ in range(2):
            G.set_rhs(b)
            G.iterate(17)
            G.iterate(23)
            hs = G.history(40)
            for h in hs:
                assert np.array_equal(h, hs[0])
            runs.append((hs[0], G.solution()))
        G.close()
        assert np.array_equal(runs[0][0], runs[1][0]) and np.array_equal(runs[0][1], runs[1][1])
        check_history(runs[0][0], want_h)
        assert np.all(rel_gap(runs[0][1], want_x) <= 1e-10)


N_TASKS = 1  # TW_CG_TASKS


@pytest.mark.parametrize("P_", [2, 3, 4, 8])
@pytest.mark.parametrize("T", [1, 4, 16])
def test_multi_rank_persistent_dispatcher(orc, P_, T):
    """The persistent dispatcher across z-slab ranks: every rank's task table
    in ONE launch (an emulated group on one GPU; on a real node each GPU runs
    its own), the cross-rank edges being the peer protocol -- halo tasks
    storing planes into the neighbours' ghost planes and raising their
    flags, the ghost-reading SpMV tiles waiting for them, alpha / beta_res
    publishing tile-order partials and summing every rank's in rank order.
    Against the oracle under the rule; ranks agree; a re-solve (new epoch
    stamps) repeats every bit; split calls (stamps continue) too."""
    for dims in ((32, 16, 24), (30, 12, 16)):
        m = orc.stencil(*dims)
        b = orc.rhs_xorshift(m.n, 5)
        want_h, want_x, _ = orc.cg(m, b, 40)
        G = P.EmulatedRankGroup(*dims, P_, 40, variant=N_TASKS, transport="peer",
                                options=P.CgOptions(tiles=T, persistent=True, iteration_marks=False))
        assert all(s.mode()["dispatch"] == 1 for s in G.solvers)
        runs = []
        for split in ((40,), (13, 27)):
            G.set_rhs(b)
            for k in split:
                G.iterate(k)
            hs = G.history(40)
            for h in hs:
                assert np.array_equal(h, hs[0])
            runs.append((hs[0], G.solution()))
        G.close()
        assert np.array_equal(runs[0][0], runs[1][0]) and np.array_equal(runs[0][1], runs[1][1])
        check_history(runs[0][0], want_h)
        assert np.all(rel_gap(runs[0][1], want_x) <= 1e-10)


def test_cg_solve_cache_and_staged_copies(rt, orc):
    """tw_cg_solve keeps its solver per matrix between calls (same results
    call after call, a longer solve or other options rebuild it, dropping
    the staged form drops it); pageable and pinned host buffers above the
    staging threshold (8 MB) give the same bits."""
    import torch
    dims = (160, 128, 64)  # 1.3M rows: 10.5 MB vectors, above the staging threshold
    m = orc.stencil(*dims)
    A = P.ell_from_csr(m.row_ptr, m.col_idx, m.values, rt=rt)
    b = orc.rhs_xorshift(m.n, 11)
    assert b.nbytes > (8 << 20)
    want_h, want_x, _ = orc.cg(m, b, 12)
    opt = P.CgOptions(tiles=1, iteration_marks=False)
    r1 = P.cg_solve(rt, A, b, 12, opt)
    r2 = P.cg_solve(rt, A, b, 12, opt)                      # the cached solver
    bp = torch.from_numpy(b.copy()).pin_memory().numpy()
    xp = torch.empty(m.n, dtype=torch.float64).pin_memory().numpy()
    r3 = P.cg_solve(rt, A, bp, 12, opt, x_out=xp)           # pinned: direct copies
    r4 = P.cg_solve(rt, A, b, 20, opt)                      # more iterations: rebuilt
    r5 = P.cg_solve(rt, A, b, 12, P.CgOptions(tiles=4, iteration_marks=False), variant=1)
    for r in (r2, r3):
        assert np.array_equal(r.residual_history, r1.residual_history)
        assert np.array_equal(r.x, r1.x)
    assert np.array_equal(r4.residual_history[:12], r1.residual_history)
    check_history(r1.residual_history, want_h)
    check_history(r5.residual_history, want_h)
    assert np.all(rel_gap(r1.x, want_x) <= 1e-10)
    assert not A.set_x_staged(False)                         # drops the cached solver
    r6 = P.cg_solve(rt, A, b, 12, opt)
    assert np.array_equal(r6.residual_history, r1.residual_history)
    assert np.array_equal(r6.x, r1.x)


@pytest.mark.parametrize("dims,P_,T", [((32, 16, 4), 4, 1), ((48, 24, 3), 3, 1), ((48, 24, 3), 2, 2),
                                       ((32, 16, 4), 4, 3)])
def test_multi_rank_dispatcher_thin_slabs(orc, dims, P_, T):
    """One-plane slabs next to wider ones: an end slab's rows reach one plane
    fewer than a middle slab's (18 against 27 entries per row), so one launch
    holds slices of different widths -- its stages and grid are sized by the
    widest rank (found by scripts/stress_dispatcher.py: sizing them by rank
    0 overran the stages)."""
    m = orc.stencil(*dims)
    b = orc.rhs_xorshift(m.n, 5)
    want_h, want_x, _ = orc.cg(m, b, 15)
    G = P.EmulatedRankGroup(*dims, P_, 15, variant=N_TASKS, transport="peer",
                            options=P.CgOptions(tiles=T, persistent=True, iteration_marks=False))
    G.set_rhs(b)
    G.iterate(4)
    G.iterate(11)
    hs = G.history(15)
    x = G.solution()
    G.close()
    for h in hs:
        assert np.array_equal(h, hs[0])
    check_history(hs[0], want_h)
    assert np.all(rel_gap(x, want_x) <= 1e-10)


@pytest.mark.parametrize("dims,T", [((7, 1, 1), 1), ((3, 1, 12), 16), ((5, 3, 2), 2)])
def test_dispatcher_x_update_on_tiny_stages(rt, orc, dims, T):
    """Grids so small that the dispatcher's stages hold 3-operand but not
    4-operand TMA blocks: with the x update placed in the p-update chunks,
    the x/r chunks (register path) must not update x as well
    (scripts/stress_random.py found x updated twice)."""
    m = orc.stencil(*dims)
    b = orc.rhs_xorshift(m.n, 2)
    A = P.gen_stencil_matrix(*dims, rt=rt)
    for xu in ("k2", "k3"):
        res = P.cg_tasks(rt, A, b, 6, P.CgOptions(tiles=T, persistent=True, x_update=xu))
        want_h, want_x, _ = orc.cg(m, b, 6)
        check_history(res.residual_history, want_h)
        assert np.all(rel_gap(res.x, want_x) <= 1e-10), xu


@pytest.mark.parametrize("how", ["streams", "graph_chunks", "graph_marks", "timed_graph",
                                 "tasks_streams", "tasks_graph_chunks", "tasks_graph_marks",
                                 "tasks_fold_chunks", "tasks_persistent", "tasks_persistent_marks"])
def test_x_update_pairs_bit_identical(rt, orc, how):
    """Paired x updates (CgOptions.x_update="k3_pairs", the default of a
    one-rank monolithic solve from 4M rows): the first K3 of each pair of
    iterations writes p_k+1 to a second buffer and leaves x alone, the second
    applies x = (x + a_k p_k) + a_k+1 p_k+1 -- the two roundings of two single
    updates in the same order.  Histories, x, r and p (at every call
    boundary: an odd call's last iteration is a single update) must be
    bit-identical to the x update in every K3, for calls of odd and even
    lengths on every monolithic executor and on the block-task DAG's streams
    and graphs and in the persistent dispatcher (one rank: the p-update
    tiles / chunks alternate the buffers, the iteration's global reductions
    order the buffer reuse)."""
    from paper_2602_21897_b200 import _native as N
    dims = (64, 40, 36)
    n = int(np.prod(dims))
    b = orc.rhs_xorshift(n, 6)
    A = P.gen_stencil_matrix(*dims, rt=rt)
    calls = (1, 2, 3, 5, 16, 17, 4)
    total = sum(calls)
    kw = dict(streams=dict(use_graph=False),
              graph_chunks=dict(use_graph=True, iteration_marks=False),
              graph_marks=dict(use_graph=True, iteration_marks=True),
              timed_graph=dict(use_graph=True, iteration_marks=False),
              tasks_streams=dict(tiles=5, use_graph=False),
              tasks_graph_chunks=dict(tiles=7, use_graph=True, iteration_marks=False),
              tasks_graph_marks=dict(tiles=6, use_graph=True, iteration_marks=True),
              tasks_fold_chunks=dict(tiles=3, use_graph=True, iteration_marks=False),
              tasks_persistent=dict(tiles=16, persistent=True, iteration_marks=False),
              tasks_persistent_marks=dict(tiles=5, persistent=True, iteration_marks=True))[how]
    variant = N.TW_CG_TASKS if how.startswith("tasks") else N.TW_CG_MONOLITHIC
    out = {}
    for xu in ("k3", "k3_pairs", None):
        S = P.CgSolver(rt, A, total, P.CgOptions(x_update=xu, **kw), variant=variant)
        want_mode = {"k3": 1, "k3_pairs": 2, None: 0}[xu]  # auto below 4M rows: K2
        assert S.mode()["x_in_k3"] == want_mode
        if how == "timed_graph":
            S.enable_kernel_timing(True)
        if variant == N.TW_CG_TASKS:
            assert S.mode()["dispatch"] == (N.TW_DISPATCH_PERSISTENT if "persistent" in how
                                            else N.TW_DISPATCH_STREAMS)
        S.set_rhs(b)
        snaps = []
        for c in calls:
            S.iterate(c)
            S.wait()
            xp, rp, pp, _ = S.vectors()
            for ptr in (xp, rp, pp):
                h = np.empty(n, np.float64)
                N.check(N.load().tw_memcpy(rt.h, h.ctypes.data_as(N.C.c_void_p), N.C.c_void_p(ptr),
                                           h.nbytes, None))
                rt.synchronize()
                snaps.append(h)
        out[xu] = (S.history(total), snaps)
        S.close()
    for xu in ("k3_pairs", None):
        assert np.array_equal(out[xu][0], out["k3"][0]), xu
        for k, (a, c) in enumerate(zip(out[xu][1], out["k3"][1])):
            assert np.array_equal(a, c), (xu, k // 3, "xrp"[k % 3])
    want_h, want_x, _ = orc.cg(orc.stencil(*dims), b, total)
    check_history(out["k3"][0], want_h)
    assert np.all(rel_gap(out["k3"][1][-3], want_x) <= 1e-10)


@pytest.mark.parametrize("dims,xu", [((64, 40, 36), "k3_pairs"), ((64, 40, 36), None),
                                     ((128, 64, 96), None)])
@pytest.mark.parametrize("graph", [True, False])
def test_k1_programmatic_launch_bit_identical(rt, orc, dims, xu, graph):
    """The one-rank monolithic chain launches K1 programmatically after K3
    (griddepcontrol.wait before the slice's x runs; tw_cg.cpp TW_MONO_PDL);
    the per-kernel timing pass launches it plainly (events between the
    kernels).  Histories and x, r, p after every call must be bit-identical
    between the two, for chunked graphs and plain streams, paired and single
    x updates and the 786k-row grid (x-staged K1, x update in K3), and
    within the rule of the oracle."""
    from paper_2602_21897_b200 import _native as N
    n = int(np.prod(dims))
    b = orc.rhs_xorshift(n, 11)
    A = P.gen_stencil_matrix(*dims, rt=rt)
    assert A.x_staged
    calls = (1, 6, 3, 20)
    total = sum(calls)
    out = []
    for timed in (False, True):
        S = P.CgSolver(rt, A, total, P.CgOptions(use_graph=graph, iteration_marks=False,
                                                 x_update=xu), variant=N.TW_CG_MONOLITHIC)
        assert S.mode()["k1_form"] == N.TW_K1_STAGED
        if timed:
            S.enable_kernel_timing(True)
        S.set_rhs(b)
        snaps = []
        for c in calls:
            S.iterate(c)
            S.wait()
            for ptr in S.vectors()[:3]:
                h = np.empty(n, np.float64)
                N.check(N.load().tw_memcpy(rt.h, h.ctypes.data_as(N.C.c_void_p), N.C.c_void_p(ptr),
                                           h.nbytes, None))
                rt.synchronize()
                snaps.append(h)
        out.append((S.history(total), snaps))
        S.close()
    assert np.array_equal(out[0][0], out[1][0])
    for k, (a, c) in enumerate(zip(out[0][1], out[1][1])):
        assert np.array_equal(a, c), (k // 3, "xrp"[k % 3])
    want_h, want_x = orc.cg_stencil(*dims, b, total)
    check_history(out[0][0], want_h)
    assert np.all(rel_gap(out[0][1][-3], want_x) <= 1e-10)


@pytest.mark.parametrize("dims,T", [((64, 40, 36), 1), ((64, 40, 36), 2), ((64, 40, 36), 3),
                                    ((64, 40, 36), 4), ((64, 40, 36), 7), ((64, 40, 36), 16),
                                    ((128, 64, 96), 4), ((256, 256, 96), 2)])
@pytest.mark.parametrize("graph", [False, True])
def test_tasks_programmatic_chain(rt, orc, dims, T, graph):
    """TW_DISPATCH_CHAIN: the block-task DAG's tile kernels in DAG order on
    one stream, each launched programmatically (a phase's first tile waits
    for every grid before it, the others start behind it without a wait).
    Histories and x bit-identical to the stream / event executor (same tile
    kernels, same tile partials and alpha / beta_res orders) for calls of
    odd and even lengths, with and without graphs, single and paired x
    updates (the 786k-row grid), the plainly launched x/r gate of tiles of
    3M rows and more (256 x 256 x 96 in 2 tiles), and within the rule of
    the oracle."""
    from paper_2602_21897_b200 import _native as N
    n = int(np.prod(dims))
    b = orc.rhs_xorshift(n, 13)
    A = P.gen_stencil_matrix(*dims, rt=rt)
    calls = (1, 4, 3, 16)
    total = sum(calls)
    out = []
    for chain in (False, True):
        S = P.CgSolver(rt, A, total, P.CgOptions(tiles=T, use_graph=graph, iteration_marks=False,
                                                 chain=chain), variant=N.TW_CG_TASKS)
        assert S.mode()["dispatch"] == (N.TW_DISPATCH_CHAIN if chain else N.TW_DISPATCH_STREAMS)
        S.set_rhs(b)
        for c in calls:
            S.iterate(c)
        S.wait()
        out.append((S.history(total), S.solution()))
        S.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
    want_h, want_x = orc.cg_stencil_mt(*dims, b, total)
    check_history(out[1][0], want_h)
    assert np.all(rel_gap(out[1][1], want_x) <= 1e-10)


def test_tasks_programmatic_chain_marks(rt, orc):
    """Host cg_iter marks and device iteration times under the chain (all
    its work on the compute stream, where the marks are recorded): positive,
    non-decreasing marks, positive iteration times, and the automatic
    dispatch picking the chain for 4 tiles of 50k+ rows."""
    from paper_2602_21897_b200 import _native as N
    dims = (64, 48, 72)  # 221k rows: 4 tiles of 55k
    A = P.gen_stencil_matrix(*dims, rt=rt)
    b = orc.rhs_xorshift(A.n, 5)
    want_h, want_x = orc.cg_stencil(*dims, b, 30)
    s = P.CgSolver(rt, A, 30, P.CgOptions(tiles=4, auto_dispatch=True, iteration_marks=True),
                   variant=N.TW_CG_TASKS)
    assert s.mode()["dispatch"] == N.TW_DISPATCH_CHAIN
    s.set_rhs(b)
    s.iterate(12)
    s.iterate(18)
    s.wait()
    check_history(s.history(30), want_h)
    assert np.all(rel_gap(s.solution(), want_x) <= 1e-10)
    m = s.marks(30)
    assert np.all(m > 0) and np.all(np.diff(m) >= 0)
    t = s.iteration_times(30)
    assert np.all(t > 0)
    s.close()


def test_tasks_programmatic_chain_refusals(rt):
    """The chain runs the tasks variant (on one rank, over an x-staged matrix)."""
    from paper_2602_21897_b200 import _native as N
    A = P.gen_stencil_matrix(64, 8, 8, rt=rt)
    with pytest.raises(P.ConfigError):
        P.CgSolver(rt, A, 4, P.CgOptions(tiles=1, chain=True), variant=N.TW_CG_MONOLITHIC)
    with pytest.raises(P.ConfigError):
        P.CgOptions(tiles=2, chain=True, persistent=True).to_c(N.TW_CG_TASKS)


@pytest.mark.parametrize("transport", ["loopback", "peer"])
@pytest.mark.parametrize("nranks", [2, 3])
def test_x_update_pairs_across_ranks(orc, transport, nranks):
    """Paired x updates across z-slab ranks (monolithic): the halo alternates
    buffers with the x updates -- the loopback / NCCL halo exchanges the pair
    buffer's planes before the second iteration of a pair, the peer K3 of the
    first stores its edge planes into the neighbours' pair-buffer ghost
    planes (a second set of links).  Histories and x bit-identical to the x
    update in every K3 for calls of odd and even lengths, also with the
    concurrent group (single updates) interleaved, and within the rule of
    the oracle."""
    dims = (64, 40, 48)
    b = orc.rhs_xorshift(int(np.prod(dims)), 9)
    calls = (1, 4, 3, 2, 5)
    total = sum(calls)
    out = {}
    for xu in ("k3", "k3_pairs"):
        G = P.EmulatedRankGroup(*dims, nranks, total, transport=transport,
                                 options=P.CgOptions(iteration_marks=False, x_update=xu))
        assert G.solvers[0].mode()["x_in_k3"] == (2 if xu == "k3_pairs" else 1)
        G.set_rhs(b)
        xs = []
        for j, c in enumerate(calls):
            if transport == "peer" and j == 2:
                G.iterate_concurrent(c)  # single updates in one cooperative kernel
            else:
                G.iterate(c)
            xs.append(G.solution())
        hs = G.history(total)
        for h in hs:
            assert np.array_equal(h, hs[0])
        out[xu] = (hs[0], xs)
        G.close()
    assert np.array_equal(out["k3"][0], out["k3_pairs"][0])
    for a, c in zip(out["k3"][1], out["k3_pairs"][1]):
        assert np.array_equal(a, c)
    want_h, want_x, _ = orc.cg(orc.stencil(*dims), b, total)
    check_history(out["k3_pairs"][0], want_h)
    assert np.all(rel_gap(out["k3_pairs"][1][-1], want_x) <= 1e-10)


@pytest.mark.parametrize("how", ["streams", "persistent"])
@pytest.mark.parametrize("nranks", [2, 3])
def test_x_update_pairs_tasks_across_ranks(orc, how, nranks):
    """Paired x updates in the block-task DAG across z-slab ranks: the halo
    task alternates buffers with the pairs (loopback copies of the NCCL
    executor; the dispatcher's halo chunks store the pair buffer's planes
    through the second set of peer links), the p-update tiles / chunks
    alternate them as on one rank.  Bit-identical to the x update in every
    p update for calls of odd and even lengths; ranks agree; the oracle's
    rule holds."""
    dims = (32, 16, 24)
    b = orc.rhs_xorshift(int(np.prod(dims)), 11)
    calls = (3, 6, 1, 4)
    total = sum(calls)
    out = {}
    for xu in ("k3", "k3_pairs"):
        opt = P.CgOptions(tiles=4, persistent=how == "persistent", iteration_marks=False,
                          x_update=xu)
        G = P.EmulatedRankGroup(*dims, nranks, total, variant=N_TASKS, options=opt,
                                transport="peer" if how == "persistent" else "loopback")
        assert G.solvers[0].mode()["x_in_k3"] == (2 if xu == "k3_pairs" else 1)
        G.set_rhs(b)
        xs = []
        for c in calls:
            G.iterate(c)
            xs.append(G.solution())
        hs = G.history(total)
        for h in hs:
            assert np.array_equal(h, hs[0])
        out[xu] = (hs[0], xs)
        G.close()
    assert np.array_equal(out["k3"][0], out["k3_pairs"][0])
    for a, c in zip(out["k3"][1], out["k3_pairs"][1]):
        assert np.array_equal(a, c)
    want_h, want_x, _ = orc.cg(orc.stencil(*dims), b, total)
    check_history(out["k3_pairs"][0], want_h)
    assert np.all(rel_gap(out["k3_pairs"][1][-1], want_x) <= 1e-10)
