"""CPU tests of the block-task DAG: the edges the
B200 build's host runtime infers from spawn_iteration's access regions
(libtw_hpccg.so, tw_task_dag_edges -- no device needed) must equal the edges
the reference's own depsys records for cg_tasks (golden vectors made by
running oracle/_ref, tests/golden/make_golden.py)."""
import numpy as np
import pytest

import paper_2602_21897_b200 as P

CASES = [((4, 4, 4), 4, 2), ((5, 4, 3), 3, 3), ((8, 8, 8), 16, 2), ((6, 5, 4), 7, 2),
         ((3, 3, 3), 1, 3)]


def plan(orc, dims, T):
    m = orc.stencil(*dims)
    r0, r1, lo, hi = orc.tile_plan(m, T)
    return m.n, [P.Tile(int(a), int(b), int(c), int(d)) for a, b, c, d in zip(r0, r1, lo, hi)]


@pytest.mark.parametrize("dims,T,its", CASES)
def test_dag_edges_equal_reference_depsys(orc, golden, dims, T, its):
    n, tiles = plan(orc, dims, T)
    got = sorted(" ".join(e) for e in P.task_dag_edges(n, tiles, its))
    want = sorted(str(e) for e in golden["dag_%dx%dx%d_T%d_it%d_edges" % (dims + (T, its))])
    assert got == want


@pytest.mark.parametrize("dims,T", [((7, 6, 5), 9), ((16, 16, 16), 64)])
def test_dag_edges_equal_live_reference(orc, ref, dims, T):
    n, tiles = plan(orc, dims, T)
    got = sorted(" ".join(e) for e in P.task_dag_edges(n, tiles, 3))
    M = ref.stencil(*dims)
    want = sorted(" ".join(e) for e in ref.cg_task_edges(M, orc.rhs_xorshift(n, 7), 3, T))
    assert got == want


def test_dag_war_edge_on_p_band(orc):
    """The WAR edge SURVEY 3.3 calls out: p_up of a tile waits for the spmv of
    every tile whose column band overlaps its rows."""
    n, tiles = plan(orc, (8, 8, 8), 8)
    edges = set(P.task_dag_edges(n, tiles, 1))
    for t, tl in enumerate(tiles):
        for u, tu in enumerate(tiles):
            overlap = not (tu.band_hi < tl.r0 or tu.band_lo >= tl.r1)
            assert ((f"spmv:0:{u}", f"p_up:0:{t}") in edges) == overlap


def test_dag_halo_task_for_ranks(orc):
    """Across ranks a halo task refreshes p's ghost planes: the next
    iteration's SpMV tiles that read a ghost plane depend on it, and it waits
    for the p_up tiles owning the boundary planes (RAW) and the SpMV tiles
    reading the old ghosts (WAR)."""
    nx, ny, nzl = 4, 4, 6
    plane = nx * ny
    n = plane * nzl
    ds = plane  # lower ghost plane present
    T = 3
    tiles = []
    for t in range(T):
        a, b = n * t // T, n * (t + 1) // T
        # band in local x coordinates: rows +- (plane + nx + 1) clipped to [0, n + 2 plane)
        lo = max(a + ds - (plane + nx + 1), 0)
        hi = min(b - 1 + ds + plane + nx + 1, n + 2 * plane - 1)
        tiles.append(P.Tile(a, b, lo, hi))
    edges = set(P.task_dag_edges(n, tiles, 2, diag_shift=ds, plane=plane, ghost_lo=True,
                                 ghost_hi=True))
    assert ("halo:1:0", "spmv:1:0") in edges and ("halo:1:0", "spmv:1:2") in edges
    assert ("p_up:0:0", "halo:1:0") in edges and ("p_up:0:2", "halo:1:0") in edges
    assert ("spmv:0:0", "halo:1:0") in edges
    # the middle tile reads no ghost plane, so it does not wait for the halo
    assert ("halo:1:0", "spmv:1:1") not in edges


def test_dag_rejects_bad_plans():
    with pytest.raises(P.ConfigError):
        P.task_dag_edges(4, [], 1)
    with pytest.raises(P.ConfigError):
        P.task_dag_edges(4, [P.Tile(0, 4, 0, 3)], 0)
