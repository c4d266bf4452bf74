"""Multi-rank (z-slab) path on CPU: world_size 2 and 3 over torch.distributed
gloo, one process per rank, 127.0.0.1 rendezvous.

Each rank takes its slab from the product's own host plan
(libtw_hpccg.so: tw_slab_partition / tw_slab_plan -- the geometry the CUDA
path generates its matrix and halo from), renumbers its rows' columns into
local x coordinates, and runs the device algorithm's data movement on the
host: halo send/recv of the boundary planes of p into the ghost planes at the
plan's offsets, SpMV split into interior rows (overlapping the halo) and
boundary rows, per-rank partial dots allgathered and summed in rank order.
The arithmetic is the oracle's (the checker).  The result must match the
single-rank reference CG within the SURVEY.md 8(c) rule, and the SpMV must
match bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import check_history, rel_gap


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, dims, iters, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import paper_2602_21897_b200 as P
    from oracle import Csr, Oracle

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    nx, ny, nz = dims
    o = Oracle()
    zb, ze = P.slab_partition(nz, rank, world)
    sp = P.slab_plan(nx, ny, nz, zb, ze)
    assert (sp.ghost_lo == 1) == (rank > 0) and (sp.ghost_hi == 1) == (rank < world - 1)
    m = o.stencil(nx, ny, nz)
    r0, r1 = sp.row_offset, sp.row_offset + sp.n_rows
    rp = m.row_ptr[r0:r1 + 1] - m.row_ptr[r0]
    ci = m.col_idx[m.row_ptr[r0]:m.row_ptr[r1]] - sp.col_offset
    va = m.values[m.row_ptr[r0]:m.row_ptr[r1]]
    assert ci.min() >= 0 and ci.max() < sp.x_len
    assert len(ci) == sp.nnz
    loc = Csr(sp.n_rows, rp, ci, va)
    n, ds, pl = sp.n_rows, sp.diag_shift, sp.plane

    def allgather_sum(v):
        t = torch.tensor([v], dtype=torch.float64)
        parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, t)
        s = 0.0
        for q in parts:  # rank order, like the device combine kernel
            s += float(q.item())
        return s

    def halo(p):
        reqs = []
        bufs = []
        if sp.ghost_lo:
            lo = torch.from_numpy(p[sp.recv_lo:sp.recv_lo + pl])
            reqs.append(dist.irecv(lo, src=rank - 1))
            reqs.append(dist.isend(torch.from_numpy(p[sp.send_lo:sp.send_lo + pl].copy()),
                                   dst=rank - 1))
            bufs.append(lo)
        if sp.ghost_hi:
            hi = torch.from_numpy(p[sp.recv_hi:sp.recv_hi + pl])
            reqs.append(dist.irecv(hi, src=rank + 1))
            reqs.append(dist.isend(torch.from_numpy(p[sp.send_hi:sp.send_hi + pl].copy()),
                                   dst=rank + 1))
            bufs.append(hi)
        for q in reqs:
            q.wait()

    b_all = o.rhs_xorshift(nx * ny * nz, 7)
    b = b_all[r0:r1].copy()
    p = np.zeros(sp.x_len)
    p[ds:ds + n] = b
    r = b.copy()
    x = np.zeros(n)
    Ap = np.zeros(n)
    rtrans = allgather_sum(o.dot(r, r))
    hist = []
    spmv_ok = True
    for it in range(iters):
        # interior rows first (no ghost reads), then halo, then boundary rows
        o.spmv(loc, p, sp.interior_r0, sp.interior_r1, y=Ap)
        halo(p)
        o.spmv(loc, p, 0, sp.interior_r0, y=Ap)
        o.spmv(loc, p, sp.interior_r1, n, y=Ap)
        if it == 0:
            # bit-exact against the global SpMV of the same p
            pg = np.zeros(nx * ny * nz)
            pg[r0:r1] = p[ds:ds + n]
            pieces = [torch.zeros(nx * ny * nz, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(pieces, torch.from_numpy(pg))
            pfull = sum(q.numpy() for q in pieces)
            spmv_ok = np.array_equal(o.spmv(m, pfull)[r0:r1], Ap)
        po = p[ds:ds + n]
        part = o.dot(po, Ap, sp.interior_r0, sp.interior_r1) + \
            (o.dot(po, Ap, 0, sp.interior_r0) + o.dot(po, Ap, sp.interior_r1, n))
        pAp = allgather_sum(part)
        alpha = rtrans / pAp
        o.waxpby(1.0, x, alpha, po, x)
        o.waxpby(1.0, r, -alpha, Ap, r)
        rr = allgather_sum(o.dot(r, r))
        beta = rr / rtrans
        rtrans = rr
        hist.append(np.sqrt(rr))
        p[ds:ds + n] = o.waxpby(1.0, r, beta, po)
    np.save(os.path.join(out_dir, f"x{rank}.npy"), x)
    np.save(os.path.join(out_dir, f"h{rank}.npy"), np.array(hist))
    np.save(os.path.join(out_dir, f"ok{rank}.npy"), np.array([spmv_ok]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,dims", [(2, (12, 10, 16)), (3, (8, 9, 13)), (2, (6, 6, 2))])
def test_slab_cg_matches_single_rank(tmp_path, orc, world, dims):
    iters = 30
    mp.spawn(_rank_main, args=(world, _free_port(), dims, iters, str(tmp_path)), nprocs=world,
             join=True)
    m = orc.stencil(*dims)
    want_h, want_x, _ = orc.cg(m, orc.rhs_xorshift(m.n, 7), iters)
    x = np.concatenate([np.load(tmp_path / f"x{r}.npy") for r in range(world)])
    for r in range(world):
        assert bool(np.load(tmp_path / f"ok{r}.npy")[0]), f"rank {r} SpMV not bit-exact"
        h = np.load(tmp_path / f"h{r}.npy")
        check_history(h, want_h)
    assert np.all(rel_gap(x, want_x) <= 1e-10)


def test_partition_covers_grid():
    import paper_2602_21897_b200 as P
    for nz, R in [(256, 8), (512, 8), (10, 3), (7, 7)]:
        spans = [P.slab_partition(nz, r, R) for r in range(R)]
        assert spans[0][0] == 0 and spans[-1][1] == nz
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        tot_rows = sum(P.slab_plan(16, 16, nz, a, b).n_rows for a, b in spans)
        tot_nnz = sum(P.slab_plan(16, 16, nz, a, b).nnz for a, b in spans)
        assert tot_rows == 16 * 16 * nz
        assert tot_nnz == (3 * 16 - 2) ** 2 * (3 * nz - 2 if nz > 1 else 1)
    with pytest.raises(P.ConfigError):
        P.slab_partition(3, 0, 4)
    with pytest.raises(P.ContractViolation):
        P.slab_plan(4, 4, 4, 3, 3)


def _rank_tasks_main(rank, world, port, dims, T, iters, seed, out_dir):
    """cg_tasks across ranks on the host: this rank's logical block-task DAG
    as the product infers it (tw_task_dag_edges, halo task included) run in
    a RANDOM topological order (seeded per rank); the collective tasks --
    halo:i, alpha:i, beta_res:i -- therefore run in whatever order the edges
    force, so the ranks only agree on them (and do not deadlock) if the edges
    order them.  Arithmetic: the oracle's, tile order then rank order."""
    import random
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import paper_2602_21897_b200 as P
    from oracle import Csr, Oracle

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    nx, ny, nz = dims
    o = Oracle()
    zb, ze = P.slab_partition(nz, rank, world)
    sp = P.slab_plan(nx, ny, nz, zb, ze)
    m = o.stencil(nx, ny, nz)
    r0, r1 = sp.row_offset, sp.row_offset + sp.n_rows
    loc = Csr(sp.n_rows, m.row_ptr[r0:r1 + 1] - m.row_ptr[r0],
              m.col_idx[m.row_ptr[r0]:m.row_ptr[r1]] - sp.col_offset,
              m.values[m.row_ptr[r0]:m.row_ptr[r1]])
    n, ds, pl = sp.n_rows, sp.diag_shift, sp.plane
    tr0, tr1, tlo, thi = o.tile_plan(loc, T)
    tiles = [P.Tile(int(a), int(b), int(c), int(d)) for a, b, c, d in zip(tr0, tr1, tlo, thi)]
    edges = P.task_dag_edges(n, tiles, iters, diag_shift=ds, plane=pl,
                             ghost_lo=bool(sp.ghost_lo), ghost_hi=bool(sp.ghost_hi))
    fams = (["halo"] if (sp.ghost_lo or sp.ghost_hi) else []) + \
        ["spmv", "dot_pAp", "alpha", "x_up", "r_up", "dot_rr", "beta_res", "p_up"]
    tasks = [f"{f}:{i}:{t}" for i in range(iters) for f in fams
             for t in (range(T) if f not in ("halo", "alpha", "beta_res") else [0])]
    preds = {k: set() for k in tasks}
    succ = {k: [] for k in tasks}
    for a, b in edges:
        preds[b].add(a)
        succ[a].append(b)
    rng = random.Random(seed * 101 + rank)
    ready = [k for k in tasks if not preds[k]]
    order = []
    while ready:
        k = ready.pop(rng.randrange(len(ready)))
        order.append(k)
        for s in succ[k]:
            preds[s].discard(k)
            if not preds[s]:
                ready.append(s)
    assert len(order) == len(tasks)

    def allgather_sum(v):
        parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.tensor([v], dtype=torch.float64))
        s = 0.0
        for q in parts:
            s += float(q.item())
        return s

    b_all = o.rhs_xorshift(nx * ny * nz, 7)
    b = b_all[r0:r1].copy()
    p = np.zeros(sp.x_len)
    p[ds:ds + n] = b
    r, x, Ap = b.copy(), np.zeros(n), np.zeros(n)
    pa, rrp = np.zeros(T), np.zeros(T)
    st = {"rtrans": allgather_sum(o.dot(r, r)), "alpha": 0.0, "beta": 0.0}
    hist = [0.0] * iters
    colls = []
    for k in order:
        f, i, t = k.split(":")
        i, t = int(i), int(t)
        a0, a1 = int(tr0[t]), int(tr1[t])
        po = p[ds:ds + n]
        if f == "halo":
            colls.append(k)
            reqs = []
            if sp.ghost_lo:
                reqs.append(dist.irecv(torch.from_numpy(p[sp.recv_lo:sp.recv_lo + pl]), src=rank - 1))
                reqs.append(dist.isend(torch.from_numpy(p[sp.send_lo:sp.send_lo + pl].copy()),
                                       dst=rank - 1))
            if sp.ghost_hi:
                reqs.append(dist.irecv(torch.from_numpy(p[sp.recv_hi:sp.recv_hi + pl]), src=rank + 1))
                reqs.append(dist.isend(torch.from_numpy(p[sp.send_hi:sp.send_hi + pl].copy()),
                                       dst=rank + 1))
            for q in reqs:
                q.wait()
        elif f == "spmv":
            o.spmv(loc, p, a0, a1, y=Ap)
        elif f == "dot_pAp":
            pa[t] = o.dot(po, Ap, a0, a1)
        elif f == "alpha":
            colls.append(k)
            s = 0.0
            for v in pa:  # tile order (cg.cpp:218-221), then rank order
                s += v
            st["alpha"] = st["rtrans"] / allgather_sum(s)
        elif f == "x_up":
            o.waxpby(1.0, x, st["alpha"], po, x, a0, a1)
        elif f == "r_up":
            o.waxpby(1.0, r, -st["alpha"], Ap, r, a0, a1)
        elif f == "dot_rr":
            rrp[t] = o.dot(r, r, a0, a1)
        elif f == "beta_res":
            colls.append(k)
            s = 0.0
            for v in rrp:
                s += v
            rr = allgather_sum(s)
            st["beta"] = rr / st["rtrans"]
            st["rtrans"] = rr
            hist[i] = np.sqrt(rr)
        elif f == "p_up":
            p[ds + a0:ds + a1] = o.waxpby(1.0, r, st["beta"], po, None, a0, a1)[a0:a1]
    np.save(os.path.join(out_dir, f"x{rank}.npy"), x)
    np.save(os.path.join(out_dir, f"h{rank}.npy"), np.array(hist))
    with open(os.path.join(out_dir, f"c{rank}.txt"), "w") as fh:
        fh.write("\n".join(colls))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,dims,T", [(2, (8, 6, 10), 3), (3, (6, 5, 12), 2), (2, (5, 4, 6), 1)])
def test_tasks_dag_across_ranks_random_order(tmp_path, orc, world, dims, T):
    """The multi-rank block-task DAG's edges are complete and order every
    rank's collectives identically: two random topological orders per rank
    give the same history and x bit for bit, within the rule of the
    single-rank reference."""
    iters = 12
    outs = []
    for seed in (1, 2):
        d = tmp_path / f"s{seed}"
        d.mkdir()
        mp.spawn(_rank_tasks_main, args=(world, _free_port(), dims, T, iters, seed, str(d)),
                 nprocs=world, join=True)
        hs = [np.load(d / f"h{r}.npy") for r in range(world)]
        for h in hs:
            assert np.array_equal(h, hs[0])
        colls = [(d / f"c{r}.txt").read_text() for r in range(world)]
        assert all(c.replace("halo", "") == colls[0].replace("halo", "") for c in colls)
        outs.append((hs[0], np.concatenate([np.load(d / f"x{r}.npy") for r in range(world)])))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    m = orc.stencil(*dims)
    want_h, want_x, _ = orc.cg(m, orc.rhs_xorshift(m.n, 7), iters)
    check_history(outs[0][0], want_h)
    assert np.all(rel_gap(outs[0][1], want_x) <= 1e-10)
