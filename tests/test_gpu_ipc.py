"""CUDA-IPC setup of the NVLink peer transport across processes.

One process per rank exports its blob (IPC handles of its flag window and p
buffer), the blobs are all-gathered over a CPU gloo group, and every rank
maps its peers' memory (tw_cg_peer_connect).  The ranks share the one B200
here, which CUDA IPC supports; no iteration runs, because kernels that wait
on one another across processes must not share a GPU -- the iteration
itself is covered by the emulated group (test_gpu_parity.py)."""
import os
import socket

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, q, xu=None):
    import torch.distributed as dist

    import paper_2602_21897_b200 as P
    from paper_2602_21897_b200 import _native as N

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rt = P.Runtime(0)
        rt.init_emulated_rank(rank, world)
        zb, ze = P.slab_partition(24, rank, world)
        A = P.gen_stencil_matrix(16, 16, 24, rt=rt, z_begin=zb, z_end=ze)
        # xu: "k3_pairs" on every rank, or "mixed" (rank 0 pairs, the others not)
        mine = "k3_pairs" if xu == "k3_pairs" or (xu == "mixed" and rank == 0) else None
        s = P.CgSolver(rt, A, 4, P.CgOptions(x_update=mine), variant=N.TW_CG_MONOLITHIC)
        blob = s.peer_export()
        assert len(blob) == P.CgSolver.PEER_BLOB_BYTES
        # [160, 168): the pair buffer's offset in the p allocation, 0 without pairs
        assert (int.from_bytes(blob[160:168], "little") != 0) == (mine == "k3_pairs")
        try:
            s.enable_peer_transport()  # allgather over gloo + cudaIpcOpenMemHandle
        except P.ContractViolation as ex:
            q.put((rank, "refused", str(ex)))
        else:
            q.put((rank, s.launches_per_iteration(), blob[144:148]))
        dist.barrier()  # peers keep their buffers alive until all have mapped
        s.close()
        rt.close()
    except Exception as ex:  # reported to the parent
        q.put((rank, "error", repr(ex)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("xu", [None, "k3_pairs", "mixed"])
@pytest.mark.parametrize("world", [2, 3])
def test_peer_ipc_export_connect(world, xu):
    """With paired x updates the blob carries the pair buffer's offset and
    the neighbours' pair-buffer ghost planes are reached through the same
    mapping; ranks that pair differently are refused at connect."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q, xu)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, lpi, tag in out:
        assert lpi != "error", tag
        if xu == "mixed":
            assert lpi == "refused" and "pairs its x updates differently" in tag
            continue
        assert lpi == (4, 0)
        assert int.from_bytes(tag, "little") == rank
