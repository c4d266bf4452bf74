"""Tasks-variant tile grids (tuning tool): streams and the chain at 2 / 3 / 4 / 6
tiles, 128^3 and 256^3, us per iteration (the side-by-side SpMV tiles' grids
must fit on the SMs together)."""
import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2602_21897_b200 as P
rt = P.Runtime(0)
stream = torch.cuda.ExternalStream(rt.compute_stream)
tag = os.path.basename(os.environ.get("TW_HPCCG_LIB", "default"))
for nx, K in ((128, 400), (256, 60)):
    A = P.gen_stencil_matrix(nx, nx, nx, rt=rt)
    b = P.rhs_xorshift(rt, A.n, 7)
    out = []
    for T in ((2, 3, 4, 6) if not os.environ.get("TILES") else tuple(int(t) for t in os.environ["TILES"].split(","))):
        for name, kw in (("streams", {}), ("chain", dict(chain=True))):
            S = P.CgSolver(rt, A, K + 5, P.CgOptions(tiles=T, iteration_marks=False, **kw), variant=1)
            best = 1e9
            for _ in range(2):
                S.set_rhs(b); S.iterate(5); S.wait()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize(); e0.record(stream); S.iterate(K); e1.record(stream); torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) / K)
            S.close()
            out.append(f"T{T} {name} {1e3*best:.1f}")
    print(tag, f"{nx}^3:", " | ".join(out), flush=True)
    del A
