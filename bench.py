#!/usr/bin/env python
"""HPCCG CG benchmark on B200 (BASELINE.json metric: CG GFLOP/s and iters/s,
fraction of the HBM roofline, beside the reference CPU path).

A step is one CG iteration (K1 spmv_pAp + K2 update_xr + K3 update_p) on the
configuration the metric is quoted on: a 256^3 grid per GPU, weak scaling
over z-slabs (global 256 x 256 x 256N), b = xorshift seed 7
(acceptance.cpp:48-58), x0 = 0.  The working set (6.9 GB per iteration) is
far larger than L2, so no flush is needed between iterations.

  python bench.py [--gpus N --steps K --warmup W]           # our arm
  python bench.py --impl reference ...                      # reference CPU arm
  torchrun --nproc-per-node N bench.py --gpus N ...         # N GPUs, one rank each

Prints ONE JSON line (rank 0).  Algorithmic work per iteration:
FLOPs = 2 nnz + 10 n; bytes = 12 nnz + 88 n; K1 alone: 12 nnz + 16 n.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}
HBM_SPEC_GBS = 8000.0  # B200 HBM3e data-sheet bandwidth (reported beside the measured peak)
X_UPDATE_IN = {0: "K2", 1: "K3", 2: "K3 pairs"}  # tw_cg_mode_t.x_in_k3


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--nx", type=int, default=256)
    ap.add_argument("--ny", type=int, default=256)
    ap.add_argument("--nz", type=int, default=256, help="planes per GPU (weak scaling)")
    ap.add_argument("--strong", action="store_true", help="nz is the GLOBAL plane count")
    ap.add_argument("--variant", choices=["mono", "tasks"], default="mono")
    ap.add_argument("--tiles", type=int, default=4)
    ap.add_argument("--dispatch", choices=["auto", "streams", "persistent", "chain"], default="auto",
                    help="tasks variant: one launch per task (streams / graphs), the persistent "
                         "device-side dispatcher (across ranks over the NVLink peer transport) or "
                         "the programmatic chain (one rank); "
                         "auto = the library's choice on one rank, persistent from 8 tiles per "
                         "GPU across ranks")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch kernels one by one instead of replaying a captured CUDA graph")
    ap.add_argument("--e2e-runs", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--transport", choices=["auto", "nccl", "peer"], default="auto",
                    help="multi-rank data path: NVLink peer stores fused into the kernels "
                         "(CUDA IPC; auto = peer for the monolithic variant, validated "
                         "against the NCCL path before timing) or NCCL halo + allgathers")
    ap.add_argument("--comm", action="store_true",
                    help="attach an NCCL communicator even at N=1 (exercises the multi-GPU path)")
    ap.add_argument("--cpu-sample-nz", type=int, default=0,
                    help="planes of the CPU sample (0 = the full per-GPU workload)")
    ap.add_argument("--cpu-sample-iters", type=int, default=40)
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the extra single-GPU configurations (C2 128^3 monolithic vs "
                         "block-task DAG, the C5 granularity share, C4 512^3, the CSR drop-in)")
    return ap.parse_args()


def baseline_metric() -> str:
    """BASELINE.json's metric, verbatim (the line reports that metric)."""
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as f:
            return json.load(f)["metric"]
    except Exception:
        return "CG GFLOP/s and iters/s at 1/2/4/8 B200; % of HBM roofline; vs host-CPU ref"


def l2_note(args) -> str:
    n, nnz = work(args.nx, args.ny, 0, args.nz, args.nz)
    gb = (12 * nnz + 88 * n) / 1e9
    where = "larger than" if gb > 0.126 else "SMALLER than"
    return f"inputs {where} L2 ({gb:.3g} GB/iteration per GPU vs 126 MB); no flush"


def workload_config(args, world: int) -> dict:
    """The `config` both arms report (BASELINE.json configs[2]/[3])."""
    nz = args.nz if args.strong else args.nz * world
    return {"workload": (f"HPCCG {args.nx}x{args.ny}x{args.nz} " +
                         ("global strong scaling" if args.strong else
                          "per GPU weak scaling (z-slab)")),
            "global_grid": [args.nx, args.ny, nz],
            "l2": l2_note(args),
            "parallelism": f"z-slab x{world}"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return PEAKS_FALLBACK["hbm_gbs"], "fallback"


def read_bandwidth(torch, device) -> float:
    """Context for roofline.frac: a read-only stream (torch's sum over a
    4.3 GB f64 tensor, best of 5, CUDA events).  The measured copy peak
    moves as many bytes in as out; K1 is 98 % reads, so it can exceed the
    copy figure but not this one."""
    x = torch.ones(1 << 29, dtype=torch.float64, device=device)
    best = float("inf")
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x.sum()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del x
    return (8 << 29) / (best / 1e3) / 1e9


def work(nx, ny, zb, ze, nz):
    """(n, nnz) owned by the slab [zb, ze) of an nx*ny*nz grid."""
    sx = 1 if nx == 1 else 3 * nx - 2
    sy = 1 if ny == 1 else 3 * ny - 2
    zspan = sum(1 + (z > 0) + (z + 1 < nz) for z in range(zb, ze))
    return nx * ny * (ze - zb), sx * sy * zspan


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device: int, period_s: float = 0.005):
        self.samples, self.reasons = [], set()
        self.ok = False
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _sample(self):
        nv = self.nv
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
            mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in self.REASONS.items():
                if mask & bit and bit != 0x1:
                    self.reasons.add(name)
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._sample()  # at least one sample at the end of the region, whatever the thread got
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        return dist, rank, world, local
    return None, 0, 1, 0


def barrier(dist):
    if dist is not None:
        dist.barrier()


def max_over_ranks(dist, v: float) -> float:
    if dist is None:
        return v
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def min_over_ranks(dist, v: float) -> float:
    if dist is None:
        return v
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return float(t.item())


def sum_over_ranks(dist, v: float) -> float:
    if dist is None:
        return v
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def load_traffic(kernel: str = "k1"):
    """ncu dram bytes per launch of K1 / K2 / K3 from the committed profile
    summaries (profiles/k?_traffic.json, one ncu --set full capture), if any."""
    p = os.path.join(ROOT, "profiles", f"{kernel}_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d
    except Exception:
        return None


# ------------------------------------------------------------ CPU baseline

def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_reference_sample(nx, ny, nz_sample, iters, threads):
    """The reference's own CPU paths (oracle/_ref, compiled from its sources)
    on a bounded z-slab sample of the workload, BASELINE.md section 4:
      (i)   cg_reference (cg.cpp:372-395) on 1 core;
      (ii)  cg_tasks on the threaded substrate, real_seconds_per_unit = 0,
            tiles = nproc;
      (iii) the same with tiles = 8 x nproc (the headline CPU figure).
    The cg_tasks legs are timed by the reference's own cg_iter marks after
    one warm-up iteration (scenario.cpp:116-124); cg_reference by the wall
    clock around the call (its setup_state included)."""
    from oracle import Oracle, Reference
    R = Reference()
    o = Oracle()
    M = R.stencil(nx, ny, nz_sample)
    b = o.rhs_xorshift(M.n, 7)
    flops_it = 2 * M.nnz + 10 * M.n
    legs = []
    k_ref = max(2, iters // 8)
    t0 = time.perf_counter()
    R.cg_reference(M, b, k_ref)
    secs = time.perf_counter() - t0
    legs.append({"leg": "cg_reference, 1 core", "cores": 1, "tiles": 1, "iterations": k_ref,
                 "value": flops_it * k_ref / secs / 1e9, "iters_per_s": k_ref / secs,
                 "secs": secs})
    for tiles in (min(threads, M.n), min(8 * threads, M.n)):
        _, _, _, marks = R.cg_tasks_marks(M, b, 1 + iters, tiles=tiles, workers=threads,
                                          real_threads=True)
        secs = float(marks[iters] - marks[0])
        legs.append({"leg": f"cg_tasks real threads, tiles={tiles}", "cores": threads,
                     "tiles": tiles, "iterations": iters, "value": flops_it * iters / secs / 1e9,
                     "iters_per_s": iters / secs, "secs": secs})
    head = legs[-1]
    return {"value": head["value"], "unit": "GFLOP/s", "cores": threads, "kind": "reference",
            "iters_per_s": head["iters_per_s"], "cpu_model": cpu_model(),
            "sample": f"reference cg_tasks (oracle/_ref, real threads, tiles={head['tiles']}) on "
                      f"a {nx}x{ny}x{nz_sample} grid (the per-GPU workload when nz matches), "
                      f"{iters} CG iterations after 1 warm-up, {head['secs']:.2f} s wall",
            "legs": legs}


def run_reference_arm(args, dist, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    from oracle import Oracle, Reference
    R = Reference()
    o = Oracle()
    nzs = args.cpu_sample_nz or args.nz
    M = R.stencil(args.nx, args.ny, nzs)
    b = o.rhs_xorshift(M.n, 7)
    tiles = min(8 * threads, M.n)
    # W warm-up + K timed iterations in one cg_tasks run; the K steps are
    # timed by the reference's own cg_iter marks (scenario.cpp:116-124):
    # mark[W+K-1] - mark[W-1] (from the runtime start when W = 0)
    W, K = args.warmup, args.steps
    _, _, _, marks = R.cg_tasks_marks(M, b, W + K, tiles=tiles, workers=threads,
                                      real_threads=True)
    secs = float(marks[W + K - 1] - (marks[W - 1] if W > 0 else 0.0))
    flops = (2 * M.nnz + 10 * M.n) * args.steps
    v = flops / secs / 1e9
    line = {
        "impl": "reference", "metric": baseline_metric(), "value": v,
        "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (xorshift64 seed 7 rhs)",
        "iters_per_s": args.steps / secs,
        "config": {**workload_config(args, world),
                   "variant": "cg_tasks (the reference, on the host cores)",
                   "reference_step": f"one CG iteration on the {args.nx}x{args.ny}x{nzs} grid"},
        "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": threads, "kind": "reference",
                         "sample": f"cg_tasks real threads tiles={tiles} on {args.nx}x{args.ny}x{nzs}, "
                                   f"{args.steps} iterations after {args.warmup} warm-up, "
                                   f"timed by the reference's cg_iter marks"},
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm

def time_iterations(torch, S, b, K, W, stream):
    """W untimed iterations from x0 = 0, then K timed by CUDA events on the
    solver's launch stream; returns (ms per iteration, history).  One
    untimed pass of the same shape first, so the graphs / dispatcher tables
    of these call lengths are built (and cached) outside the timed region."""
    S.set_rhs(b)
    if W:
        S.iterate(W)
    S.iterate(K)
    S.wait()
    S.set_rhs(b)
    if W:
        S.iterate(W)
    S.wait()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    S.iterate(K)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K, S.history(W + K)


def dispatch_name(N, m) -> str:
    """The executor a solver runs (tw_cg_mode)."""
    if m["dispatch"] == N.TW_DISPATCH_PERSISTENT:
        return "persistent"
    chain = m["dispatch"] == N.TW_DISPATCH_CHAIN
    return ("chain " if chain else "") + ("graph" if m["use_graph"] else "streams")


def extra_configs(torch, P, N, rt, A, b, stream, peak):
    """Single-GPU figures of BASELINE configs beside the headline (rank 0,
    N = 1): the reference-API drop-in at the headline size, C2 (128^3
    monolithic vs block-task DAG), C5's per-GPU share (256^3, 1-64 tiles per
    GPU = 8-512 blocks over 8 GPUs) and C4's 1-GPU point (512^3)."""
    out = {}
    W = 5

    def opts(**kw):
        return P.CgOptions(iteration_marks=False, **kw)

    def solve_rate(Am, bm, K, variant, opt):
        S = P.CgSolver(rt, Am, W + K, opt, variant=variant)
        ms, hist = time_iterations(torch, S, bm, K, W, stream)
        m = S.mode()
        S.close()
        assert np.all(np.isfinite(hist)) and hist[-1] < hist[0]
        return ms, m, hist

    def gflops(Am, ms):
        return (2 * Am.nnz() + 10 * Am.n) / (ms / 1e3) / 1e9

    # ---- the reference-API drop-in: a host CsrMatrix (here the device
    # matrix's own export, i.e. gen_stencil_matrix's CSR) -> tw_ell_from_csr
    # (validated, uploaded, converted; x-staged through the run table) ->
    # tw_cg_solve with host b in and host history + x out, every call
    rp, ci, va = A.to_csr()
    t0 = time.perf_counter()
    Ac = P.ell_from_csr(rp, ci, va, rt=rt)
    rt.synchronize()
    setup_s = time.perf_counter() - t0
    del rp, ci, va
    bh = np.empty(A.n)
    import ctypes
    N.check(N.load().tw_memcpy(rt.h, bh.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(b.ptr),
                               8 * A.n, None))
    rt.synchronize()
    K = 100
    xh = np.empty(A.n)
    best, res = float("inf"), None
    for _ in range(3):
        t0 = time.perf_counter()
        res = P.cg_solve(rt, Ac, bh, K, opts(tiles=1), N.TW_CG_MONOLITHIC, x_out=xh)
        best = min(best, time.perf_counter() - t0)
    ref = P.cg_solve(rt, A, bh, K, opts(tiles=1), N.TW_CG_MONOLITHIC)
    Sc = P.CgSolver(rt, Ac, 1, opts(tiles=1), variant=N.TW_CG_MONOLITHIC)
    mc = Sc.mode()
    Sc.close()
    flops = (2 * A.nnz() + 10 * A.n) * K
    out["e2e_csr_drop_in"] = {
        "value": flops / best / 1e9, "unit": "GFLOP/s", "iterations_per_call": K,
        "h2d_bytes_per_step": 8 * A.n / K, "d2h_bytes_per_step": (8 * A.n + 8 * K) / K,
        "setup_s": setup_s, "k1": mc["k1_kernel"],
        "bit_identical_to_device_generated": bool(
            np.array_equal(res.residual_history, ref.residual_history)
            and np.array_equal(res.x, ref.x)),
        "api": "tw_ell_from_csr(host CsrMatrix arrays) once (setup_s: validation, upload, "
               "sliced ELL + run table), then per call tw_cg_solve(host b) -> host history + x"}
    del Ac

    # ---- K0: gen_stencil_matrix on the device at the headline size (one-time
    # setup: widths, slice-offset scan, the 128-bit fill of values, int32 and
    # x-staged columns), host wall clock around the whole call
    # (best of two; the first call right after the drop-in's device frees
    # once took 0.39 s against 8-36 ms in scripts/k0_probe.py's situations,
    # so both are reported: k0_gen_stencil_first_ms)
    k0 = []
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Ak = P.gen_stencil_matrix(A.info.nx, A.info.ny, A.info.nz, rt=rt)
        k0.append((time.perf_counter() - t0) * 1e3)
        del Ak
    out["k0_gen_stencil_ms"] = min(k0)
    out["k0_gen_stencil_first_ms"] = k0[0]

    # ---- C2: 128^3 on one GPU, monolithic vs the block-task DAG
    A2 = P.gen_stencil_matrix(128, 128, 128, rt=rt)
    b2 = P.rhs_xorshift(rt, A2.n, 7)
    K2 = 800
    rows = {}
    mono = None
    for name, variant, opt in (
            ("mono_graph", N.TW_CG_MONOLITHIC, opts(tiles=1, use_graph=True)),
            ("mono_streams", N.TW_CG_MONOLITHIC, opts(tiles=1)),
            ("tasks_T4_graph", N.TW_CG_TASKS, opts(tiles=4, use_graph=True)),
            ("tasks_T4_auto", N.TW_CG_TASKS, opts(tiles=4, auto_dispatch=True)),
            ("tasks_T16_auto", N.TW_CG_TASKS, opts(tiles=16, auto_dispatch=True)),
            ("tasks_T64_persistent", N.TW_CG_TASKS, opts(tiles=64, persistent=True))):
        ms, m, _ = solve_rate(A2, b2, K2, variant, opt)
        mono = ms if mono is None else mono
        rows[name] = {"ms_per_iter": ms, "gflops": gflops(A2, ms), "vs_mono_graph": ms / mono,
                      "dispatch": dispatch_name(N, m)}
    out["c2_128_mono_vs_tasks"] = rows
    del A2, b2

    # ---- C5's per-GPU share: 256^3 per GPU, 8-512 blocks over 8 GPUs =
    # 1-64 tiles per GPU (the library's automatic dispatch choice)
    rows = {}
    for T in (1, 2, 4, 8, 16, 32, 64):
        variant = N.TW_CG_MONOLITHIC if T == 1 else N.TW_CG_TASKS
        ms, m, _ = solve_rate(A, b, 100, variant,
                              opts(tiles=T, use_graph=T == 1, auto_dispatch=T > 1))
        rows[f"T{T}"] = {"blocks_over_8_gpus": 8 * T, "ms_per_iter": ms, "gflops": gflops(A, ms),
                         "dispatch": dispatch_name(N, m)}
    out["c5_256_per_gpu_share"] = rows

    # ---- C4's 1-GPU point: 512^3 (43 GB of sliced ELL), the headline path
    A4 = P.gen_stencil_matrix(512, 512, 512, rt=rt)
    b4 = P.rhs_xorshift(rt, A4.n, 7)
    ms, m, _ = solve_rate(A4, b4, 20, N.TW_CG_MONOLITHIC, opts(tiles=1, use_graph=True))
    by = 12 * A4.nnz() + 88 * A4.n
    out["c4_512_1gpu"] = {"ms_per_iter": ms, "gflops": gflops(A4, ms),
                          "iters_per_s": 1e3 / ms, "roofline_frac": by / (ms / 1e3) / 1e9 / peak,
                          "k1": m["k1_kernel"]}
    del A4, b4
    return out


def run_ours(args, dist, rank, world, local):
    import torch

    import paper_2602_21897_b200 as P
    from paper_2602_21897_b200 import _native as N

    nx, ny = args.nx, args.ny
    if args.strong:
        nz = args.nz
        zb, ze = nz * rank // world, nz * (rank + 1) // world
    else:
        nz = args.nz * world
        zb, ze = args.nz * rank, args.nz * (rank + 1)
    rt = P.Runtime(local)
    if world > 1:
        obj = [P.Runtime.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        rt.init_comm(rank, world, obj[0])
    elif args.comm:
        rt.init_comm(0, 1, P.Runtime.comm_unique_id())
    A = P.gen_stencil_matrix(nx, ny, nz, rt=rt, z_begin=zb, z_end=ze)
    n, nnz = A.n, A.nnz()
    assert (n, nnz) == work(nx, ny, zb, ze, nz)
    flops_it = 2 * nnz + 10 * n
    bytes_it = 12 * nnz + 88 * n
    k1_bytes = 12 * nnz + 16 * n
    b = P.rhs_xorshift(rt, n, 7, first=A.info.row_offset)
    variant = 0 if args.variant == "mono" else 1
    K, W = args.steps, args.warmup
    # Long runs are split into repetitions of at most REP timed iterations,
    # each restarting from x0 = 0 after its own W warm-up iterations (the
    # paper's repetition methodology): an unrestarted CG
    # residual underflows to 0/0 after ~1300 iterations at 256^3.
    REP = 250
    reps = [min(REP, K - i) for i in range(0, K, REP)] or [0]
    KR = reps[0]
    multi = world > 1 or args.comm
    persistent = variant == 1 and (args.dispatch == "persistent" or
                                   (args.dispatch == "auto" and multi and args.tiles >= 8))
    use_graph = not args.no_graph and not persistent
    if args.dispatch == "chain" and (variant != 1 or multi):
        raise SystemExit("--dispatch chain runs the tasks variant on one rank")
    opt = P.CgOptions(tiles=args.tiles, use_graph=use_graph, iteration_marks=False,
                      persistent=persistent, chain=args.dispatch == "chain",
                      auto_dispatch=variant == 1 and args.dispatch == "auto" and not multi)
    S = P.CgSolver(rt, A, W + KR, opt, variant=variant)
    want_peer = multi and (args.transport == "peer" or
                           (args.transport == "auto" and (variant == 0 or persistent)))
    if want_peer and variant != 0 and not persistent:
        raise SystemExit("--transport peer runs the monolithic variant or the persistent dispatcher")
    transport = ("peer" if want_peer else "nccl") if multi else None
    # the NCCL fallback of a persistent run: the tasks executor on streams
    opt_nccl = P.CgOptions(tiles=args.tiles, use_graph=not args.no_graph, iteration_marks=False)
    if want_peer:
        # CUDA-IPC setup, collective and failure-tolerant: every rank takes
        # part in the allgather even if its export failed, and all fall back
        # together if any rank could not connect
        note = ""
        try:
            blob = S.peer_export()
        except Exception as ex:
            blob, note = None, f"export: {ex}"
        if world > 1:
            blobs = [None] * world
            dist.all_gather_object(blobs, blob)
        else:
            blobs = [blob]
        ok = 1.0 if all(x is not None for x in blobs) else 0.0
        if ok:
            try:
                S.peer_connect(blobs)
            except Exception as ex:
                ok, note = 0.0, f"connect: {ex}"
        if min_over_ranks(dist, ok) >= 1.0:
            # transport check: every rank's store must become visible in
            # every window within 2 s (a bounded wait that reports, never traps)
            S.peer_ping_send()
            barrier(dist)
            if not S.peer_ping_check(2000):
                ok, note = 0.0, "ping: a peer's store never became visible"
        if min_over_ranks(dist, ok) < 1.0:
            if args.transport == "peer":
                raise SystemExit(f"peer transport setup failed ({note or 'on another rank'})")
            S.close()
            S = P.CgSolver(rt, A, W + KR, opt_nccl if persistent else opt, variant=variant)
            want_peer, persistent = False, False
            transport = f"nccl (peer setup failed: {note or 'on another rank'})"
    if want_peer:
        # validation before timing, against the NCCL path: the monolithic
        # peer path sums the same partials in the same order, so its history
        # must be identical; the persistent dispatcher's tile partials are
        # chunk-order sums, so its history must agree within 1e-10 relative
        kv = min(20, W + KR)
        S0 = P.CgSolver(rt, A, kv, opt_nccl if persistent else
                        P.CgOptions(use_graph=False, iteration_marks=False), variant=variant)
        S0.set_rhs(b)
        S0.iterate(kv)
        h0 = S0.history(kv)
        S0.close()
        S.set_rhs(b)
        S.iterate(kv)
        h1 = S.history(kv)
        ok = float(np.all(np.abs(h1 - h0) <= 1e-10 * np.abs(h0)) if persistent else
                   np.array_equal(h1, h0))
        if min_over_ranks(dist, ok) < 1.0:
            if args.transport == "peer":
                raise SystemExit("peer transport disagrees with the NCCL path")
            S.close()  # auto: fall back to the NCCL transport, and say so
            S = P.CgSolver(rt, A, W + KR, opt_nccl if persistent else opt, variant=variant)
            persistent = False
            transport = "nccl (peer validation failed)"
    kern_timing = variant == 0
    stream = torch.cuda.ExternalStream(rt.compute_stream, device=torch.device("cuda", local))
    if use_graph:
        # untimed: capture (and cache) the graphs the timed passes replay --
        # the one-iteration graph of the headline pass and the KR-iteration
        # graph that carries the per-kernel timing events
        S.set_rhs(b)
        S.iterate(1)
        S.set_rhs(b)
        if kern_timing:
            S.enable_kernel_timing(True)
        S.iterate(KR)
        S.wait()
        if kern_timing:
            S.enable_kernel_timing(False)

    def timed_rep(kr, timing):
        S.set_rhs(b)
        S.iterate(W)
        S.wait()
        if timing:
            S.enable_kernel_timing(True)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier(dist)
        torch.cuda.synchronize()
        e0.record(stream)
        S.iterate(kr)
        e1.record(stream)
        rt.synchronize()  # the long wait in a ctypes call (GIL released: the clock sampler runs)
        torch.cuda.synchronize()
        barrier(dist)
        kt = S.kernel_times() if timing else None
        if timing:
            S.enable_kernel_timing(False)
        hist = S.history(W + kr)
        # finite and decaying (CG minimises the A-norm of the error, so the
        # residual 2-norm need not fall at every single iteration)
        assert np.all(np.isfinite(hist)) and hist[-1] < hist[0]
        return e0.elapsed_time(e1), kt, hist

    def timed_run():
        # the headline: K iterations with no instrumentation inside (per-kernel
        # events in the graph cost ~1 % of the step, so they get their own pass)
        ms, hist = 0.0, None
        with ClockSampler(local) as clk:
            for kr in reps:
                m, _, hist = timed_rep(kr, False)
                ms += m
        return ms, clk.summary(), hist

    ms, clocks, hist = timed_run()
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    rejected = []
    if set(clocks["reasons"]) & bad:
        # rejected (throttled): kept in the line, and re-measured once
        rejected.append({"ms_per_step": ms / K, "clocks": clocks})
        ms, clocks, hist = timed_run()
    # the kernel-timing pass: KR iterations with K1 / K2 / K3 events recorded
    # around every kernel on its launch stream (roofline.achieved)
    kt_pass_ms, kt = None, None
    if kern_timing:
        kt_pass_ms, kt, _ = timed_rep(KR, True)
    ms_max = max_over_ranks(dist, ms)
    kernels_it, colls_it = S.launches_per_iteration()
    mode = S.mode()  # what the solver executes (tw_cg_mode)
    total_flops = sum_over_ranks(dist, float(flops_it))
    total_bytes = sum_over_ranks(dist, float(bytes_it))
    gflops = total_flops * K / (ms_max / 1e3) / 1e9
    its = K / (ms_max / 1e3)
    peak, peak_kind = peaks()

    roofline = None
    if kt is not None:
        k1_ms, k2_ms, k3_ms, nt = kt
        k1_avg = k1_ms / nt
        ach = k1_bytes / (k1_avg / 1e3) / 1e9
        k3_launches = nt
        wl = f"{nx}x{ny}x{args.nz}"

        # stencil matrices and z-slabs with nx % 32 == 0 carry the x-staged
        # form: K1 then reads 16-bit column indices (10 B per nonzero instead
        # of SURVEY 8(d)'s 12) and its operands from per-slice x windows staged
        # by the same TMA transaction; `achieved` stays on SURVEY's
        # algorithmic bytes, the format's own bytes are reported beside it
        staged = mode["k1_form"] in (N.TW_K1_STAGED, N.TW_K1_STAGED_TABLE)
        k1_format_bytes = (10 * nnz + 16 * n) if staged else k1_bytes
        slab = world > 1 or args.comm
        kname = (f"spmv_tma_staged_kernel<SPLIT={int(slab and transport == 'peer')},"
                 f"KEEP={mode['k1_l2_keep']}> (K1: TMA-staged matrix + x windows, 16-bit columns, p.Ap"
                 + ("; z-slab: interior rows, then the ghost-reading boundary rows)" if slab else ")")
                 if staged else "spmv_tma_kernel<true> (K1: TMA-staged SpMV + p.Ap)")

        def traffic_of(k):
            tr = load_traffic(k)
            ok = tr and tr.get("workload") == wl and world == 1
            if ok and k == "k1":  # the capture must be of the kernel this run used
                ok = ("staged" in tr.get("kernel", "")) == staged
            return tr.get("dram_bytes_per_launch") if ok else None

        traffic = traffic_of("k1")
        # the library moves the x update (x += alpha p_old) from K2 into K3
        # from 4M rows per rank (CgOptions.x_update): K2 then streams 24 n
        # bytes and K3 40 n, 8 n less per iteration; on one rank the K3s of
        # each pair of iterations share one x pass (x_in_k3 == 2): 24 n and
        # 48 n, 36 n per K3 on average, 12 n less than the x update in K2
        xk3 = mode["x_in_k3"]
        k2_alg, k3_alg = {0: (48 * n, 24 * n), 1: (24 * n, 40 * n), 2: (24 * n, 36 * n)}[xk3]
        roofline = {"bound": "hbm", "kernel": kname,
                    "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                    "traffic": traffic, "algorithmic_bytes": k1_bytes,
                    "format_bytes": k1_format_bytes,
                    "achieved_format": k1_format_bytes / (k1_avg / 1e3) / 1e9,
                    "frac_format": k1_format_bytes / (k1_avg / 1e3) / 1e9 / peak,
                    "avg_launch_ms": k1_avg, "peak_source": f"{peak_kind} hbm_gbs",
                    "share_of_step": k1_ms / kt_pass_ms,
                    "kernel_timing": (f"separate timed pass of {nt} iterations with events around "
                                      f"each kernel: {kt_pass_ms / nt:.4f} ms/iteration there, "
                                      f"{ms_max / K:.4f} in the event-free headline"),
                    "x_update_in": X_UPDATE_IN[xk3],
                    "k2_update_xr_gbs": k2_alg / (k2_ms / nt / 1e3) / 1e9,
                    "k3_update_p_gbs": k3_alg / (k3_ms / k3_launches / 1e3) / 1e9,
                    "k3_launches": k3_launches,
                    "k2_traffic": traffic_of("k2"), "k2_algorithmic_bytes": k2_alg,
                    "k3_traffic": traffic_of("k3"), "k3_algorithmic_bytes": k3_alg}
        if world == 1:
            rb = read_bandwidth(torch, torch.device("cuda", local))
            roofline["read_stream_gbs"] = rb
            roofline["frac_of_read_stream"] = k1_format_bytes / (k1_avg / 1e3) / 1e9 / rb
    iter_gbs = total_bytes / (ms_max / 1e3 / K) / 1e9
    roofline_iter = {"bound": "hbm", "achieved": iter_gbs, "peak": peak * world, "unit": "GB/s",
                     "frac": iter_gbs / (peak * world), "algorithmic_bytes_per_iter": total_bytes}
    if roofline and roofline.get("format_bytes") != k1_bytes:
        fb = (bytes_it - k1_bytes + roofline["format_bytes"]
              - {"K2": 0, "K3": 8 * n, "K3 pairs": 12 * n}[roofline.get("x_update_in")]) * world
        roofline_iter["format_bytes_per_iter"] = fb
        roofline_iter["achieved_format"] = fb / (ms_max / 1e3 / K) / 1e9
        roofline_iter["frac_format"] = roofline_iter["achieved_format"] / (peak * world)
    # next to the measured copy bandwidth, the HBM3e spec figure
    roofline_iter["spec_gbs"] = HBM_SPEC_GBS * world
    roofline_iter["frac_of_spec"] = iter_gbs / (HBM_SPEC_GBS * world)
    if "achieved_format" in roofline_iter:
        roofline_iter["frac_format_of_spec"] = roofline_iter["achieved_format"] / (HBM_SPEC_GBS * world)

    # ---- e2e: through the public API with host buffers (pinned b in, history + x out)
    b_host = torch.empty(n, dtype=torch.float64).pin_memory()
    bh = b_host.numpy()
    torch.cuda.synchronize()
    import ctypes
    N.check(N.load().tw_memcpy(rt.h, ctypes.c_void_p(b_host.data_ptr()), ctypes.c_void_p(b.ptr),
                               8 * n, None))
    rt.synchronize()
    x_host = torch.empty(n, dtype=torch.float64).pin_memory()
    e2e_times = []
    for _ in range(max(args.e2e_runs, 1)):
        barrier(dist)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = None
        for kr in reps:
            S.set_rhs(bh)                   # H2D of b (pinned)
            S.iterate(kr)
            h = S.history(kr)               # D2H of the residual history
            N.check(N.load().tw_cg_solution(S.h, ctypes.cast(x_host.data_ptr(),
                                                                 ctypes.POINTER(ctypes.c_double))))
        t1 = time.perf_counter()
        barrier(dist)
        e2e_times.append(max_over_ranks(dist, t1 - t0))
        assert np.all(np.isfinite(h))
    e2e_t = min(e2e_times)
    e2e = {"value": total_flops * K / e2e_t / 1e9, "unit": "GFLOP/s",
           "h2d_bytes_per_step": 8 * n * len(reps) / K,
           "d2h_bytes_per_step": (8 * n * len(reps) + 8 * K) / K,
           "iters_per_s": K / e2e_t,
           "api": "CgSolver.set_rhs(host b) + iterate(K) + history + solution (C ABI tw_cg_*)"}

    extras = None
    if rank == 0 and world == 1 and not args.no_extras and not args.strong:
        extras = extra_configs(torch, P, N, rt, A, b, stream, peak)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_sample(nx, ny, min(args.cpu_sample_nz or args.nz, nz),
                                       args.cpu_sample_iters, os.cpu_count() or 1)
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "unit": "GFLOP/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {type(ex).__name__}: {ex}"}

    if rank == 0:
        line = {
            "metric": baseline_metric(), "value": gflops, "unit": "GFLOP/s",
            "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms_max / K,
            "higher_is_better": True, "scaling": "strong" if args.strong else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: gen_stencil_matrix on device, b = xorshift64 seed 7, x0 = 0",
            "iters_per_s": its,
            "config": {**workload_config(args, world), "variant": args.variant,
                       "tiles": 1 if variant == 0 else args.tiles, "cuda_graph": use_graph,
                       "dispatch": {N.TW_DISPATCH_PERSISTENT: "persistent",
                                    N.TW_DISPATCH_CHAIN: "chain"}.get(mode["dispatch"], "streams"),
                       "rows_per_gpu": n, "nnz_per_gpu": nnz,
                       "nccl_comm": world > 1 or args.comm,
                       "transport": transport,
                       "k1": mode["k1_kernel"], "x_update_in": X_UPDATE_IN[mode["x_in_k3"]]},
            "roofline": roofline, "roofline_iteration": roofline_iter,
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            # the persistent dispatcher runs every iteration of a call in ONE launch
            "gpu_launches": (len(reps) if mode["dispatch"] == N.TW_DISPATCH_PERSISTENT
                             else kernels_it * K),
            "nccl_calls": colls_it * K,
            "residual_last": float(hist[-1]),
        }
        if rejected:
            line["rejected_runs"] = rejected
        if extras:
            line["configs_single_gpu"] = extras
        print(json.dumps(line), flush=True)
    # release the solver, the matrix and the NCCL communicator while the
    # process group is still up (not in interpreter-exit destructors)
    S.close()
    del A
    rt.close()


def main():
    args = parse()
    dist, rank, world, local = dist_setup(args)
    try:
        if args.impl == "reference":
            run_reference_arm(args, dist, rank, world)
        else:
            run_ours(args, dist, rank, world, local)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
