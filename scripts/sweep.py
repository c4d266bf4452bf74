"""Config sweeps on one B200 (BASELINE.json configs 2, 4, 5; one JSON line each).

  C2  128^3: monolithic vs block-task DAG (tiles 4/8/16/64), streams vs CUDA graph
  C4  512^3 on one GPU (the P=1 point of the strong-scaling config)
  C5  256^3 task granularity: tiles per GPU 1..512 (the 8-GPU sweep's per-GPU
      share is B/8), streams vs CUDA graph

Timing: CUDA events on the solver's compute stream around K iterations after
W warm-up iterations (stream-joined, so all pooled streams are inside).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_21897_b200 as P  # noqa: E402


def measure(rt, A, variant, tiles, graph, K, W, persistent=False):
    s = torch.cuda.ExternalStream(rt.compute_stream)
    S = P.CgSolver(rt, A, W + 2 * K, P.CgOptions(tiles=tiles, use_graph=graph,
                                                 iteration_marks=False, persistent=persistent),
                   variant=variant)
    b = P.rhs_xorshift(rt, A.n, 7)
    S.set_rhs(b)
    S.iterate(K)  # untimed: builds the graph / dispatcher table for K
    S.set_rhs(b)
    t_enq0 = time.perf_counter()
    S.iterate(W)
    S.wait()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    t0 = time.perf_counter()
    S.iterate(K)
    t_host = time.perf_counter() - t0
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    h = S.history(W + K)
    kl, cl = S.launches_per_iteration()
    S.close()
    del t_enq0
    n, nnz = A.n, A.nnz()
    return {"ms_per_iter": ms, "gflops": (2 * nnz + 10 * n) / (ms / 1e3) / 1e9,
            "gbs": (12 * nnz + 88 * n) / (ms / 1e3) / 1e9, "iters_per_s": 1e3 / ms,
            "host_enqueue_ms_per_iter": t_host * 1e3 / K, "kernels_per_iter": kl,
            "residual_last": float(h[-1])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2,c5,c4")
    ap.add_argument("--K", type=int, default=30)
    ap.add_argument("--W", type=int, default=5)
    ap.add_argument("--tiles", default="1,2,4,8,16,32,64,128,256,512")
    ap.add_argument("--only-persistent", action="store_true")
    a = ap.parse_args()
    rt = P.Runtime(0, stream_pool_capacity=4)
    cfgs = a.configs.split(",")
    if "c2" in cfgs:
        A = P.gen_stencil_matrix(128, 128, 128, rt=rt)
        for variant, tiles in [(0, 1), (1, 1), (1, 4), (1, 8), (1, 16), (1, 64)]:
            for graph in (False, True):
                r = measure(rt, A, variant, tiles, graph, 100, 10)
                print(json.dumps({"config": "C2 HPCCG 128^3 1xB200",
                                  "variant": "monolithic" if variant == 0 else "tasks",
                                  "tiles": tiles, "cuda_graph": graph, **r}), flush=True)
            if variant == 1:
                r = measure(rt, A, 1, tiles, False, 100, 10, persistent=True)
                print(json.dumps({"config": "C2 HPCCG 128^3 1xB200", "variant": "tasks",
                                  "tiles": tiles, "dispatch": "persistent", **r}), flush=True)
        del A
    if "c5" in cfgs:
        A = P.gen_stencil_matrix(256, 256, 256, rt=rt)
        for tiles in [int(t) for t in a.tiles.split(",")]:
            for graph in (() if a.only_persistent else (False, True)):
                r = measure(rt, A, 1, tiles, graph, a.K, a.W)
                print(json.dumps({"config": "C5 HPCCG 256^3 granularity, per-GPU tiles",
                                  "blocks_total_8gpu_equiv": tiles * 8, "tiles": tiles,
                                  "cuda_graph": graph, **r}), flush=True)
            r = measure(rt, A, 1, tiles, False, a.K, a.W, persistent=True)
            print(json.dumps({"config": "C5 HPCCG 256^3 granularity, per-GPU tiles",
                              "blocks_total_8gpu_equiv": tiles * 8, "tiles": tiles,
                              "dispatch": "persistent", **r}), flush=True)
        r = measure(rt, A, 0, 1, True, a.K, a.W)
        print(json.dumps({"config": "C5 HPCCG 256^3 monolithic reference point", "tiles": 1,
                          "cuda_graph": True, **r}), flush=True)
        del A
    if "c4" in cfgs:
        torch.cuda.synchronize()
        A = P.gen_stencil_matrix(512, 512, 512, rt=rt)
        for graph in (False, True):
            r = measure(rt, A, 0, 1, graph, 20, 3)
            print(json.dumps({"config": "C4 HPCCG 512^3 on 1xB200 (strong-scaling P=1 point)",
                              "nnz": A.nnz(), "cuda_graph": graph, **r}), flush=True)
        del A


if __name__ == "__main__":
    main()
