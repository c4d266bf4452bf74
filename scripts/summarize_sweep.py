"""profiles/r01_sweep_summary.md from the final C2 / C5 sweep
(profiles/r01_sweep_c2_c5_final.jsonl) and C4 (profiles/r01_sweep_c4_final.jsonl)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")


def mode(d):
    return "persistent" if d.get("dispatch") == "persistent" else ("graph" if d.get("cuda_graph") else "streams")


c2, c5, mono = [], {}, None
for line in open(os.path.join(P, "r01_sweep_c2_c5_final.jsonl")):
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    if d["config"].startswith("C2"):
        c2.append(d)
    elif "monolithic reference" in d["config"]:
        mono = d
    else:
        c5.setdefault(d["tiles"], {})[mode(d)] = d
c4 = [json.loads(l) for l in open(os.path.join(P, "r01_sweep_c4_final.jsonl")) if l.startswith("{")]
m = mono["ms_per_iter"]
out = ["# r01 sweep on 1x B200 (scripts/sweep.py, final round-1 build): ms/iter, GFLOP/s, host enqueue ms/iter",
       "",
       "x-staged K1 everywhere it applies (monolithic, tasks tiles, dispatcher SpMV chunks); the",
       "dispatcher's update chunks stream their operands by TMA; from 4M rows the x update rides",
       "on the p update (K3 / p-update tiles / chunks).  Data: `r01_sweep_c2_c5_final.jsonl`,",
       "`r01_sweep_c4_final.jsonl` (`scripts/summarize_sweep.py` writes this file).",
       "",
       "## C2 128^3: monolithic vs block-task DAG (streams, CUDA graph, persistent dispatcher)",
       "| variant | tiles | dispatch | ms/iter | GFLOP/s | kernels/iter | host enqueue ms/iter |",
       "|---|---|---|---|---|---|---|"]
for d in c2:
    out.append(f"| {d['variant']} | {d['tiles']} | {mode(d)} | {d['ms_per_iter']:.4f} | {d['gflops']:.0f} | "
               f"{d.get('kernels_per_iter', 0)} | {d['host_enqueue_ms_per_iter']:.4f} |")
out += ["", "## C5 256^3 granularity (tiles per GPU; the 8-GPU sweep's 8..512 blocks total = 1..64 per GPU)",
        "| tiles/GPU | streams | graph | persistent | persistent vs monolithic | kernels/iter (streams, graph) |",
        "|---|---|---|---|---|---|"]
for t in sorted(c5):
    r = c5[t]
    out.append(f"| {t} | {r['streams']['ms_per_iter']:.4f} | {r['graph']['ms_per_iter']:.4f} | "
               f"{r['persistent']['ms_per_iter']:.4f} | {r['persistent']['ms_per_iter'] / m:.3f} | "
               f"{r['streams'].get('kernels_per_iter', '')} |")
out.append(f"| monolithic (graph) | | {m:.4f} | | 1.000 | 3 |")
out += ["", "## C4 512^3 on one B200", "| graph | ms/iter | GFLOP/s |", "|---|---|---|"]
for d in c4:
    out.append(f"| {d['cuda_graph']} | {d['ms_per_iter']:.3f} | {d['gflops']:.0f} |")
out += ["", "Tile kernels of a phase get min(T, stream-pool capacity) shares of the resident grid when T <= 8.", ""]
open(os.path.join(P, "r01_sweep_summary.md"), "w").write("\n".join(out))
print("\n".join(out))
