"""Summarise a gpurun ncu capture into profiles/ (launch list + full-set metrics
of K1, and of K2 / K3 when their reports exist next to K1's).
usage: python scripts/summarize_ncu.py <launches.csv> <prof_k1.ncu-rep> <round tag>"""
import os
import collections
import csv
import json
import subprocess
import sys

launches, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(launches)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
per, names = collections.defaultdict(dict), {}
for r in rows[hi + 1:]:
    per[r[0]][r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
    names[r[0]] = r[h.index("Kernel Name")]
agg = collections.OrderedDict()
for k, m in per.items():
    nm = names[k].split("(")[0].replace("void ", "").split("::")[-1]
    a = agg.setdefault(nm, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0)
    a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
it = [k for k in agg if k.startswith(("spmv", "update"))]
# x-update pairs: the two K3 kernels alternate, one of them per iteration
# x-update pairs: the pair's two K3 kernels alternate, one of them per
# iteration; the single-update K3 then only ends a call of odd length
pairs = "update_p_kernel<0, 2>" in agg  # update_p_kernel<PEER, XU>: XU 2 = the pair's second K3
half = {"update_p_kernel<0, 0>", "update_p_kernel<0, 2>"} if pairs else set()
wgt = {k: 0.5 if k in half else 0.0 if pairs and k == "update_p_kernel<0, 1>" else 1.0
       for k in it}
tot = sum(wgt[k] * agg[k][1] / agg[k][0] for k in it)
out = [f"# ncu launch list ({tag}): bench.py --steps 6 --warmup 3 at 256^3, 1 B200, --clock-control none",
       "# kernel, launches, avg us, avg dram bytes/launch, share of the iteration's kernels"]
for k, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    ours = k.startswith(("spmv", "update", "stencil", "band", "rhs", "dot", "scan", "combine",
                         "fill", "csr", "ell", "rank_group", "dag", "peer", "waxpby"))
    sh = ("odd-length call's last K3 (single x update)" if k in it and wgt[k] == 0 else
          f"share_of_iteration={wgt[k] * t / c / tot:.3f}" if k in it else
          "setup (once per solve)" if ours else "not this library (torch: bench's read-stream reference)")
    out.append(f"{k:28s} {c:4d} {t / c / 1e3:10.1f} us {b / c / 1e9:8.3f} GB  {sh}")
open(f"profiles/{tag}_ncu_launches_summary.txt", "w").write("\n".join(out) + "\n")
print("\n".join(out))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
NNZ, N = 449455096, 16777216  # 256^3


def summarize(rep_path, kernel, algorithmic, out_json=None, format_bytes=None):
    raw = subprocess.run(["ncu", "-i", rep_path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    H, U, V = r[0], r[1], r[2]
    summ = {k: [V[H.index(k)], U[H.index(k)]] for k in KEYS if k in H}
    traffic = sum(float(summ[k][0]) * SCALE[summ[k][1]]
                  for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    d = {"kernel": kernel, "workload": "256x256x256", "round": tag,
         "source": "ncu --set full --clock-control none, bench.py --steps 6 --warmup 3",
         "dram_bytes_per_launch": traffic, "algorithmic_bytes": algorithmic, "metrics": summ}
    if format_bytes:
        d["format_bytes"] = format_bytes  # 16-bit staged columns: 10 B per nonzero
    if out_json:
        json.dump(d, open(out_json, "w"), indent=1)
        print(json.dumps(d, indent=1))
    return d


# the K1 capture is whichever TMA SpMV the bench ran (-k regex:spmv_tma)
_k1 = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
_staged = "staged" in _k1.split("\n", 3)[2] if _k1.count("\n") > 2 else False
summarize(rep, "spmv_tma_staged_kernel (K1, x-staged)" if _staged else "spmv_tma_kernel<true> (K1)",
          12 * NNZ + 16 * N, "profiles/k1_traffic.json",
          format_bytes=(10 * NNZ + 16 * N) if _staged else None)
base = os.path.dirname(rep)


def _name_of(path):  # demangled kernel name of a one-kernel capture
    t = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                       text=True).stdout
    return t.split("\n", 3)[2] if t.count("\n") > 2 else ""


# from 4M rows the x update runs in K3 (update_xr_kernel<false> streams
# r, Ap -> r: 24 n; update_p_kernel<false, true> r, p, x -> p, x: 40 n); a
# one-GPU monolithic solve pairs it (prof_k3p: update_p_kernel<false, 2>,
# r, p, p_prev, x -> p, x: 48 n; prof_k3 then holds the pair's first K3,
# update_p_kernel<false, 0>, r, p -> p: 24 n)
_xk3 = "update_xr_kernel<0>" in _name_of(os.path.join(base, "prof_k2.ncu-rep"))
_k3p = os.path.join(base, "prof_k3p.ncu-rep")
_pairs = os.path.exists(_k3p)
if os.path.exists(os.path.join(base, "prof_k2.ncu-rep")):
    summarize(os.path.join(base, "prof_k2.ncu-rep"),
              "update_xr_kernel (K2%s)" % (", r only" if _xk3 else ""), (24 if _xk3 else 48) * N,
              "profiles/k2_traffic.json")
_k3 = os.path.join(base, "prof_k3.ncu-rep")
if _pairs and os.path.exists(_k3):
    a = summarize(_k3, "update_p_kernel<false, 0> (K3, first of an x pair)", 24 * N)
    b = summarize(_k3p, "update_p_kernel<false, 2> (K3, second of an x pair)", 48 * N)
    d = {"kernel": "K3 x-update pair: update_p_kernel<false, 0> + update_p_kernel<false, 2>, "
                   "per launch averaged over the pair",
         "workload": "256x256x256", "round": tag, "source": a["source"],
         "dram_bytes_per_launch": (a["dram_bytes_per_launch"] + b["dram_bytes_per_launch"]) / 2,
         "algorithmic_bytes": 36 * N, "launches": {"first": a, "second": b}}
    json.dump(d, open("profiles/k3_traffic.json", "w"), indent=1)
    print(json.dumps(d, indent=1))
elif os.path.exists(_k3):
    summarize(_k3, "update_p_kernel<false%s> (K3)" % (", true" if _xk3 else ""),
              (40 if _xk3 else 24) * N, "profiles/k3_traffic.json")
