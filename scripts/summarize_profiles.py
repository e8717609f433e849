"""Summarize ncu captures (gpurun_out/*.ncu-rep, launch-list CSV) into profiles/.

  python scripts/summarize_profiles.py ROUND WORKLOAD rep1.ncu-rep [rep2 ...] --launches launches.csv

Writes profiles/<ROUND>_<WORKLOAD>_kernels.md (per-kernel key metrics),
profiles/<ROUND>_<WORKLOAD>_launches.md (launch-list shares) and merges
the per-Hv DRAM traffic into profiles/traffic.json for bench.py.
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__cycles_active.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        stalls = {}
        for h, u, v in zip(hdr, units, r):
            if h in KEYS:
                d[h] = (v, u)
            if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
                try:
                    stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v.replace(",", ""))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        d["top_stalls"] = sorted(((k, round(100 * v / tot, 1)) for k, v in stalls.items()),
                                 key=lambda x: -x[1])[:4]
        res.append(d)
    return res


def to_bytes(v, u):
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return x * scale


def to_us(v, u):
    x = float(v.replace(",", ""))
    return x * {"nsecond": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "ns": 1e-3}.get(u, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("round")
    ap.add_argument("workload")
    ap.add_argument("reps", nargs="*")
    ap.add_argument("--launches")
    ap.add_argument("--hv-kernels", default="csr_dv,seg_spmv,seg_fixup")
    args = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lines = [f"# {args.round} {args.workload}: ncu --set full --clock-control none (cold caches, "
             "one launch per kernel)", "",
             "| kernel | us | DRAM read MB | DRAM write MB | DRAM %peak | warps active % | regs | "
             "grid x block | top stalls |", "|---|---|---|---|---|---|---|---|---|"]
    traffic = 0.0
    hv_names = args.hv_kernels.split(",")
    seen = set()
    for rep in args.reps:
        for d in raw(rep):
            name = d["kernel"].split("(")[0].replace("void ", "").replace("tb::<unnamed>::", "")
            us = to_us(*d["gpu__time_duration.sum"])
            rd = to_bytes(*d["dram__bytes_read.sum"]) / 1e6
            wr = to_bytes(*d["dram__bytes_write.sum"]) / 1e6
            lines.append(f"| `{name[:60]}` | {us:.1f} | {rd:.1f} | {wr:.1f} | "
                         f"{d.get('dram__cycles_active.avg.pct_of_peak_sustained_elapsed', ('?',))[0]} | "
                         f"{d.get('sm__warps_active.avg.pct_of_peak_sustained_active', ('?',))[0]} | "
                         f"{d.get('launch__registers_per_thread', ('?',))[0]} | "
                         f"{d.get('launch__grid_size', ('?',))[0]} x {d.get('launch__block_size', ('?',))[0]} | "
                         f"{', '.join(f'{k} {v}%' for k, v in d['top_stalls'])} |")
            base = name.split("<")[0]
            if any(h in base for h in hv_names) and base not in seen:
                seen.add(base)
                traffic += (rd + wr) * 1e6
    with open(os.path.join(ROOT, "profiles", f"{args.round}_{args.workload}_kernels.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic > 0:
        path = os.path.join(ROOT, "profiles", "traffic.json")
        try:
            tj = json.load(open(path))
        except Exception:
            tj = {}
        tj[args.workload] = traffic
        json.dump(tj, open(path, "w"), indent=1)
    if args.launches:
        rows = list(csv.reader(open(args.launches)))
        hdr = None
        agg = defaultdict(lambda: [0, 0.0])
        for r in rows:
            if r and r[0] == "ID":
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                d = dict(zip(hdr, r))
                if d["Metric Name"] == "gpu__time_duration.sum":
                    k = d["Kernel Name"].split("(")[0].replace("void ", "").replace("tb::<unnamed>::", "")
                    agg[k][0] += 1
                    agg[k][1] += to_us(d["Metric Value"], d["Metric Unit"])
        tot = sum(v[1] for v in agg.values()) or 1.0
        out = [f"# {args.round} {args.workload}: launch list (ncu --metrics gpu__time_duration.sum "
               "--clock-control none; TRON_B200_NO_GRAPH=1 so CG-loop kernels are profiled "
               "individually; includes warm-up, setup and the bench's kernel timing loop)", "",
               "| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            out.append(f"| `{k[:70]}` | {v[0]} | {v[1]:.1f} | {v[1] / v[0]:.2f} | {100 * v[1] / tot:.1f}% |")
        with open(os.path.join(ROOT, "profiles", f"{args.round}_{args.workload}_launches.md"), "w") as f:
            f.write("\n".join(out) + "\n")
    print("traffic per Hv (bytes):", traffic)


if __name__ == "__main__":
    main()
