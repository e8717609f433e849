"""Per-kernel times of scripts/one_solve.py under ncu (launch list CSV)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/p1_one_solve.csv")))
h, out = None, []
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            out.append((d["Kernel Name"].split("(")[0][-50:], float(d["Metric Value"].replace(",", "")) / 1e3))
out = [o for o in out if "transpose" not in o[0]]
agg = collections.OrderedDict()
for k, v in out:
    a = agg.setdefault(k, [0, 0.0, []])
    a[0] += 1
    a[1] += v
    a[2].append(round(v, 1))
print("total us", round(sum(v for _, v in out), 1), "launches", len(out))
for k, (c, v, l) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:50s} {c:4d} {v:9.1f} us", l if c <= 6 else "")
