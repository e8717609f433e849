#!/bin/bash
# ncu launch list (gpu__time_duration per kernel) of profile_n1.py on a workload, default lib or $LIBV.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
W=${1:-N1}; TAG=${2:-default}
[ -n "$LIBV" ] && export TRON_B200_LIB=$PWD/build/$LIBV/libtron_b200.so
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/list_${W}_${TAG}.csv python scripts/profile_n1.py $W > /dev/null 2>&1
echo "ncu rc=$?"
python3 - gpurun_out/list_${W}_${TAG}.csv <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; rows = rows[1:]
iK, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    agg[r[iK][:70]][r[iM]].append(float(r[iV].replace(",", "")))
for k, m in agg.items():
    t = m["gpu__time_duration.sum"]
    print(f"{k:72s} n={len(t):3d} med_us={sorted(t)[len(t)//2]/1e3:8.1f} rdMB={sorted(m['dram__bytes_read.sum'])[len(t)//2]/1e6:7.1f} wrMB={sorted(m['dram__bytes_write.sum'])[len(t)//2]/1e6:6.1f}")
PY
