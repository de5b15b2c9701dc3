"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list.
  python tools/launch_summary.py launches.csv "header line" > summary.txt"""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if r]
h = None; agg = collections.OrderedDict(); tot = 0.0
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
for r in rows:
    if "Kernel Name" in r:
        h = r; continue
    if h is None or len(r) != len(h):
        continue
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    ms = float(d["Metric Value"].replace(",", "")) * scale.get(d.get("Metric Unit", "ns"), 1e-6)
    k = d["Kernel Name"].split("(")[0]
    a = agg.setdefault(k, [0, 0.0]); a[0] += 1; a[1] += ms; tot += ms
print(sys.argv[2] if len(sys.argv) > 2 else "# launch list")
print("# kernel, launches, total ms, mean ms, share of all listed time")
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k}, {n}, {ms:.3f}, {ms / n:.4f}, {100 * ms / tot:.1f}%")
