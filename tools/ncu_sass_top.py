"""Top SASS instructions by warp-stall samples from an ncu --page source csv
(one kernel), with the stall reason columns that dominate.
  ncu -i rep --page source --csv --print-source=sass > x.csv; python tools/ncu_sass_top.py x.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kernels, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}; kernels.append(cur); hdr = None; continue
    if r and r[0] == "Address":
        cur["hdr"] = r; continue
    if cur is not None and "hdr" in cur and len(r) == len(cur["hdr"]):
        cur["rows"].append(r)
for k in kernels:
    h = k["hdr"]; ix = h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") or "Stall" in c and "Sampling" not in c]
    tot = sum(int(r[ix] or 0) for r in k["rows"])
    print("==", k["name"][:80], "total samples", tot, "instructions", len(k["rows"]))
    base = int(k["rows"][0][0], 16)
    order = sorted(range(len(k["rows"])), key=lambda i: -int(k["rows"][i][ix] or 0))[:N]
    for i in sorted(order):
        r = k["rows"][i]
        print(f"{int(r[0],16)-base:6x} {int(r[ix] or 0):6d} {100*int(r[ix] or 0)/max(tot,1):5.1f}%  {r[1].strip()[:70]}")
