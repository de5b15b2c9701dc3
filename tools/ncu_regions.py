"""Stall/instruction split of each kernel in an ncu source export between the
FFMA2 (consumer) region and everything else.
  ncu -i rep --page source --csv --print-source=sass > x.csv; python tools/ncu_regions.py x.csv"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}; blocks.append(cur); continue
    if r and r[0] == "Address":
        cur["hdr"] = r; continue
    if cur and "hdr" in cur and len(r) == len(cur["hdr"]):
        cur["rows"].append(r)
seen = set()
for b in blocks:
    if b["name"] in seen:
        continue
    seen.add(b["name"])
    h = b["hdr"]; ix = h.index("Warp Stall Sampling (All Samples)"); ie = h.index("Instructions Executed")
    cols = {c: i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c}
    rs = b["rows"]
    ff = [i for i, r in enumerate(rs) if "FFMA2" in r[1]]
    if not ff:
        continue
    lo, hi = min(ff), max(ff)

    def agg(sel):
        st = collections.Counter(); n = e = 0
        ops = collections.Counter()
        for i in sel:
            r = rs[i]; n += int(r[ix] or 0); e += int(r[ie] or 0)
            t = r[1].split(); o = t[1] if t[0].startswith("@") else t[0]
            ops[o.split(".")[0]] += int(r[ie] or 0)
            for c, j in cols.items():
                st[c] += int(r[j] or 0)
        return n, e, st.most_common(7), ops.most_common(8)
    print(b["name"][:60])
    for nm, sel in (("consumer", range(lo, hi + 1)), ("other", [i for i in range(len(rs)) if i < lo or i > hi])):
        n, e, st, ops = agg(sel)
        print(f"  {nm}: samples {n} instr {e}\n    stalls {st}\n    ops {ops}")
