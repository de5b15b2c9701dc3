"""Opcode histogram of the innermost FFMA2 loop of a kernel (SASS, offline)."""
import re, subprocess, sys, collections
lib, fn = sys.argv[1], sys.argv[2]
full = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
parts = full.split("Function : ")
out = next(p for p in parts if p.startswith(fn))
ins = []
for line in out.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
# find backward branches whose body contains FFMA2
best = None
for i, (addr, txt) in enumerate(ins):
    m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", txt)
    if not m:
        continue
    tgt = m.group(1)
    if tgt is None:
        continue
    t = int(tgt, 16)
    if t < addr:
        body = [x for a, x in ins if t <= a <= addr]
        n2 = sum("FFMA2" in x for x in body)
        if n2 and (best is None or len(body) < len(best)):
            best = body
if best is None:
    # fall back to labels
    print("no loop found"); sys.exit()
c = collections.Counter()
for x in best:
    op = x.split()[0] if not x.startswith("@") else x.split()[1]
    c[op.split(".")[0]] += 1
print(len(best), c.most_common(14))
