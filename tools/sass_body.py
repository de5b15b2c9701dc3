import re, subprocess, sys
lib, fn = sys.argv[1], sys.argv[2]
full = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
out = next(p for p in full.split("Function : ") if p.startswith(fn))
ins=[]
for line in out.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m: ins.append((int(m.group(1),16), m.group(2).strip()))
best=None
for i,(addr,txt) in enumerate(ins):
    m=re.search(r"BRA\s+0x([0-9a-f]+)", txt)
    if m and int(m.group(1),16) < addr:
        t=int(m.group(1),16)
        body=[x for a,x in ins if t<=a<=addr]
        if any('FFMA2' in x for x in body) and (best is None or len(body)<len(best)): best=body
for x in best:
    if len(sys.argv) > 3 or 'FFMA2' not in x: print(x)
