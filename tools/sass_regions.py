"""Attribute an ncu SASS-level source export (ncu -i R --page source --csv --print-source sass) to the CUDA lines
of one function, using nvdisasm -gi line tables (inline call sites): every instruction counts for the
outermost frame that lies inside [lo, hi] of FILE.
usage: python tools/sass_regions.py SASS_CSV NVDISASM_OUT MANGLED_NAME FILE LO HI [TOP]"""
import csv, re, sys
from collections import defaultdict
csvp, disp, fn, fname, lo, hi = sys.argv[1:7]
lo, hi = int(lo), int(hi)
top = int(sys.argv[7]) if len(sys.argv) > 7 else 60
rows = list(csv.reader(open(csvp)))
hdr = rows[1]
ie, ad = hdr.index("Instructions Executed"), hdr.index("Address")
sc = hdr.index("Warp Stall Sampling (All Samples)") if "Warp Stall Sampling (All Samples)" in hdr else None
data = [r for r in rows[2:] if len(r) > ie]
base = int(data[0][ad], 16)
cnt = {int(r[ad], 16) - base: float(r[ie] or 0) for r in data}
stl = {int(r[ad], 16) - base: float(r[sc] or 0) for r in data} if sc is not None else {}
# parse the function's section of nvdisasm -gi output
lines = open(disp).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + fn + ":"))
frames, pend, attr = [], [], {}
pat = re.compile(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?')
ins = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(.*?);")
for l in lines[start + 1:]:
    if l.startswith(".text.") or "\t.section" in l:
        break
    m = pat.search(l)
    if m:
        pend.append((m.group(1).split("/")[-1], int(m.group(2))))
        continue
    m = ins.search(l)
    if m:
        if pend:
            frames = pend
            pend = []
        off = int(m.group(1), 16)
        # frames: innermost first, then the call sites outward; take the outermost frame inside [lo, hi]
        key = None
        for f, ln in frames:
            if f == fname and lo <= ln <= hi:
                key = ln
        attr[off] = (key, frames[0] if frames else None, m.group(2).split()[0] if m.group(2).split() else "?")
tot = sum(cnt.values())
by_line, by_inner, by_stall = defaultdict(float), defaultdict(float), defaultdict(float)
for off, c in cnt.items():
    k, inner, op = attr.get(off, (None, None, "?"))
    by_line[k] += c
    by_inner[inner] += c
    by_stall[k] += stl.get(off, 0.0)
tst = sum(stl.values()) or 1.0
src = open([p for p in [fname] if p][0] if False else "/root/repo/paper_2603_11340_b200/csrc/" + fname).read().split("\n")
print(f"total warp instructions {tot:.4e}")
key = (lambda x: -by_stall[x[0]]) if "--by-stall" in sys.argv else (lambda x: -x[1])
for k, v in sorted(by_line.items(), key=key)[:top]:
    txt = src[k - 1].strip()[:100] if k else "(outside)"
    print(f"{100 * v / tot:6.2f}% inst {100 * by_stall[k] / tst:6.2f}% stall  {k}  {txt}")
