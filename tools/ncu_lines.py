"""Per-CUDA-source-line instruction and stall totals from an ncu report (needs -lineinfo).
usage: python tools/ncu_lines.py REPORT [TOP] [KERNEL_REGEX]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 3:
    cmd += ["-k", "regex:" + sys.argv[3]]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = "?"
hdr = None
acc = []
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        ie = float(r[7]); st = float(r[4])
    except (ValueError, IndexError):
        continue
    acc.append((ie, st, fname, r[0], r[1][:90]))
tot = sum(a[0] for a in acc); tst = sum(a[1] for a in acc)
print(f"total warp instructions {tot:.3e}, stall samples {tst:.0f}")
for ie, st, f, ln, src in sorted(acc, reverse=True)[:top]:
    print(f"{100*ie/tot:6.2f}% inst {100*st/tst:6.2f}% stall  {f}:{ln}  {src}")
