"""Dynamic instruction totals per source region from an ncu report (needs -lineinfo):
python tools/ncu_regions.py report.ncu-rep 'name:file:lo-hi' ..."""
import csv, io, subprocess, sys
rep = sys.argv[1]
regions = []
for a in sys.argv[2:]:
    name, f, rng = a.split(":")
    lo, hi = rng.split("-")
    regions.append((name, f, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, tot, acc = "?", None, 0.0, {}
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
        ie = float(r[7]); ln = int(r[0])
    except (ValueError, IndexError):
        continue
    tot += ie
    key = "other:" + fname
    for name, f, lo, hi in regions:
        if f == fname and lo <= ln <= hi:
            key = name
            break
    acc[key] = acc.get(key, 0.0) + ie
print(f"total {tot:.4e}")
for k, v in sorted(acc.items(), key=lambda x: -x[1]):
    print(f"{100 * v / tot:6.2f}%  {v:.3e}  {k}")
