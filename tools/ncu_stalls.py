"""Warp-stall breakdown (pc-sampling percentages) of every kernel row in an ncu --page raw --csv export."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
for r in rows[2:]:
    st = [(h[i], r[i]) for i in range(len(h)) if "smsp__pcsamp_warps_issue_stalled" in h[i] and not h[i].endswith("not_issued")]
    tot = sum(float(x[1] or 0) for x in st) or 1.0
    top = sorted(st, key=lambda t: -float(t[1] or 0))[:10]
    print(r[h.index("Kernel Name")] if "Kernel Name" in h else "?", "stalls %:",
          ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * float(x) / tot:.1f}" for k, x in top))
