"""Print the last N launches of an ncu --csv launch list (ID, kernel, gpu__time_duration)."""
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
for r in rows[1:][-int(sys.argv[2] if len(sys.argv) > 2 else 40):]:
    print(r[ii], r[ki][:70], r[vi])
