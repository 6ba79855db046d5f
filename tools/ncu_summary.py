"""Summarise an ncu report (raw metrics + SASS opcode mix + hottest instructions) for profiles/."""
import csv
import io
import json
import subprocess
import sys
from collections import Counter

KEYS = ["gpu__time_duration.sum", "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size",
        "launch__block_size", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_per_inst_issued.ratio", "sm__cycles_elapsed.avg.per_second",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, out_json):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    metrics = {k: (vals[hdr.index(k)], units[hdr.index(k)]) for k in KEYS if k in hdr}
    kernel = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    srows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    h = srows[1]
    ie, src, st = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    at = h.index("Avg. Threads Executed")
    tot = sum(float(r[ie] or 0) for r in srows[2:])
    ops, stalls = Counter(), Counter()
    for r in srows[2:]:
        toks = r[src].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        ops[op.split(".")[0]] += float(r[ie] or 0)
        stalls[op.split(".")[0]] += float(r[st] or 0)
    lanes = sum(float(r[ie] or 0) * float(r[at] or 0) for r in srows[2:]) / max(tot, 1)
    summary = {"report": rep, "kernel": kernel, "metrics": metrics, "warp_instructions": tot,
               "avg_threads_per_instruction": lanes,
               "opcode_mix_pct": {k: round(100 * v / tot, 2) for k, v in ops.most_common(20)},
               "stall_samples_by_opcode": dict(stalls.most_common(12))}
    json.dump(summary, open(out_json, "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
