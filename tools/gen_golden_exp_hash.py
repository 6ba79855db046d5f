"""Writes tests/golden/exp_q32_block_hash.txt: per 2^20-input block, the order-free hash of the ORACLE's
E_q(u) over all 2^32 u (tests/harness/oracle_exhaustive.c calls only oracle/).  The device's
exhaustive transform test (tests/test_gpu_exhaustive.py) compares its own block hashes against this file;
tests/test_oracle_exhaustive.py re-derives it from the oracle so the file cannot drift."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import harness  # noqa: E402

h, nonmono, maxerr = harness.exp_scan()
path = os.path.join(ROOT, "tests", "golden", "exp_q32_block_hash.txt")
with open(path, "w") as fh:
    fh.write("# E_q (DESIGN.md §2.2) of the CPU oracle over all 2^32 inputs: block b = [b 2^20, (b+1) 2^20),\n")
    fh.write("# hash_b = sum_u (E_q(u) ^ (u * 0x9E3779B97F4A7C15)) * 0xBF58476D1CE4E5B9 mod 2^64.\n")
    fh.write("# Written by tools/gen_golden_exp_hash.py (calls only oracle/).\n")
    fh.write(f"# nonmono {nonmono}\n")
    for b, v in enumerate(h):
        fh.write(f"{b} {v:016x}\n")
print(f"wrote {path}: nonmono={nonmono} maxerr={maxerr:.3e}")
