"""Exhaustive pins of the oracle's integer transforms over all 2^32 inputs (SURVEY §8(c) pins table).

* Noise ("light noise"): f(w) = 10^6 + (b0+b1+b2+b3 - 510)·step takes exactly the 1,021
  lattice values 10^6 + (k - 510)·step, k = 0..1020, with multiplicities equal to the 4-fold convolution of
  the uniform byte law (Irwin–Hall of four bytes), mean exactly 10^6 and range ±510·step.  The counts are
  computed here by numpy's convolution, independently of the oracle.
* E_q: |E_q(u)/2^32 − (−ln((u+1)/2^32))| ≤ 2^−26 for every u (libm in double), and the
  oracle's block hashes equal the golden file the device test compares against (tools/gen_golden_exp_hash.py).
"""
import os

import numpy as np
import pytest

import harness

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _byte_sum_law():
    one = np.ones(256, dtype=object)       # exact integers
    c = one
    for _ in range(3):
        c = np.convolve(c, one)
    return [int(x) for x in c]             # 1,021 counts of b0+b1+b2+b3 = 0..1020


@pytest.mark.parametrize("step", [0, 1, 338, 1960])
def test_noise_factor_law_exhaustive(step):
    counts, off, total = harness.noise_scan(step)
    assert off == 0                                   # every f lies on the lattice 10^6 + (k - 510) step
    if step == 0:
        assert counts[510] == 2 ** 32 and sum(counts) == 2 ** 32
        assert total == 10 ** 6 * 2 ** 32
        return
    law = _byte_sum_law()
    assert sum(law) == 2 ** 32 and law[0] == 1 and law[510] == max(law)
    assert counts == law                              # Irwin–Hall of four uniform bytes, exactly
    assert sum(1 for c in counts if c) == 1021        # 1,021 distinct values
    assert total == 10 ** 6 * 2 ** 32                 # mean exactly 10^6 ppm (symmetric law about 510)
    # range: 10^6 ± 510 step (k = 0 and k = 1020 occur exactly once each: all bytes 0 / all 255)
    assert counts[0] == 1 and counts[1020] == 1


def test_noise_factor_examples(orc):
    assert orc.noise_factor(0x00000000, 338) == 10 ** 6 - 510 * 338
    assert orc.noise_factor(0xFFFFFFFF, 338) == 10 ** 6 + 510 * 338
    assert orc.noise_factor(0x7F7F8080, 338) == 10 ** 6           # 127 + 127 + 128 + 128 = 510
    assert orc.noise_factor(0x01020304, 1) == 10 ** 6 + 10 - 510
    assert orc.noise_factor(0x12345678, 0) == 10 ** 6


def test_exp_q32_exhaustive_bound_and_golden():
    hashes, nonmono, maxerr = harness.exp_scan()
    assert maxerr <= 2.0 ** -26                       # DESIGN.md §2.2 accuracy, every u
    # E_q is NOT monotone in u at the 2^-26 scale (the floored polynomial); nothing in the model needs it
    # (R27).  The count is recorded in DESIGN.md, not asserted.
    assert nonmono < 2 ** 32 // 100
    gold = {}
    with open(os.path.join(GOLD, "exp_q32_block_hash.txt")) as fh:
        for line in fh:
            if line.startswith("#"):
                continue
            b, v = line.split()
            gold[int(b)] = int(v, 16)
    assert [gold[b] for b in range(4096)] == hashes
