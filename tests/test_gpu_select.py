"""K1b (slo_select_rows) against the definition of the nearest-rank order statistic ("p99"; S:123,
S:165: the ceil(q n)-th smallest), computed here by sorting each row with numpy.  The rows are adversarial for
the kernel's log-scale bucket + shared-memory path: full-range uniform values, constant rows, values below 16
(the exact-value buckets), one bucket holding more than the 1,024 values shared memory takes (row fallback),
a bucket of 257..1,024 values (radix passes in shared memory), latency-like log-normal rows, rows whose length
is not a multiple of 4 (unaligned rows: scalar loads), very short rows, and uncounted UINT32_MAX entries
(the stop rule's convention)."""
import numpy as np
import pytest
import torch

from paper_2603_11340_b200 import inputs, sim

pytestmark = pytest.mark.gpu
U32MAX = 0xFFFFFFFF


def expected(rows: np.ndarray, nm: np.ndarray, q: int) -> np.ndarray:
    out = []
    for row, m in zip(rows, nm):
        s = np.sort(row.astype(np.uint64))
        rq = (q * int(m) + 99) // 100
        out.append(int(s[rq - 1]) if rq > 0 else int(s[-1]))
    return np.array(out, dtype=np.uint64)


def families(rng: np.random.Generator, n: int) -> np.ndarray:
    rows = [
        rng.integers(0, 2**32, n, dtype=np.uint64),                        # full range
        np.full(n, 7, dtype=np.uint64),                                     # constant, exact bucket
        np.full(n, 123_456, dtype=np.uint64),
        np.full(n, U32MAX, dtype=np.uint64),
        rng.integers(0, 16, n, dtype=np.uint64),                            # exact-value buckets
        np.where(rng.random(n) < 0.5, 1_000_000, rng.integers(0, 2**20, n)).astype(np.uint64),  # huge bucket
        np.minimum(np.round(np.exp(rng.normal(13.5, 0.6, n))), U32MAX).astype(np.uint64),        # latency-like
        rng.integers(0, 2, n, dtype=np.uint64) * 2**31,                     # two values
    ]
    mid = rng.integers(0, 2**16, n, dtype=np.uint64)                        # a 257..1,024-value top bucket
    k = min(n, 600)
    mid[rng.choice(n, k, replace=False)] = rng.integers(2**24, 2**24 + 2**20, k, dtype=np.uint64)
    rows.append(mid)
    return np.stack(rows)


@pytest.fixture(scope="module")
def S():
    return sim.Simulator([inputs.preset_ll()], device=0)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 17, 100, 2000, 4099, 10_000])
def test_select_rows_matches_sorted_definition(S, n):
    rng = np.random.default_rng(1000 + n)
    rows = families(rng, n)
    nm = np.full(len(rows), n, dtype=np.uint64)
    dev = torch.device("cuda", 0)
    t = torch.from_numpy(rows.astype(np.uint32).view(np.int32)).to(dev)
    out = S.select_rows(t, percentiles=True)
    torch.cuda.synchronize()
    for key, q in (("p99_us", 99), ("p50_us", 50), ("p95_us", 95)):
        got = out[key].cpu().numpy().view(np.uint32).astype(np.uint64)
        np.testing.assert_array_equal(got, expected(rows, nm, q), err_msg=f"{key} n={n}")


def test_select_rows_uncounted_entries(S):
    """Rows whose last n - m entries are UINT32_MAX (uncounted), with per-row counts m (m = 0: the largest)."""
    rng = np.random.default_rng(7)
    n, R = 3001, 64
    rows = np.minimum(np.round(np.exp(rng.normal(13.5, 0.8, (R, n)))), U32MAX).astype(np.uint64)
    nm = rng.integers(0, n + 1, R).astype(np.uint64)
    nm[:4] = [0, 1, n, n - 1]
    for r in range(R):
        rows[r, int(nm[r]):] = U32MAX
    dev = torch.device("cuda", 0)
    t = torch.from_numpy(rows.astype(np.uint32).view(np.int32)).to(dev)
    tn = torch.from_numpy(nm.astype(np.int32)).to(dev)
    out = S.select_rows(t, n_measured=tn, percentiles=True)
    torch.cuda.synchronize()
    for key, q in (("p99_us", 99), ("p50_us", 50), ("p95_us", 95)):
        got = out[key].cpu().numpy().view(np.uint32).astype(np.uint64)
        np.testing.assert_array_equal(got, expected(rows, nm, q), err_msg=key)


def test_select_rows_many_rows_one_wave(S):
    """More rows than one wave of resident blocks (grid-stride rows), random lengths of latency-like values."""
    rng = np.random.default_rng(11)
    R, n = 5000, 257
    rows = np.minimum(np.round(np.exp(rng.normal(12.0, 1.0, (R, n)))), U32MAX).astype(np.uint64)
    nm = np.full(R, n, dtype=np.uint64)
    t = torch.from_numpy(rows.astype(np.uint32).view(np.int32)).to(torch.device("cuda", 0))
    out = S.select_rows(t)
    torch.cuda.synchronize()
    got = out["p99_us"].cpu().numpy().view(np.uint32).astype(np.uint64)
    np.testing.assert_array_equal(got, expected(rows, nm, 99))


@pytest.mark.parametrize("n", [1, 5, 700, 3000, 5001])
def test_select_rows_block_sizes(S, n):
    """More rows than SMs, so K1b takes its row-length block size (64 / 128 / 256 threads for these lengths);
    every adversarial family repeated over 300 rows."""
    rng = np.random.default_rng(50 + n)
    fam = families(rng, n)
    rows = np.concatenate([fam] * (300 // len(fam) + 1))[:300]
    rows[::7] = rng.integers(0, 2**32, (len(rows[::7]), n), dtype=np.uint64)
    nm = np.full(len(rows), n, dtype=np.uint64)
    t = torch.from_numpy(rows.astype(np.uint32).view(np.int32)).to(torch.device("cuda", 0))
    out = S.select_rows(t, percentiles=True)
    torch.cuda.synchronize()
    for key, q in (("p99_us", 99), ("p50_us", 50), ("p95_us", 95)):
        got = out[key].cpu().numpy().view(np.uint32).astype(np.uint64)
        np.testing.assert_array_equal(got, expected(rows, nm, q), err_msg=f"{key} n={n}")
