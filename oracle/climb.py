"""oracle.climb — TEST INFRASTRUCTURE ONLY.

Plain-Python aggregation, score, neighbour generation and Alg. 1 step of SLO-Tuner (arXiv 2603.11340),
written from DESIGN.md §2.9 with Python's unbounded integers (no overflow reasoning needed).

* hw_cost — Eq. (2); weights 0.01/0.01/0.02, as micro-units.
* score   — Eq. (3); lambda = 5.0.
* neighbours — PAPER.md:142 (live stencil), S:83 (sim stencil), R21 (wide-32).
* step    — Alg. 1; move rule P:142 / P:164.
* simulator-controller variant: violation term x viol_mult (10 for the
  simulator: "multiplying the violation term by 10 lambda"), draft/verifier cost w_W*W + w_k*(k_max - k)
  added to Eq. (2) when speculation is on, and the current point judged by the EMA of its p99,
  p_hat(t) = beta p99(t) + (1 - beta) p_hat(t-1) (beta in Q16, floor), started at the first sample.
"""
from __future__ import annotations

import itertools
from typing import Dict, List, Sequence, Tuple

INT64_MIN = -(1 << 63)
DIMS = ("conc", "max_num_seqs", "draft_len", "draft_width", "max_wait_us")


def aggregate(results: Sequence[Dict]) -> Dict:
    """Sum per-seed replica results of one config."""
    agg = dict(sum_p99_us=0, sum_slo_met=0, sum_window_us=0, n_seeds=0, flags=0)
    for r in results:
        agg["sum_p99_us"] += r["p99_us"]
        agg["sum_slo_met"] += r["slo_met"]
        agg["sum_window_us"] += r["window_us"]
        agg["n_seeds"] += 1
        agg["flags"] |= r["flags"]
    return agg


def hw_cost_micro(k: Dict, sp: Dict) -> int:
    """Eq. (2): w_conc*concurrency + w_max*max_num_seqs + w_spec*num_spec_tokens (0 when spec is off),
    plus the simulator's draft/verifier cost w_W*W + w_k*(k_max - k) when speculation is on."""
    gamma = k["draft_len"] if k["spec_on"] else 0
    cost = sp["w_conc_micro"] * k["conc"] + sp["w_max_micro"] * k["max_num_seqs"] + sp["w_spec_micro"] * gamma
    if gamma > 0:
        cost += sp.get("w_W_micro", 0) * k["draft_width"] + sp.get("w_k_micro", 0) * (sp.get("k_max", 16) - gamma)
    return cost


def score_micro(agg: Dict, k: Dict, sp: Dict, p99_ema_us=None) -> int:
    """Eq. (3) in micro-rps: goodput - m*lambda*max(0, p99 - SLO) - hw_cost, pooled over seeds (R17).
    With p99_ema_us the violation uses that EMA value (integer us) instead of the seed-mean p99."""
    n = agg["n_seeds"]
    if n == 0 or (agg["flags"] & 1):
        return INT64_MIN
    mult = sp.get("viol_mult", 1)
    goodput = (agg["sum_slo_met"] * 10**12) // agg["sum_window_us"]
    if p99_ema_us is None:
        excess = max(0, agg["sum_p99_us"] - n * sp["slo_us"])
        penalty = (mult * sp["lambda_milli"] * excess) // (1000 * n)
    else:
        penalty = (mult * sp["lambda_milli"] * max(0, p99_ema_us - sp["slo_us"])) // 1000
    return goodput - penalty - hw_cost_micro(k, sp)


def ema_update(prev, sample: int, beta_q16: int) -> int:
    """p_hat(t) = beta p99(t) + (1 - beta) p_hat(t-1) in integer us (floor); the first sample starts it."""
    if prev is None:
        return sample
    return (beta_q16 * sample + (65536 - beta_q16) * prev) >> 16


def _clamp(v: int, lo: int, hi: int) -> int:
    return lo if v < lo else hi if v > hi else v


def _with(k: Dict, **kw) -> Dict:
    d = dict(k)
    d.update(kw)
    return d


def neighbours(space: Dict, k: Dict) -> List[Dict]:
    """Deterministic neighbour list: clamped to bounds, self and duplicates dropped (first kept)."""
    lo = dict(zip(DIMS, space["lo"]))
    hi = dict(zip(DIMS, space["hi"]))
    st = dict(zip(DIMS, space["step"]))

    def moved(dim, sign):
        return _with(k, **{dim: _clamp(k[dim] + sign * st[dim], lo[dim], hi[dim])})

    raw = []
    toggle = _with(k, spec_on=1 - k["spec_on"])
    if space["stencil"] == 0:
        for dim in ("conc", "max_num_seqs", "draft_len"):
            raw += [moved(dim, -1), moved(dim, +1)]
        raw.append(toggle)
    elif space["stencil"] == 1:        # W, k, B, max_wait
        for dim in ("draft_width", "draft_len", "max_num_seqs", "max_wait_us"):
            raw += [moved(dim, -1), moved(dim, +1)]
    elif space["stencil"] == 2:        # wide-32 (R21)
        for dc, db, dg in itertools.product((-1, 0, 1), repeat=3):
            if dc == db == dg == 0:
                continue
            raw.append(_with(k, conc=_clamp(k["conc"] + dc * st["conc"], lo["conc"], hi["conc"]),
                             max_num_seqs=_clamp(k["max_num_seqs"] + db * st["max_num_seqs"],
                                                 lo["max_num_seqs"], hi["max_num_seqs"]),
                             draft_len=_clamp(k["draft_len"] + dg * st["draft_len"],
                                              lo["draft_len"], hi["draft_len"])))
        raw += [moved("draft_width", -1), moved("draft_width", +1),
                moved("max_wait_us", -1), moved("max_wait_us", +1), toggle]
    else:
        raise ValueError("unknown stencil")
    out: List[Dict] = []
    for c in raw:
        if c == k or c in out:
            continue
        out.append(c)
    return out


def decide_move(s0: int, p99_violated: bool, s_star: int, delta_micro: int) -> bool:
    """Alg. 1: S(K*) - S(K) >= delta  OR  (p99(K) > SLO AND S(K*) > S(K))."""
    return (s_star - s0 >= delta_micro) or (p99_violated and s_star > s0)


def step(state: Dict, cands: Sequence[Dict], aggs: Sequence[Dict], sp: Dict) -> Tuple[Dict, bool, int, List[int]]:
    """One Alg. 1 iteration given measured candidates [K, neighbours...] (cands[0] == state['K']).

    Returns (new_state, moved, argmax_index, scores)."""
    st = dict(state)
    beta = sp.get("ema_beta_q16", 0)
    ema = None
    a0 = aggs[0]
    if beta and a0["n_seeds"] > 0 and not (a0["flags"] & 1):
        ema = ema_update(st.get("ema") if st.get("has_ema") else None, a0["sum_p99_us"] // a0["n_seeds"], beta)
        st["ema"], st["has_ema"] = ema, 1
    scores = [score_micro(a, c, sp, ema if i == 0 else None) for i, (a, c) in enumerate(zip(aggs, cands))]
    s0 = scores[0]
    if not st["has_best"] or s0 > st["S_best"]:
        st["S_best"], st["K_best"], st["has_best"] = s0, cands[0], 1
    moved, idx = False, 0
    if len(cands) > 1:
        idx = max(range(1, len(cands)), key=lambda i: (scores[i], -i))
        if ema is not None:
            violated = ema > sp["slo_us"]
        else:
            violated = a0["n_seeds"] > 0 and a0["sum_p99_us"] > a0["n_seeds"] * sp["slo_us"]
        moved = decide_move(s0, violated, scores[idx], sp["delta_micro"])
        if not sp["strict_alg1"] and scores[idx] > st["S_best"]:
            st["S_best"], st["K_best"] = scores[idx], cands[idx]
    st["K"] = cands[idx] if moved else cands[0]
    st["step"] = st["step"] + 1
    return st, moved, idx, scores


def initial_state(k0: Dict) -> Dict:
    return dict(K=dict(k0), K_best=dict(k0), S_best=INT64_MIN, step=0, has_best=0, ema=0, has_ema=0)
