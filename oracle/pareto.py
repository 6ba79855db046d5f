"""oracle.pareto — TEST INFRASTRUCTURE ONLY.

The Pareto front of a sweep ("The resulting Pareto front in the steady regime", Fig. 2-4;
SPEC S:521 `pareto_front(rows, objectives: maximize goodput, minimize p99)`), written from DESIGN.md §2.13
as the plain O(n^2) definition:

* objectives of a config from its aggregate over seeds (§2.9): mean p99 = floor(sum_p99 / n) us, and
  goodput = floor(sum_slo_met * 10^12 / sum_window) micro-requests/s (the score's goodput term, Eq. 1 pooled);
* a config with an invalid seed (flags bit 0) or no seeds is never on the front;
* config j dominates i iff p_j <= p_i and g_j >= g_i with at least one strict; i is on the front iff it is
  valid and no valid j dominates it (equal points do not dominate each other).
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple


def objectives(agg: Dict) -> Tuple[bool, int, int]:
    n = agg["n_seeds"]
    if n == 0 or agg["flags"] & 1 or agg["sum_window_us"] == 0:
        return False, 0, 0
    return True, agg["sum_p99_us"] // n, agg["sum_slo_met"] * 10**12 // agg["sum_window_us"]


def dominates(pj: int, gj: int, pi: int, gi: int) -> bool:
    return pj <= pi and gj >= gi and (pj < pi or gj > gi)


def pareto_front(aggs: Sequence[Dict]) -> List[bool]:
    obj = [objectives(a) for a in aggs]
    front = []
    for i, (vi, pi, gi) in enumerate(obj):
        front.append(vi and not any(vj and dominates(pj, gj, pi, gi) for j, (vj, pj, gj) in enumerate(obj)
                                    if j != i))
    return front
