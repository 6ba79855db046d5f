"""Pins of oracle/pareto.py."""
import random

from oracle import pareto


def _agg(p99, gp_rps, n=1, flags=0):
    # sum_window 10^6 us and slo_met = gp_rps make goodput exactly gp_rps * 10^6 micro-rps
    return dict(sum_p99_us=p99 * n, sum_slo_met=gp_rps * n, sum_window_us=10**6 * n, n_seeds=n, flags=flags)


def test_hand_example():
    """Minimise p99, maximise goodput: (1,1) twice (equal points do not dominate each other), (2,2) and (3,3)
    are on the front; (2,1) is dominated by (1,1); (3,2) by (2,2); the invalid record never is."""
    pts = [(1, 1), (2, 2), (2, 1), (3, 3), (1, 1), (3, 2), (0, 9)]
    aggs = [_agg(p, g) for p, g in pts]
    aggs[6]["flags"] = 1
    assert pareto.pareto_front(aggs) == [True, True, False, True, True, False, False]


def test_objectives_are_the_score_terms():
    a = dict(sum_p99_us=1_000_001, sum_slo_met=7, sum_window_us=3_000_000, n_seeds=2, flags=0)
    assert pareto.objectives(a) == (True, 500_000, 2_333_333)          # floors, micro-rps
    assert pareto.objectives(dict(a, n_seeds=0))[0] is False


def test_front_properties_random():
    """Properties any correct front has, checked against the definition: sorted by p99 the front's goodput
    strictly increases (unless points are equal), every valid point off the front is dominated by a point
    on it, and the front of the front is itself."""
    rng = random.Random(3)
    for _ in range(30):
        n = rng.randrange(1, 80)
        aggs = [_agg(rng.randrange(0, 12), rng.randrange(0, 12), n=rng.randrange(1, 4),
                     flags=1 if rng.random() < 0.05 else 0) for _ in range(n)]
        f = pareto.pareto_front(aggs)
        obj = [pareto.objectives(a) for a in aggs]
        on = sorted({(obj[i][1], obj[i][2]) for i in range(n) if f[i]})
        for (p1, g1), (p2, g2) in zip(on, on[1:]):
            assert p1 < p2 and g1 < g2
        for i in range(n):
            if obj[i][0] and not f[i]:
                assert any(f[j] and pareto.dominates(obj[j][1], obj[j][2], obj[i][1], obj[i][2]) for j in range(n))
        sub = [aggs[i] for i in range(n) if f[i]]
        assert all(pareto.pareto_front(sub))
