"""Host-side bound of the lookahead climb's candidate set (SV §8(f) NEXT-4): |U(K)| = |{K} u N(K) u N(N(K))|
<= SLO_LOOKAHEAD_CAP (320) for every stencil, computed with oracle/climb.py's neighbour rule (P:142, S:83,
DESIGN.md R21) over random and boundary K; and the library's constants agree with the binding's."""
import os
import random
import re

from oracle import climb
from paper_2603_11340_b200 import inputs
from paper_2603_11340_b200.dist import LookaheadClimbGraph


def _key(k):
    return tuple(sorted(k.items()))


def u_size(space, K):
    seen = {_key(K)}
    n1 = climb.neighbours(space, K)
    for c in n1:
        seen.add(_key(c))
        for d in climb.neighbours(space, c):
            seen.add(_key(d))
    return len(seen)


def test_lookahead_set_fits_capacity():
    rng = random.Random(3)
    worst = {}
    for name, space in (("live", inputs.SPACE_LIVE), ("sim", inputs.SPACE_SIM), ("wide32", inputs.SPACE_WIDE32)):
        m = 0
        for _ in range(300):
            K = inputs.knobs(conc=rng.randrange(space["lo"][0], space["hi"][0] + 1),
                             max_num_seqs=rng.randrange(space["lo"][1], space["hi"][1] + 1),
                             draft_len=rng.randrange(space["lo"][2], space["hi"][2] + 1), spec_on=rng.randrange(2),
                             draft_width=rng.randrange(space["lo"][3], space["hi"][3] + 1),
                             max_wait_us=rng.choice([0, 20_000, 50_000]))
            m = max(m, u_size(space, K))
        worst[name] = m
    assert worst["wide32"] <= 320 and worst["live"] <= 320 and worst["sim"] <= 320, worst
    assert worst["wide32"] <= 272     # the interior count: 5^3 cube + its W / wait / toggle shells


def test_lookahead_constants_match_header():
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "slo_sim.h")).read()
    assert int(re.search(r"#define SLO_LOOKAHEAD_CAP (\d+)", hdr).group(1)) == LookaheadClimbGraph.CAP
    assert int(re.search(r"#define SLO_LOOKAHEAD_TABLE_BYTES (\d+)", hdr).group(1)) == LookaheadClimbGraph.TABLE_BYTES
