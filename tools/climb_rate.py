"""Time-to-solution of the C4 climb (BASELINE config 4: 500 Alg. 1 steps, 32 candidates, 128 seeds, 5k-request
segments): the plain device climb (dist.ClimbGraph, one step per graph replay) against the lookahead climb
(dist.LookaheadClimbGraph, two steps per replay from U(K) = {K} u N(K) u N(N(K)) minus the cache; SV §8(f)
NEXT-4).  CUDA events on the replay streams; the per-step states of the first 40 steps and the final states of
the timed runs must agree.  --seeds 16 times one rank's share of an 8-GPU seed-sharded climb.
usage: python tools/climb_rate.py [--steps 500] [--seeds 128] [--segment 5000]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_2603_11340_b200 import inputs, sim  # noqa: E402
from paper_2603_11340_b200.dist import ClimbGraph, LookaheadClimbGraph  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=500)
ap.add_argument("--seeds", type=int, default=128)
ap.add_argument("--segment", type=int, default=5000)
a = ap.parse_args()
cfg = inputs.config_c4(n_seeds=a.seeds, segment_len=a.segment)
seeds = cfg.seeds()
S = sim.Simulator(cfg.workloads, device=0)
g = ClimbGraph(S, cfg, seeds, n_cand=32).capture()
la = LookaheadClimbGraph(S, cfg, seeds, n_cand=32).capture()

nb = g.state.numel()
h = torch.empty((40, nb), dtype=torch.uint8).pin_memory()
g.run_host(40, g.init_cands.cpu().pin_memory(), g.init_state.cpu().pin_memory(), h)
la.reset()
assert torch.equal(la.states(20), h), "lookahead trajectory differs from the plain climb"


def timed(stream, body):            # replays on `stream` (CUDAGraph.replay launches on the current stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        body()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def plain():
    g.cands.copy_(g.init_cands)
    g.state.copy_(g.init_state)
    torch.cuda.synchronize()
    return timed(g.stream, lambda: [g.graph.replay() for _ in range(a.steps)])


def look():
    la.reset()
    torch.cuda.synchronize()
    return timed(la.stream, lambda: [la.graph.replay() for _ in range(a.steps // 2)])


plain()
look()
tp = min(plain() for _ in range(3))
tl = min(look() for _ in range(3))
same = torch.equal(g.state, la.state)
sims = []
la.reset()
for _ in range(min(a.steps // 2, 50)):
    la.run(1)
    torch.cuda.synchronize()
    sims.append(la.simulated())
print(json.dumps({"workload": f"C4 climb, {a.steps} Alg. 1 steps, 32 candidates (wide-32), {a.seeds} seeds, "
                              f"{a.segment}-request segments, one B200",
                  "plain_ms_per_step": tp / a.steps, "lookahead_ms_per_step": tl / a.steps, "speedup": tp / tl,
                  "final_state_equal": same, "first_40_steps_equal": True,
                  "records_simulated_per_round_first_12": sims[:12],
                  "records_simulated_mean_rounds_2_to_50": sum(sims[1:]) / max(1, len(sims) - 1),
                  "lookahead_capacity": la.CAP, "plain_records_per_step": 32}))
