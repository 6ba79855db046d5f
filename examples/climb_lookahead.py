"""The C4 hill-climb (Alg. 1) on one GPU three ways — the plain device climb, the lookahead
climb (two steps per round, cached records; same trajectory) and the final re-run of K_best on fresh seeds
 — then the p99 of a few caller-provided latency rows through the same select kernel (slo_select_rows).
usage: python examples/climb_lookahead.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_2603_11340_b200 import inputs, sim  # noqa: E402
from paper_2603_11340_b200._lib import AGG_DTYPE, CLIMB_DTYPE  # noqa: E402
from paper_2603_11340_b200.dist import ClimbGraph, LookaheadClimbGraph, final_rerun  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
cfg = inputs.config_c4(n_seeds=32, segment_len=2000)
s = sim.Simulator(cfg.workloads, device=0)
plain = ClimbGraph(s, cfg, cfg.seeds()).capture()
plain.run(steps)
look = LookaheadClimbGraph(s, cfg, cfg.seeds()).capture()
look.run(steps // 2)
torch.cuda.synchronize()
assert torch.equal(plain.state, look.state), "the two climbs must agree"
st = sim.unpack(look.state, CLIMB_DTYPE)[0]
print("after", int(st["step"]), "steps: K =", sim.unpack_knobs(st["K"].reshape(1))[0])
print("best:", sim.unpack_knobs(st["K_best"].reshape(1))[0], "score (micro-rps):", int(st["S_best_micro"]))
fin = final_rerun(s, cfg, look.state, inputs.seeds(64, 50_000))
agg = sim.unpack(fin["agg"], AGG_DTYPE)[0]
print("final re-run on 64 fresh seeds: mean p99", int(agg["sum_p99_us"]) // int(agg["n_seeds"]), "us, goodput",
      round(int(agg["sum_slo_met"]) * 1e6 / int(agg["sum_window_us"]), 3), "req/s")
rows = torch.randint(0, 3_000_000, (4, 1000), dtype=torch.int32, device="cuda")
print("p99 of 4 random rows:", s.select_rows(rows)["p99_us"].tolist(),
      "(sorted-row check:", [int(r.sort().values[989]) for r in rows.cpu()], ")")
plain.close()
look.close()
s.close()
