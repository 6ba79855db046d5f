"""Time K1c on subsets of the C2-cont grid (by concurrency) to see whether the step is bound by throughput
or by the longest replica chains."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2603_11340_b200 import inputs, sim

cfg = inputs.config_c2_cont()
S = sim.Simulator(cfg.workloads, device=0)
seeds = sim.seeds_tensor(cfg.seeds(), device=torch.device("cuda", 0))


def t(ks, reps=2):
    kt = sim.knobs_tensor(ks, device=torch.device("cuda", 0))
    out = S.alloc_outputs(len(ks) * cfg.n_seeds)
    S.run_batch(kt, seeds, cfg.segment_len, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        S.run_batch(kt, seeds, cfg.segment_len, out=out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


print("all", round(t(cfg.knobs), 1))
for cs in ([1], [2], [3, 4], list(range(5, 9)), list(range(9, 17))):
    ks = [k for k in cfg.knobs if k["conc"] in cs]
    print("C in", cs, len(ks), "configs", round(t(ks), 1), "ms")
ks = [k for k in cfg.knobs if k["conc"] >= 3]
print("C >= 3", len(ks), round(t(ks), 1))
