"""Tiny run of every kernel (K0, K1 in all three lane-group modes, K1b, K2, K2b, K3) for compute-sanitizer."""
import random
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2603_11340_b200 import inputs, sim  # noqa: E402

rng = random.Random(3)
wls = [inputs.preset_ll(), inputs.preset_sim(), inputs.preset_stress(kind=1), inputs.preset_stress(kind=2)]
ks = [inputs.random_knobs(rng, n_wl=len(wls)) for _ in range(12)] + [inputs.knobs(conc=0)]
s = sim.Simulator(wls, device=0)
out = s.run_batch(sim.knobs_tensor(ks), sim.seeds_tensor(inputs.seeds(3)), 150, warmup_len=10, latencies=True,
                  stats=True)
agg = s.aggregate(out["detail"], len(ks), 3)
red = s.aggregate_reduce(torch.cat([agg, agg]), 2, len(ks))
cfg = inputs.config_c4(n_seeds=2, segment_len=100)
cands = s.candidates(cfg.extra["space"], cfg.knobs[0], 32)
st = s.climb_state(cfg.knobs[0])
o2 = s.run_batch(cands, sim.seeds_tensor(cfg.seeds()), 100)
a2 = s.aggregate(o2["detail"], 32, 2)
s.hillclimb_step(cfg.extra["space"], cfg.extra["score"], cands, a2, 1, st)
torch.cuda.synchronize()
print("sanitize run ok")
