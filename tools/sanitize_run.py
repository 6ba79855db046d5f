"""Tiny run of every kernel (K0, K1g, K1s incl. its scans, K1, K1t and K1c in all lane-group modes, K1b at every
block size and on caller rows, K2, K2b, K3, the lookahead climb's K3L) for compute-sanitizer."""
import random
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2603_11340_b200 import inputs, sim  # noqa: E402

rng = random.Random(3)
wls = [inputs.preset_ll(), inputs.preset_sim(), inputs.preset_stress(kind=1), inputs.preset_stress(kind=2)]
wls += [inputs.continuous(w) for w in wls] + [inputs.continuous(inputs.preset_closed())]   # K1c
wls += [inputs.preset_closed(think_us=20_000), inputs.preset_closed(think_us=0)]          # K1t (kind 4, §2.11)
wls += [inputs.continuous(inputs.preset_closed(think_us=20_000))]                          # K1c, THINK
ks = [inputs.random_knobs(rng, n_wl=len(wls)) for _ in range(24)] + [inputs.knobs(conc=0)]
ks += [inputs.knobs(max_num_seqs=b, conc=c, workload=w, draft_len=4, spec_on=1) for b, c, w in
       ((4, 12, 4), (12, 3, 5), (32, 32, 6), (8, 8, 8), (32, 32, 9), (3, 5, 10), (12, 6, 9), (6, 20, 11),
                      (32, 32, 11))]
# min(C, B) = 1 (the K1s / K1e max-plus scans) and <= 4 (G = 4 groups), static and continuous
ks += [inputs.knobs(max_num_seqs=b, conc=c, workload=w, draft_len=3, spec_on=1, max_wait_us=mw) for b, c, w, mw in
       ((1, 9, 0, 0), (7, 1, 0, 20_000), (1, 1, 2, 0), (3, 4, 0, 0), (1, 5, 4, 0), (6, 1, 6, 0), (4, 2, 5, 0))]
for pol, gen in ((1, 2), (2, 2), (1, 1)):   # narrow / wide lane groups, split (K1g + K1s / K1c) / inline K1
    sp = sim.Simulator(wls, device=0, group_policy=pol, gen_policy=gen)
    sp.run_batch(sim.knobs_tensor(ks), sim.seeds_tensor(inputs.seeds(3)), 150, warmup_len=10, latencies=True,
                 stats=True)
    torch.cuda.synchronize()
    sp.close()
s = sim.Simulator(wls, device=0)
out = s.run_batch(sim.knobs_tensor(ks), sim.seeds_tensor(inputs.seeds(3)), 150, warmup_len=10, latencies=True,
                  stats=True)
s.run_batch(sim.knobs_tensor(ks), sim.seeds_tensor(inputs.seeds(3)), 150, warmup_len=10, latencies=True,
            percentiles=True, stop_n_min=40, stop_t_min_us=500_000)                # stop-rule kernels (§2.14)
agg0 = s.aggregate(out["detail"], len(ks), 3)
s.pareto_front(agg0, count=True)                                                    # K5
agg = s.aggregate(out["detail"], len(ks), 3)
red = s.aggregate_reduce(torch.cat([agg, agg]), 2, len(ks))
cfg = inputs.config_c4(n_seeds=2, segment_len=100)
cands = s.candidates(cfg.extra["space"], cfg.knobs[0], 32)
st = s.climb_state(cfg.knobs[0])
o2 = s.run_batch(cands, sim.seeds_tensor(cfg.seeds()), 100)
a2 = s.aggregate(o2["detail"], 32, 2)
s.hillclimb_step(cfg.extra["space"], cfg.extra["score"], cands, a2, 1, st)
torch.cuda.synchronize()
# K1b on caller rows: 64 / 128 / 256-thread blocks (row lengths 700 / 3000 / 5000; more rows than SMs), and a
# bucket above the shared-memory capacity
for n, R in ((700, 300), (3000, 200), (5000, 160)):
    g = torch.Generator().manual_seed(n)
    rows = torch.randint(0, 1 << 22, (R, n), generator=g, dtype=torch.int64)
    rows[: R // 2, : n // 2] = 1_000_000
    s.select_rows(rows.to(torch.int32).cuda(), percentiles=True)
torch.cuda.synchronize()
# the lookahead climb: prepare (U(K), cache lookup) -> simulate -> aggregate -> two steps, twice (cache hits)
table = torch.zeros(34576, dtype=torch.uint8, device="cuda")
sim_list = torch.zeros((320, 32), dtype=torch.uint8, device="cuda")
traj = torch.empty((2, 104), dtype=torch.uint8, device="cuda")
st2 = s.climb_state(cfg.knobs[0])
for _ in range(2):
    s.lookahead_prepare(cfg.extra["space"], st2, table, sim_list)
    o3 = s.run_batch(sim_list, sim.seeds_tensor(cfg.seeds()), 100)
    a3 = s.aggregate(o3["detail"], 320, 2)
    s.lookahead_step(cfg.extra["space"], cfg.extra["score"], table, a3, 1, 32, st2, traj)
torch.cuda.synchronize()
print("sanitize run ok")
