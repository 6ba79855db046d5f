"""Randomised parity soak: `python tests/soak_parity.py BLOCKS` runs BLOCKS random blocks (20 knob records x 2
seeds each) across lane-group policies, static/continuous batching, arrival kinds (kind-4 think-time loops included), warmup and the stop rule,
and compares every latency and output with the oracle (test infrastructure: it imports oracle/)."""
import os, random, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2603_11340_b200 import inputs, sim
from paper_2603_11340_b200._lib import RESULT_DTYPE
oracle.build()
c = inputs.continuous
wls = [inputs.preset_ll(), inputs.preset_sim(), inputs.preset_stress(kind=1), inputs.preset_stress(kind=2),
       inputs.preset_ll(rate=40.0, stream_id=7), inputs.preset_closed(stream_id=3),
       c(inputs.preset_ll()), c(inputs.preset_sim()), c(inputs.preset_stress(kind=1)), c(inputs.preset_closed(stream_id=4)),
       c(inputs.workload(kind=0, rate=200.0, timing=dict(inputs.LL_TIMING, noise_step_ppm=0), stream_id=5)),
       inputs.preset_closed(stream_id=11, think_us=200_000), inputs.preset_closed(stream_id=12, think_us=0),
       inputs.preset_closed(stream_id=13, think_us=3_000), c(inputs.preset_closed(stream_id=14, think_us=150_000)),
       c(inputs.preset_closed(stream_id=15, think_us=2_000))]
bad = 0
total = 0
for block in range(int(sys.argv[1]) if len(sys.argv) > 1 else 40):
    rng = random.Random(10_000 + block)
    pol = rng.choice([0, 1, 2, 3])
    s = sim.Simulator(wls, device=0, group_policy=pol)
    ks = [inputs.random_knobs(rng, n_wl=len(wls)) for _ in range(20)]
    seeds = inputs.seeds(2, 31 * block + 7)
    N = rng.choice([1, 17, 64, 333, 900])
    warm = rng.choice([0, 0, 5, 50])
    stop = rng.choice([(0, 0), (0, 0), (max(1, N // 3), 0), (1, 2_000_000), (N, 10**9)])
    out = s.run_batch(sim.knobs_tensor(ks), sim.seeds_tensor(seeds), N, warmup_len=warm, latencies=True,
                      percentiles=True, stop_n_min=stop[0], stop_t_min_us=stop[1])
    torch.cuda.synchronize()
    lat = out["latencies"].cpu().numpy().view(np.uint32).reshape(-1, N + warm)
    det = sim.unpack(out["detail"], RESULT_DTYPE)
    p99 = out["p99_us"].cpu().numpy().view(np.uint32)
    gp = out["goodput"].cpu().numpy()
    for ci, k in enumerate(ks):
        for si, sd in enumerate(seeds):
            r = ci * 2 + si
            total += 1
            if not oracle.knobs_valid(k, len(wls)):
                ok = p99[r] == 0xFFFFFFFF and gp[r] == -1.0
            else:
                ref = oracle.run(wls, k, sd, N, warmup_len=warm, latencies=True, stop_n_min=stop[0], stop_t_min_us=stop[1])
                ok = (np.array_equal(lat[r], ref["latencies"]) and int(p99[r]) == ref["p99_us"] and gp[r] == ref["goodput"]
                      and all(int(det[r][f]) == ref[f] for f in ("slo_met", "n_measured", "window_us", "sum_latency_us", "flags")))
            if not ok:
                bad += 1
                print("MISMATCH block", block, "policy", pol, "N", N, "warm", warm, "stop", stop, "knobs", k, "seed", sd)
    s.close()
print(f"soak: {total} replicas, {bad} mismatches")
