"""Full-size parity at BASELINE sizes, in the launch configuration bench.py times, and round-2 guards.

* C4 (BASELINE config 4): two whole climb steps — 32 candidates (wide-32 stencil) x 128 seeds x 5,000-request
  segments = 4,096 replicas per step — replayed through dist.ClimbGraph exactly as `bench.py --workload c4`
  runs them; every replica's (p99, slo_met, n_measured, flags, window, Σℓ) and goodput, every per-config
  aggregate, the K3 scores, argmax, move, best-so-far and next candidates equal the oracle's (oracle replicas in
  a process pool, oracle/climb.py for the step).
* W > 1 in the timing (R28) through full-size replicas of a W sweep.
* The stop rule refuses workloads that allow zero-duration batches; a handle whose scratch a captured graph
  holds refuses to regrow it.
"""
import multiprocessing as mp

import numpy as np
import pytest

from paper_2603_11340_b200 import inputs

pytestmark = pytest.mark.gpu


def _orc_task(args):
    import oracle
    wls, k, seed, n = args
    return oracle.run(wls, k, seed, n)


def _oracle_many(tasks):
    ctx = mp.get_context("spawn")
    with ctx.Pool() as pool:
        return pool.map(_orc_task, tasks, chunksize=16)


def test_c4_full_size_two_steps(orc):
    import torch
    from oracle import climb
    from paper_2603_11340_b200 import sim as S
    from paper_2603_11340_b200._lib import CLIMB_DTYPE, RESULT_DTYPE
    from paper_2603_11340_b200.dist import ClimbGraph
    cfg = inputs.config_c4()
    assert (cfg.extra["n_cand"], cfg.n_seeds, cfg.segment_len) == (32, 128, 5000)
    space, sp = cfg.extra["space"], cfg.extra["score"]
    seeds = cfg.seeds()
    s = S.Simulator(cfg.workloads, device=0)
    g = ClimbGraph(s, cfg, seeds, n_cand=32).capture()
    K = dict(cfg.knobs[0])
    ost = climb.initial_state(K)
    ocands = [K] + climb.neighbours(space, K)
    ocands += [inputs.PAD_KNOBS] * (32 - len(ocands))
    for step in range(2):
        n_valid = sum(1 for c in ocands if c["conc"] > 0)          # padding: invalid records (no work)
        assert S.unpack_knobs(g.cands.cpu().numpy())[:n_valid] == ocands[:n_valid]
        g.graph.replay()
        torch.cuda.synchronize()
        det = S.unpack(g.out["detail"], RESULT_DTYPE)
        gp = g.out["goodput"].cpu().numpy()
        refs = _oracle_many([(cfg.workloads, c, sd, cfg.segment_len) for c in ocands for sd in seeds])
        for r, ref in enumerate(refs):
            d = det[r]
            got = (int(d["p99_us"]), int(d["slo_met"]), int(d["n_measured"]), int(d["flags"]), int(d["window_us"]),
                   int(d["sum_latency_us"]))
            exp = (ref["p99_us"], ref["slo_met"], ref["n_measured"], ref["flags"], ref["window_us"],
                   ref["sum_latency_us"])
            assert got == exp, f"step {step} replica {r} knobs {ocands[r // len(seeds)]}"
            assert gp[r] == ref["goodput"], (step, r)
        oaggs = [climb.aggregate(refs[c * len(seeds):(c + 1) * len(seeds)]) for c in range(32)]
        ost, moved, idx, oscores = climb.step(ost, ocands, oaggs, sp)
        assert g.scores.cpu().tolist() == oscores, step
        st = S.unpack(g.state, CLIMB_DTYPE)[0]
        assert int(st["moved"]) == int(moved) and int(st["argmax"]) == idx
        assert S.unpack_knobs(st["K"])[0] == ost["K"]
        assert int(st["S_best_micro"]) == ost["S_best"]
        ocands = [ost["K"]] + climb.neighbours(space, ost["K"])
        ocands += [inputs.PAD_KNOBS] * (32 - len(ocands))
    g.close()
    s.close()


def test_width_sweep_full_size_sampled(orc):
    """A C3-style sweep over W = 1..4 (γ ∈ {4, 8}, α ∈ {.3, .5, .7}) at C3's 10k-request segments: sampled
    replicas equal the oracle, and the per-config seed means show the P:232 trend the oracle pins."""
    import torch
    from paper_2603_11340_b200 import sim as S
    from paper_2603_11340_b200._lib import RESULT_DTYPE
    wls = [inputs.preset_ll(), inputs.preset_stress(kind=1)]
    ks = [inputs.knobs(conc=8, max_num_seqs=8, draft_len=g, spec_on=1, accept_q16=inputs.q16(a), draft_width=W,
                       workload=w)
          for w in (0, 1) for g in (4, 8) for a in (0.3, 0.5, 0.7) for W in (1, 2, 3, 4)]
    seeds = inputs.seeds(16, 4000)
    N = 10_000
    s = S.Simulator(wls, device=0)
    out = s.run_batch(S.knobs_tensor(ks), S.seeds_tensor(seeds), N)
    torch.cuda.synchronize()
    det = S.unpack(out["detail"], RESULT_DTYPE)
    gp = out["goodput"].cpu().numpy()
    rng = np.random.default_rng(5)
    sample = sorted(set(rng.choice(len(ks) * len(seeds), 96, replace=False).tolist()) | {0, len(ks) * len(seeds) - 1})
    refs = _oracle_many([(wls, ks[r // len(seeds)], seeds[r % len(seeds)], N) for r in sample])
    for r, ref in zip(sample, refs):
        assert (int(det[r]["p99_us"]), int(det[r]["slo_met"]), int(det[r]["window_us"])) == \
            (ref["p99_us"], ref["slo_met"], ref["window_us"]), r
        assert gp[r] == ref["goodput"]
    s.close()


def test_stop_rule_refuses_zero_duration_timing():
    import torch
    from paper_2603_11340_b200 import sim as S
    from paper_2603_11340_b200._lib import SloError
    w = inputs.preset_ll()
    w["timing"] = dict(w["timing"], pre_base_us=0, pre_tok_us=1)    # a 1-token prefill can floor to 0 us
    s = S.Simulator([w], device=0)
    ks = S.knobs_tensor([inputs.knobs()])
    sd = S.seeds_tensor(inputs.seeds(1))
    with pytest.raises(SloError):
        s.run_batch(ks, sd, 100, stop_n_min=10)
    s.run_batch(ks, sd, 100)                                        # without a stop rule it runs
    torch.cuda.synchronize()
    s.close()


def test_captured_handle_refuses_regrow():
    import torch
    from paper_2603_11340_b200 import sim as S
    from paper_2603_11340_b200._lib import SloError
    cfg = inputs.config_c4(n_seeds=4, segment_len=400)
    s = S.Simulator(cfg.workloads, device=0)
    ks = S.knobs_tensor(cfg.knobs * 8)
    sd = S.seeds_tensor(cfg.seeds())
    out = s.run_batch(ks, sd, 400)
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        s.run_batch(ks, sd, 400, out=out, stream=st)
    graph.replay()
    torch.cuda.synchronize()
    big = S.seeds_tensor(inputs.seeds(4096))
    with pytest.raises(SloError):                                   # would free the graph's scratch
        s.run_batch(ks, big, 4000)
    graph.replay()                                                  # the graph still runs on intact scratch
    torch.cuda.synchronize()
    s.close()
