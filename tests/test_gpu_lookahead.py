"""Lookahead climb (SV §8(f) NEXT-4; slo_lookahead_prepare / slo_lookahead_step, dist.LookaheadClimbGraph): two
Alg. 1 steps per round from U(K) = {K} u N(K) u N(N(K)), records measured last round taken from the cache.
Its trajectory must equal the plain device climb's (dist.ClimbGraph, itself checked step by step against
oracle/climb.py in test_gpu_parity.py) bit for bit: every field of the climb state after every step."""
import dataclasses

import numpy as np

import pytest
import torch

from paper_2603_11340_b200 import inputs, sim

pytestmark = pytest.mark.gpu

VARIANTS = {"live-wide32": (inputs.SPACE_WIDE32, dict(inputs.SCORE_DEFAULTS)),
            "sim-controller": (inputs.SPACE_WIDE32, dict(inputs.SCORE_SIM)),
            "sim-space": (inputs.SPACE_SIM, dict(inputs.SCORE_SIM, strict_alg1=0)),
            "live-stencil": (inputs.SPACE_LIVE, dict(inputs.SCORE_DEFAULTS, delta_micro=0))}


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_lookahead_trajectory_equals_plain_climb(variant):
    from paper_2603_11340_b200.dist import ClimbGraph, LookaheadClimbGraph
    space, sp = VARIANTS[variant]
    cfg = inputs.config_c4(n_seeds=4, segment_len=400)
    cfg = dataclasses.replace(cfg, extra=dict(cfg.extra, space=space, score=sp))
    seeds = inputs.seeds(4, 77)
    s = sim.Simulator(cfg.workloads, device=0)
    rounds = 6
    g = ClimbGraph(s, cfg, seeds, n_cand=32).capture()
    nb = g.state.numel()
    h_traj = torch.empty((2 * rounds, nb), dtype=torch.uint8).pin_memory()
    g.run_host(2 * rounds, g.init_cands.cpu().pin_memory(), g.init_state.cpu().pin_memory(), h_traj)
    la = LookaheadClimbGraph(s, cfg, seeds, n_cand=32).capture()
    got = la.states(rounds)
    assert torch.equal(got, h_traj), variant
    # the cache: a later round simulates only what the previous round's table lacks
    assert 0 <= la.simulated() <= la.CAP
    g.close()
    la.close()
    s.close()


def test_lookahead_cache_converged_climb_simulates_nothing():
    """Once K stops moving, U(K) is the previous round's table: a round simulates no record at all and the
    trajectory still matches the plain climb."""
    from paper_2603_11340_b200.dist import LookaheadClimbGraph
    cfg = inputs.config_c4(n_seeds=2, segment_len=300)
    sp = dict(inputs.SCORE_DEFAULTS, delta_micro=10**15, slo_us=4_000_000_000)   # never moves, never violated
    cfg = dataclasses.replace(cfg, extra=dict(cfg.extra, score=sp))
    s = sim.Simulator(cfg.workloads, device=0)
    la = LookaheadClimbGraph(s, cfg, inputs.seeds(2, 5), n_cand=32).capture()
    la.run(1)
    torch.cuda.synchronize()
    first = la.simulated()
    la.run(1)
    torch.cuda.synchronize()
    assert first > 32 and la.simulated() == 0
    la.close()
    s.close()


def test_final_rerun_of_k_best_matches_oracle():
    """Alg. 1's final re-run of K_best on a fresh seed block, read from the device climb state, equals the
    oracle's replicas of the same record on the same seeds."""
    import oracle
    from paper_2603_11340_b200._lib import CLIMB_DTYPE
    from paper_2603_11340_b200.dist import LookaheadClimbGraph, final_rerun
    cfg = inputs.config_c4(n_seeds=3, segment_len=300)
    s = sim.Simulator(cfg.workloads, device=0)
    la = LookaheadClimbGraph(s, cfg, inputs.seeds(3, 21), n_cand=32).capture()
    la.run(3)
    fresh = inputs.seeds(4, 900)
    out = final_rerun(s, cfg, la.state, fresh)
    torch.cuda.synchronize()
    kb = sim.unpack_knobs(sim.unpack(la.state, CLIMB_DTYPE)[0]["K_best"].reshape(1))[0]
    oracle.build()
    exp = [oracle.run(cfg.workloads, kb, sd, cfg.segment_len, warmup_len=cfg.warmup_len, slo_us=cfg.slo_us)
           for sd in fresh]
    got_p99 = out["p99_us"].cpu().tolist()
    assert got_p99 == [e["p99_us"] for e in exp]
    gp = out["goodput"].cpu().tolist()
    assert gp == [e["goodput"] for e in exp]
    la.close()
    s.close()


def test_live_configs_skip_padding():
    """slo_run_args.d_live_configs: configs [0, L) give exactly a plain run's outputs, later configs' outputs are
    not touched and their replicas are not counted (static, continuous and mixed knobs)."""
    import random
    from paper_2603_11340_b200._lib import STATS_DTYPE
    rng = random.Random(8)
    wls = [inputs.preset_ll(), inputs.continuous(inputs.preset_ll()), inputs.preset_stress(kind=1)]
    ks = [inputs.random_knobs(rng, n_wl=len(wls)) for _ in range(20)]
    seeds = inputs.seeds(3, 4)
    s = sim.Simulator(wls, device=0)
    dev = torch.device("cuda", 0)
    kt, st = sim.knobs_tensor(ks, device=dev), sim.seeds_tensor(seeds, device=dev)
    for L in (0, 1, 7, 20):
        live = torch.tensor([L], dtype=torch.int32, device=dev)
        out = s.alloc_outputs(len(ks) * 3, stats=True)
        out["p99_us"].fill_(-7)
        out["goodput"].fill_(-7.0)
        s.run_batch(kt, st, 400, warmup_len=20, out=out, live_configs_ptr=live.data_ptr(), stats=True)
        ref = s.run_batch(kt[:max(L, 1)], st, 400, warmup_len=20, stats=True)
        torch.cuda.synchronize()
        n = 3 * L
        assert torch.equal(out["p99_us"][:n], ref["p99_us"][:n]) and torch.equal(out["goodput"][:n], ref["goodput"][:n])
        assert bool((out["p99_us"][n:] == -7).all()) and bool((out["goodput"][n:] == -7.0).all())
        req = int(sim.unpack(out["stats"], STATS_DTYPE)[0]["requests"])
        assert req == n * 420, (L, req)
    s.close()


def test_lookahead_seed_sharded_two_ranks(tmp_path):
    """Two ranks (gloo, sharing the box's GPU) each simulate half of the seeds of every round's records; the
    all-gathered parts summed by K3L-step give every step's state bit for bit equal to one process over all
    seeds (integer sums: the pooled aggregates do not depend on the split)."""
    import json
    import os
    import subprocess
    import sys
    from paper_2603_11340_b200.dist import LookaheadClimbGraph
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    rounds, out = 3, tmp_path / "la.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29541", os.path.join(root, "tests", "lookahead_worker.py"),
           str(out), str(rounds)]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=420)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    got = json.load(open(out))["states"]
    cfg = inputs.config_c4(n_seeds=8, segment_len=400)
    s = sim.Simulator(cfg.workloads, device=0)
    la = LookaheadClimbGraph(s, cfg, cfg.seeds(), n_cand=32).capture()
    ref = la.states(rounds)
    assert [ref[i].numpy().tobytes().hex() for i in range(ref.shape[0])] == got
    la.close()
    s.close()


def test_device_neighbour_lists_equal_host_rule():
    """K3's warp-parallel neighbour generation (neighbors_warp) writes the same [K, neighbours(K), padding] list as
    the host rule (slo_neighbors, and oracle/climb.py's neighbours: P:142, R21) for random and boundary K
    on every stencil: a step whose aggregates are all invalid does not move, so it rewrites the list around K."""
    import random
    from oracle import climb
    rng = random.Random(17)
    s = sim.Simulator([inputs.preset_ll()], device=0)
    dev = torch.device("cuda", 0)
    for space in (inputs.SPACE_LIVE, inputs.SPACE_SIM, inputs.SPACE_WIDE32):
        for trial in range(40):
            lo, hi = space["lo"], space["hi"]
            pick = (lambda d: rng.choice([lo[d], hi[d], rng.randrange(lo[d], hi[d] + 1)]))
            K = inputs.knobs(conc=pick(0), max_num_seqs=pick(1), draft_len=pick(2), spec_on=rng.randrange(2),
                             draft_width=pick(3), max_wait_us=pick(4))
            cands = sim.knobs_tensor([K] + [inputs.PAD_KNOBS] * 31, device=dev)
            aggs = torch.zeros((32, 32), dtype=torch.uint8, device=dev)           # n_seeds = 0: invalid
            st = s.climb_state(K)
            s.hillclimb_step(space, dict(inputs.SCORE_DEFAULTS), cands, aggs, 1, st)
            torch.cuda.synchronize()
            got = sim.unpack_knobs(cands.cpu().numpy().view(np.uint8).view(sim._lib.KNOB_DTYPE))
            exp = [K] + climb.neighbours(space, K)
            assert got[:len(exp)] == exp, (space["stencil"], K)
            assert all(k["conc"] == 0 for k in got[len(exp):])          # padding: invalid records
    s.close()
