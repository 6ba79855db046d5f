"""bench.py — simulated requests/s of the batched SLO-Tuner simulator on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c1|c3|c4|c5] [--impl ours|reference]

One step = one pass of the whole hot path (K1 simulate every replica -> K2 per-config
aggregation -> [N>1: NCCL all-gather of the aggregates + K2b reduce] (+ K3 climb step for c4)) over one
batch of synthetic input already resident in HBM.  Default workload = BASELINE config 2 (16 C x 8 B x 4 spec
x 64 seeds, 10k-request segments, LL preset).  N>1 (torchrun): the BASELINE config itself is partitioned
(SURVEY §8(e)): sweeps are config-sharded (config c -> rank c mod N, all of its seeds local; one NCCL
all_gather_into_tensor of the per-config aggregates), the climb is seed-sharded (aggregates all-gathered and
summed by K3) — "scaling": "strong".  `--scaling weak` instead runs the full grid on every rank with its own
seed block.  value = simulated requests (counted by the kernels, invalid padding excluded) of all ranks /
max-over-ranks device time.

`--impl reference`: the CPU oracle (oracle/, as it stands) on the host cores on a bounded sample of the
same workload — the tier's reference arm.  The oracle is otherwise only used by the cpu_baseline leg.
"""
from __future__ import annotations

import argparse
import itertools
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DESCR = {
    "c1": "C1 single replica: C=8, B=16, no speculation, Poisson 10 req/s, 2,000 requests, SLO 1.2 s",
    "c2": "C2 knob grid 16 concurrency x 8 batch limits x 4 speculation settings x 64 seeds, 10k-request segments",
    "c3": "C3 speculative sweep: draft length 0-8 x acceptance .3-.9, C=B=8, 256 seeds, 10k-request segments",
    "c4": "C4 hill-climb step: 32 candidates (wide-32 stencil) x 128 seeds, 5k-request segments",
    "c2c": "C2 knob grid (16 C x 8 B x 4 spec x 64 seeds, 10k-request segments) served with continuous "
           "(iteration-level, vLLM-style) batching, DESIGN.md 2.12",
    "c5": "C5 stress grid: MMPP-2 bursty arrivals past the knee, 10^6 configs (25 C x 25 B x 8 gamma x 5 alpha x 40 rates) x 16 seeds, 2k-request segments",
    "c5s": "C5 stress grid sample: MMPP-2 bursty arrivals, every 16th of the 10^6 configs (62,500, all knob values) x 16 seeds, 2k-request segments",
}
# Philox4x32-10 minimum integer lane-ops per block: 10 rounds x (2 widening multiplies + 2 three-input
# XORs + 2 key additions) — the irreducible algorithmic work.
OPS_PER_PHILOX_BLOCK = 60


def make_config(name):
    from paper_2603_11340_b200 import inputs
    if name == "c1":
        return inputs.config_c1()
    if name == "c2":
        return inputs.config_c2()
    if name == "c2c":
        return inputs.config_c2_cont()
    if name == "c3":
        return inputs.config_c3()
    if name == "c4":
        return inputs.config_c4()
    if name == "c5":
        return inputs.config_c5()                      # the full 10^6-config grid (BASELINE config 5)
    if name == "c5s":
        return inputs.config_c5(stride=16)             # every 16th config of the 10^6 grid: 62,500
    raise SystemExit(f"unknown workload {name}")


def peaks():
    p = {"hbm_gbs": 6458.7, "sm_max_mhz": 1965.0, "source": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            m = json.load(fh)
        p.update(hbm_gbs=m["hbm_gbs"], sm_max_mhz=m["sm_max_mhz"], source="measured")
    except Exception:
        pass
    return p


# ------------------------------------------------------------------------------------------------
# CPU oracle legs (cpu_baseline and --impl reference)
# ------------------------------------------------------------------------------------------------
def _oracle_task(args):
    wls, k, seed, n = args
    import oracle
    r = oracle.run(wls, k, seed, n)
    return n, r["p99_us"]


def cpu_oracle_sample(cfg, budget_s=12.0, seed_offset=0):
    """Run the oracle on (config, seed) replicas of cfg in a fixed seed-major order on all host cores
    until ~budget_s elapse; returns (requests/s, cores, replicas, requests, seconds)."""
    import multiprocessing as mp
    import oracle
    oracle.build()
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    seeds = cfg.seeds()
    # seed-major order, bounded: the pool's feeder queues its whole input, and a budget of seconds never
    # reaches 200k replicas (the oracle does ~3k replicas/s on 16 cores)
    tasks = list(itertools.islice(((cfg.workloads, k, seeds[s], cfg.segment_len)
                                   for s in range(cfg.n_seeds) for k in cfg.knobs), 200_000))
    ctx = mp.get_context("spawn")
    done_req = 0
    done_rep = 0
    with ctx.Pool(cores) as pool:
        pool.map(_oracle_task, [tasks[0]] * cores)          # warm the workers
        t0 = time.perf_counter()
        it = pool.imap(_oracle_task, tasks, chunksize=1)
        for n, _ in it:
            done_req += n
            done_rep += 1
            if time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - t0
        pool.terminate()
    return done_req / dt, cores, done_rep, done_req, dt


def cpu_oracle_1core(cfg, budget_s=6.0):
    """The oracle on ONE host core (this process, no pool), same replica order, ~budget_s of work."""
    import oracle
    oracle.build()
    seeds = cfg.seeds()
    done_req = done_rep = 0
    t0 = time.perf_counter()
    for s in range(cfg.n_seeds):
        for k in cfg.knobs:
            oracle.run(cfg.workloads, k, seeds[s], cfg.segment_len)
            done_req += cfg.segment_len
            done_rep += 1
            if time.perf_counter() - t0 > budget_s:
                dt = time.perf_counter() - t0
                return done_req / dt, done_rep, done_req, dt
    dt = time.perf_counter() - t0
    return done_req / dt, done_rep, done_req, dt


# ------------------------------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md clocks line)
# ------------------------------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"slo_clocks_{os.getpid()}.csv")

    def start(self):
        if os.environ.get("CUDA_INJECTION64_PATH") or os.environ.get("NV_NSIGHT_INJECTION_TRANSPORT_TYPE"):
            return          # under a profiler: never spawn nvidia-smi next to ncu's injected process
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "200"], stdout=open(self.path, "w"),
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def samples(self):
        try:
            return sum(1 for line in open(self.path) if line.count(",") >= 8)
        except OSError:
            return 0

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9 and f[1].replace(".", "").isdigit():
                rows.append(f)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows]
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            for n, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][2]), "samples": len(rows),
                "reasons": sorted(reasons)}


# ------------------------------------------------------------------------------------------------
def inputs_seeds(n, offset):
    from paper_2603_11340_b200 import inputs
    return inputs.seeds(n, offset)


def climb_time_to_solution(S, cfg, seeds, graph, steps=500):
    """BASELINE config 4 is a 500-step climb: its time with the plain device climb (ClimbGraph, one step per
    replay, every step simulates its 32 candidates) and with the lookahead climb (LookaheadClimbGraph, SV §8(f)
    NEXT-4: two steps per replay from U(K) = {K} u N(K) u N(N(K)), records measured last round cached).  CUDA
    events on the replay streams; the two must end in the same climb state."""
    import torch
    from paper_2603_11340_b200 import sim
    from paper_2603_11340_b200.dist import LookaheadClimbGraph, final_rerun
    la = LookaheadClimbGraph(S, cfg, seeds, n_cand=graph.n_cand).capture()
    fresh = inputs_seeds(len(seeds), 1_000_000)           # Alg. 1's final re-run of K_best on a fresh block

    def timed(stream, body):                             # replays and re-run all on `stream`
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            body()
            e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    fresh_t = sim.seeds_tensor(fresh, device=graph.state.device)
    res = {"plain": final_rerun(S, cfg, graph.state, fresh_t), "look": final_rerun(S, cfg, graph.state, fresh_t)}
    torch.cuda.synchronize()                              # (outputs allocated outside the timed region)
    graph.cands.copy_(graph.init_cands)
    graph.state.copy_(graph.init_state)

    def plain():
        for _ in range(steps):
            graph.graph.replay()
        final_rerun(S, cfg, graph.state, fresh_t, out=res["plain"], stream=graph.stream)
    tp = timed(graph.stream, plain)
    la.reset()
    sims = []

    def rounds():
        for _ in range(steps // 2):
            la.graph.replay()
        final_rerun(S, cfg, la.state, fresh_t, out=res["look"], stream=la.stream)
    tl = timed(la.stream, rounds)
    same = bool(torch.equal(graph.state, la.state)) and bool(torch.equal(res["plain"]["agg"], res["look"]["agg"]))
    la.reset()
    for _ in range(4):
        la.run(1)
        torch.cuda.synchronize()
        sims.append(la.simulated())
    la.close()
    return {"steps": steps, "final_rerun": f"K_best on {len(fresh)} fresh seeds (inside both timings)",
            "plain_ms": tp, "lookahead_ms": tl, "final_state_equal": same,
            "lookahead_records_simulated_rounds_1_4": sims,
            "note": "plain: 32 candidates simulated every step; lookahead: U(K) minus the cache per two steps "
                    "(a converged climb simulates nothing); not the timed metric of this line"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2", choices=sorted(DESCR))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--warps-per-block", type=int, default=0, help="launch shape override (0 = library default)")
    ap.add_argument("--blocks-per-sm", type=int, default=0)
    ap.add_argument("--group-policy", type=int, default=0, choices=[0, 1, 2, 3],
                    help="lane groups: 0 auto, 1 narrow G>=min(C,B), 2 wide G>=max(C,B), 3 whole warp")
    ap.add_argument("--gen-policy", type=int, default=0, choices=[0, 1, 2],
                    help="static batching: 0 auto, 1 inline generation in K1, 2 split K1g + K1s")
    ap.add_argument("--eager-climb", action="store_true", help="c4: host loop instead of the CUDA-graph step")
    ap.add_argument("--exchange", default="nccl", choices=["p2p", "nccl"],
                    help="N>1 aggregate exchange: nccl = K2 + all_gather_into_tensor (+ K2b / K3 summing the parts); "
                         "p2p = K2x/K2w through CUDA IPC peer windows (NEXT-4; seed-sharded climb and weak sweeps)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N>1 sweeps: strong = the BASELINE grid config-sharded over ranks (SURVEY §8(e)); "
                         "weak = every rank runs the full grid on its own seed block")
    ap.add_argument("--no-graph", action="store_true",
                    help="latency-bound sweeps (<= 4 replicas per SM): stream launches instead of a CUDA-graph replay")
    ap.add_argument("--share-of", type=int, default=1,
                    help="N=1 only: time rank 0's share of a W-GPU partition of the workload on this one GPU (no "
                         "exchange) — the per-rank step of a W-GPU run, for strong-scaling analysis")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = make_config(args.workload)

    if args.impl == "reference":
        if rank != 0:
            return
        per_step = max(3.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
        vals = []
        for s in range(args.warmup + args.steps):
            v, cores, reps, reqs, dt = cpu_oracle_sample(cfg, budget_s=per_step)
            if s >= args.warmup:
                vals.append((v, reqs, dt))
        tot_req = sum(x[1] for x in vals)
        tot_t = sum(x[2] for x in vals)
        value = tot_req / tot_t
        sample = (f"per step: the first ~{per_step:.0f} s of oracle replicas of {args.workload.upper()} "
                  f"(seed-major order), {cores} worker processes")
        print(json.dumps({
            "impl": "reference", "metric": "simulated requests/s", "value": value, "unit": "requests/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * tot_t / len(vals), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": DESCR[args.workload], "replicas_per_step_sampled": vals and int(vals[0][1] / (cfg.segment_len + cfg.warmup_len))},
            "cpu_baseline": {"value": value, "unit": "requests/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "requests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }))
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import __graft_entry__
    if rank == 0 or world == 1:
        __graft_entry__.build()
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)                  # before NCCL: one process per GPU, rank -> its own device
    if world > 1:
        # NCCL over NVLink/NVSwitch in production; SLO_BENCH_BACKEND=gloo lets several ranks share one GPU
        # to exercise this code path on a single-GPU box (never used for a reported number)
        backend = os.environ.get("SLO_BENCH_BACKEND", "nccl" if torch.cuda.is_available() else "gloo")
        dist.init_process_group(backend)
        dist.barrier()
        if rank != 0:
            __graft_entry__.build()
    from paper_2603_11340_b200 import inputs, sim
    from paper_2603_11340_b200._lib import STATS_DTYPE

    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    S = sim.Simulator(cfg.workloads, device=local, warps_per_block=args.warps_per_block,
                      blocks_per_sm=args.blocks_per_sm, group_policy=args.group_policy,
                      gen_policy=args.gen_policy)
    info = S.info()

    from paper_2603_11340_b200.dist import config_shard, seed_block, sweep_seed_offset
    strong = args.scaling == "strong" or world == 1
    knobs_local = cfg.knobs
    pworld = world if world > 1 else max(1, args.share_of)   # partition width (--share-of: rank 0 of W)
    if args.workload == "c4":
        # the climb is seed-sharded (strong scaling): the pooled aggregates equal the 1-GPU ones exactly
        lo, hi = seed_block(cfg.n_seeds, rank, pworld)
        seeds = cfg.seeds()[lo:hi]
    elif strong:
        # sweeps are config-sharded: config c -> rank c mod world, all seeds local; every rank's
        # share is padded to the same length with always-invalid records (no work) for the all-gather
        seeds = cfg.seeds()
        knobs_local = config_shard(cfg.knobs, rank, pworld, pad=inputs.PAD_KNOBS)
    else:
        # weak scaling (opt-in): every rank runs the full grid on its own seed block
        seeds = inputs.seeds(cfg.n_seeds, sweep_seed_offset(cfg.n_seeds, rank, cfg.seed_offset))
    n_seeds_local = len(seeds)
    n_cfg = len(knobs_local)
    N = cfg.segment_len + cfg.warmup_len
    seeds_t = sim.seeds_tensor(seeds, device=dev)
    if args.workload == "c4":
        space, sp = cfg.extra["space"], cfg.extra["score"]
        n_cfg = cfg.extra["n_cand"]
        cands = S.candidates(space, cfg.knobs[0], n_cfg)
        state = S.climb_state(cfg.knobs[0])
    else:
        cands = sim.knobs_tensor(knobs_local, device=dev)
    R = n_cfg * n_seeds_local
    out = S.alloc_outputs(R, detail=True, stats=True)
    agg = torch.empty((n_cfg, 32), dtype=torch.uint8, device=dev)
    parts = torch.empty((world * n_cfg, 32), dtype=torch.uint8, device=dev) if world > 1 else None
    pooled = torch.empty((n_cfg, 32), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2
    k1_start = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    k1_end = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    st_end = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    # K0 count + K0 classify + simulation + K1b select + K2 aggregate (+ K2b for N>1 sweeps, K3 for the climb);
    # simulation on the split path (gen_policy != 1): K1g + K1s (static) / K1g + K1c (continuous; K1e inside),
    # inline: K1 (static) / K1c (continuous)
    split = args.gen_policy != 1
    cont = any(w.get("batching", 0) for w in cfg.workloads)
    static = any(not w.get("batching", 0) for w in cfg.workloads)
    n_sim = (1 + (1 if static else 0) + (1 if cont else 0)) if split else ((1 if static else 0) + (1 if cont else 0))
    launches_per_step = 4 + n_sim + (1 if (world > 1 and args.workload != "c4" and not strong) else 0) + \
        (1 if args.workload == "c4" else 0)

    # N > 1: the aggregate exchange through the peers' windows (K2x/K2w, NEXT-4), NCCL as the fallback
    xchg, exchange_desc = None, None
    if world > 1:
        exchange_desc = "nccl all_gather_into_tensor"
        if args.exchange == "p2p" and strong and args.workload != "c4":
            args.exchange = "nccl"           # config shards are concatenated, not summed: the gather is NCCL's
            exchange_desc = "nccl all_gather_into_tensor (config-sharded: p2p windows sum parts, not gather)"
        if args.exchange == "p2p":
            try:
                from paper_2603_11340_b200.dist import PeerExchange
                if args.workload != "c4":
                    xchg = PeerExchange(S, n_cfg)
                exchange_desc = "p2p: K2x pushes into CUDA IPC peer windows, K2w waits on epoch flags"
            except Exception as e:                                      # noqa: BLE001
                exchange_desc = f"nccl all_gather_into_tensor (p2p unavailable: {str(e)[:120]})"
                args.exchange = "nccl"
        # (K2x + K2w replace K2 + K2b: the same launch count)
    graph = None
    if args.workload == "c4" and not args.eager_climb and (world == 1 or dist.get_backend() == "nccl"
                                                          or args.exchange == "p2p"):
        from paper_2603_11340_b200.dist import ClimbGraph
        graph = ClimbGraph(S, cfg, seeds, n_cand=n_cfg, exchange=args.exchange).capture()   # one graph per step
        out_eager = out                                                 # (the untimed per-kernel profile pass)
        out = graph.out                                                 # (replayed on the current stream)
        launches_per_step = 5 + n_sim + (1 if graph.xchg is not None else 0)   # K0 x2, sim, K1b, K2 (K2x+K2w), K3

    # a latency-bound sweep (at most four replicas per SM: C1) replays one captured CUDA graph per step
    # (dist.SweepGraph) instead of its seven stream launches; per-kernel times then come from an eager replay
    sweep_graph = None
    if graph is None and world == 1 and R <= 4 * info["sm_count"] and not args.no_graph:
        from paper_2603_11340_b200.dist import SweepGraph
        sweep_graph = SweepGraph(S, cands, seeds_t, cfg.segment_len, cfg.warmup_len, cfg.slo_us).capture()
        out_eager, out = out, sweep_graph.out                          # (the graph writes its own outputs)
        launches_per_step = 4 + n_sim                                   # K0 x2, simulation, K1b, K2

    def step(i=None):
        if sweep_graph is not None:
            if i is not None:
                k1_start[i].record(stream)
            sweep_graph.graph.replay()
            if i is not None:
                k1_end[i].record(stream)
                st_end[i].record(stream)
            return
        if graph is not None:
            if i is not None:
                k1_start[i].record(stream)
            graph.graph.replay()
            if i is not None:
                k1_end[i].record(stream)
                st_end[i].record(stream)
            return
        if i is not None:
            k1_start[i].record(stream)
        S.run_batch(cands, seeds_t, cfg.segment_len, cfg.warmup_len, cfg.slo_us, out=out, stream=stream)
        if i is not None:
            k1_end[i].record(stream)
        if xchg is not None:                                         # K2x + K2w: pooled over ranks
            xchg.pooled(out["detail"], n_seeds_local, pooled, stream=stream)
            if i is not None:
                st_end[i].record(stream)
            return
        S.aggregate(out["detail"], n_cfg, n_seeds_local, out=agg, stream=stream)
        if world > 1:
            if dist.get_backend() == "nccl":
                dist.all_gather_into_tensor(parts, agg)             # the one exchange
            else:
                dist.all_gather(list(parts.view(world, n_cfg, 32).unbind(0)), agg)
        if args.workload == "c4":                                    # K3 sums the per-rank parts itself
            S.hillclimb_step(space, sp, cands, parts if world > 1 else agg, world, state, stream=stream)
        elif world > 1 and not strong:
            S.aggregate_reduce(parts, world, n_cfg, out=pooled, stream=stream)
        # (strong sweeps: `parts` is the whole grid's aggregate table, rank-major: config c at row
        #  (c mod world) * n_cfg + c div world)
        if i is not None:
            st_end[i].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stats = sim.unpack(out["stats"], STATS_DTYPE)[0]       # work of one step (the last warm-up)
    # simulated requests per step, counted by the kernels (invalid / padding records simulate nothing)
    req_local = int(stats["requests"])
    if world > 1:
        tr = torch.tensor([req_local], dtype=torch.int64, device=dev)
        dist.all_reduce(tr)
        req_all = int(tr.item())
    else:
        req_all = req_local

    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if graph is None:
        S.profile(True)            # per-kernel CUDA events on the timed launches themselves (roofline below)
    clocks.start()
    for i in range(args.steps):
        flush.zero_()                                       # L2 flush between timed steps (not timed)
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # nvidia-smi samples every 200 ms: a timed region shorter than ~0.5 s (C1, C4) is followed by untimed
    # steps of the same workload (the same count on every rank) so the sampler sees the GPU under this load
    region_s = sum(k1_start[i].elapsed_time(st_end[i]) for i in range(args.steps)) / 1000.0
    extended = 0
    if clocks.proc is not None and region_s < 0.5:
        extended = int(min(4000, math.ceil((0.6 - region_s) / max(region_s / args.steps, 1e-5))))
    if world > 1:
        te = torch.tensor([extended], dtype=torch.int64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        extended = int(te.item())
    prof = None
    if graph is None and sweep_graph is None:
        prof = S.profile_read()    # exactly the timed steps' K0 / simulation / K1b launches
        S.profile(False)
    for _ in range(extended):
        step()
    torch.cuda.synchronize()
    clk = clocks.stop()
    if graph is not None or sweep_graph is not None:
        # the graph's launches record no events: time the same kernels on the same candidates eagerly
        gc = graph.evaluated if graph is not None else cands
        S.run_batch(gc, seeds_t, cfg.segment_len, cfg.warmup_len, cfg.slo_us, out=out_eager, stream=stream)
        torch.cuda.synchronize()
        S.profile(True)
        for _ in range(args.steps):
            flush.zero_()
            S.run_batch(gc, seeds_t, cfg.segment_len, cfg.warmup_len, cfg.slo_us, out=out_eager, stream=stream)
        prof = S.profile_read()
        S.profile(False)
    if clk is not None and extended:
        clk["untimed_load_steps_for_sampling"] = extended
    step_ms = [k1_start[i].elapsed_time(st_end[i]) for i in range(args.steps)]
    k1_ms = [k1_start[i].elapsed_time(k1_end[i]) for i in range(args.steps)]
    t_total = sum(step_ms) / 1000.0
    t_k1 = sum(k1_ms) / 1000.0                         # the whole run call (K0 + simulation + K1b)
    t_gen = prof["gen_ms"] / 1000.0                    # K1g (split path; 0 with inline generation)
    t_chain = prof["sim_ms"] / 1000.0                  # the chain kernels (K1 / K1s / K1t / K1c)
    t_sim = prof["wall_ms"] / 1000.0                   # the simulation as a whole (K1g and K1s overlap)
    t_k1b = prof["k1b_ms"] / 1000.0
    if world > 1:
        tt = torch.tensor([t_total, t_k1, t_sim, t_k1b, t_gen, t_chain], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_total, t_k1, t_sim, t_k1b, t_gen, t_chain = tt.tolist()

    value = req_all * args.steps / t_total

    # ---- e2e: the public API on HOST buffers (pinned), H2D + D2H inside the timed region
    if graph is not None:
        # the climb as a caller runs it (ClimbGraph.run_host): starting candidates + climb state copied in
        # from pinned host memory, then every step's climb state (the step's result) read back to the host
        e2e_steps = max(1, args.steps)
        h_c = graph.init_cands.cpu().pin_memory()
        h_s = graph.init_state.cpu().pin_memory()
        h_traj = torch.empty((e2e_steps, h_s.numel()), dtype=torch.uint8).pin_memory()
        graph.run_host(1, h_c, h_s, h_traj)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        graph.run_host(e2e_steps, h_c, h_s, h_traj)
        t_e2e = time.perf_counter() - t0
        h2d = (h_c.numel() + h_s.numel()) / e2e_steps
        d2h = h_s.numel()
    else:
        hk = sim.knobs_tensor(knobs_local if args.workload != "c4" else sim.unpack_knobs(cands.cpu().numpy()),
                              device="cpu").pin_memory()
        hs = sim.seeds_tensor(seeds, device="cpu").pin_memory()
        hout = dict(p99_us=torch.empty(R, dtype=torch.int32).pin_memory(),
                    goodput=torch.empty(R, dtype=torch.float64).pin_memory())
        S.run_batch_host(hk, hs, cfg.segment_len, cfg.warmup_len, cfg.slo_us, out=hout)
        e2e_steps = max(1, min(args.steps, 5))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            S.run_batch_host(hk, hs, cfg.segment_len, cfg.warmup_len, cfg.slo_us, out=hout)
        t_e2e = time.perf_counter() - t0
        h2d = hk.numel() + hs.numel() * 8
        d2h = R * 4 + R * 8
    if world > 1:
        te = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        t_e2e = te.item()
    e2e = {"value": req_all * e2e_steps / t_e2e, "unit": "requests/s",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}
    if graph is not None:
        e2e["api"] = "dist.ClimbGraph.run_host: climb trajectory read back every step"

    # K5 (supplementary, untimed): the Pareto front of this step's per-config aggregates
    pareto = None
    if args.workload != "c4":
        src = (parts if strong else pooled) if world > 1 else S.aggregate(out["detail"], n_cfg, n_seeds_local)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        S.pareto_front(src, count=True)
        e0.record(stream)
        _, cnt = S.pareto_front(src, count=True)
        e1.record(stream)
        e1.synchronize()
        pareto = {"configs": len(cfg.knobs), "on_front": int(cnt.item()), "ms": e0.elapsed_time(e1)}
    x_err = 0
    if world > 1:
        xo = xchg if xchg is not None else (graph.xchg if graph is not None else None)
        x_err = xo.error() if xo is not None else 0
        te = torch.tensor([x_err], dtype=torch.int64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        x_err = int(te.item())
    if rank == 0:
        pk = peaks()
        blocks = int(stats["philox_blocks"])
        peak_gops = 148 * 4 * 32 * pk["sm_max_mhz"] * 1e6 / 1e9      # lane-ops/s at 1 warp-instr/clk/SMSP
        # K4: measured Philox4x32-10 throughput of this GPU at full occupancy (untimed, after the run)
        rng_peak_gops = S.philox_peak() * OPS_PER_PHILOX_BLOCK / 1e9
        # the Philox blocks each kernel draws: K1g the REQ and SPEC blocks of every request; the chain kernels the
        # ITER blocks of continuous batching (one per noisy decode iteration, §2.12) and the PHASE blocks of MMPP-2
        iter_blocks = int(stats["decode_steps"]) if (cont and any(w["timing"]["noise_step_ppm"] for w in cfg.workloads)) else 0
        gen_blocks = blocks - iter_blocks if t_gen > 0 else 0
        chain_blocks = blocks - gen_blocks
        # the dominant kernel (its own CUDA-event time over the timed launches) carries the roofline; a static chain
        # kernel that dominates (latency-bound launches: C1, C4) draws no Philox blocks of its own, so there the
        # simulation as a whole (K1g + K1s, its CUDA-event span) is the unit
        dom_gen = t_gen >= t_chain
        whole = not dom_gen and chain_blocks == 0
        t_dom = (t_gen if dom_gen else (t_sim if whole else t_chain)) / args.steps
        dom_blocks = gen_blocks if dom_gen else (blocks if whole else chain_blocks)
        achieved_gops = dom_blocks * OPS_PER_PHILOX_BLOCK / t_dom / 1e9
        sim_gops = blocks * OPS_PER_PHILOX_BLOCK / (t_sim / args.steps) / 1e9
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
                traffic = json.load(fh).get(args.workload + (":k1g" if dom_gen else ":chain"))
        except Exception:
            pass
        # BASELINE's "% SM issue / HBM peak": issue-slot utilisation of the kernels from their committed ncu
        # summaries (profiles/r02_*_ncu.json), and the HBM share of this run (ncu bytes over the live kernel time)
        def ncu_issue(tag):
            import glob
            fs = (sorted(glob.glob(os.path.join(ROOT, "profiles", f"r02_{tag}_ncu.json"))) +
                  sorted(glob.glob(os.path.join(ROOT, "profiles", f"r02b_{tag}_ncu.json"))))
            if not fs:
                return None
            try:
                with open(fs[-1]) as fh:
                    m = json.load(fh)["metrics"]
                return {"pct_of_peak": float(m["sm__inst_issued.avg.pct_of_peak_sustained_active"][0]),
                        "source": os.path.relpath(fs[-1], ROOT)}
            except Exception:
                return None
        wl_tag = "c2c" if args.workload == "c2c" else "c2"
        chain_tag = ("k1c" if cont else "k1s") if split else ("k1c" if cont else "k1")
        hbm = None
        if traffic:
            gbs = traffic / t_dom / 1e9
            hbm = {"gb_per_s": gbs, "peak_gb_per_s": pk["hbm_gbs"], "frac": gbs / pk["hbm_gbs"]}
        gen_name = "K1g slo_gen_kernel (per-request generation: Philox REQ + SPEC blocks, E_q, lengths, S_i)"
        chain_name = ("K1c slo_sim_cont_kernel_t (continuous-batching chains, K1e scans inside)" if cont else
                      "K1s slo_serve_kernel_t (static-batching chains)") if split else \
                     ("K1c slo_sim_cont_kernel_t" if cont else "K1 slo_sim_kernel_t (inline generation + chain)")
        roofline = {"bound": "alu", "achieved": achieved_gops, "peak": peak_gops, "unit": "Gop/s",
                    "frac": achieved_gops / peak_gops, "traffic": traffic,
                    "kernel": (gen_name if dom_gen else (("the simulation: K1g + " + chain_name) if whole else chain_name))
                              + ", its own CUDA-event time",
                    "dominant_kernel_share_of_step": t_dom * args.steps / t_total,
                    "issue_util_ncu": ncu_issue(("k1g_" + wl_tag) if dom_gen else (chain_tag + "_" + wl_tag)),
                    "hbm": hbm,
                    "note": "algorithmic int32 lane-ops = the Philox4x32-10 blocks the definition consumes (counted "
                            "exactly by the kernels) that this kernel draws x 60; peak = 148 SM x 4 SMSP x 32 lanes x "
                            "sm_max_mhz (issue limit)",
                    "measured_rng_peak": rng_peak_gops,
                    "frac_of_measured_rng_peak": achieved_gops / rng_peak_gops,
                    "measured_rng_peak_note": "K4 slo_philox_peak: Philox blocks/s x 60 of a full-occupancy kernel "
                                              "that only draws blocks (the RNG roofline of DESIGN.md §7)",
                    "kernels": {
                        "k1g": {"ms_per_step": 1000.0 * t_gen / args.steps, "philox_blocks": gen_blocks,
                                "frac_of_measured_rng_peak": (gen_blocks * OPS_PER_PHILOX_BLOCK / (t_gen / args.steps)
                                                              / 1e9 / rng_peak_gops) if t_gen > 0 else None,
                                "issue_util_ncu": ncu_issue("k1g_" + wl_tag) if t_gen > 0 else None},
                        "chain": {"kernel": chain_name, "ms_per_step": 1000.0 * t_chain / args.steps,
                                  "philox_blocks": chain_blocks, "issue_util_ncu": ncu_issue(chain_tag + "_" + wl_tag)},
                        "simulation": {"ms_per_step": 1000.0 * t_sim / args.steps, "achieved": sim_gops,
                                       "frac": sim_gops / peak_gops,
                                       "frac_of_measured_rng_peak": sim_gops / rng_peak_gops}}}
        line = {
            "metric": "simulated requests/s", "value": value, "unit": "requests/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * t_total / args.steps,
            "higher_is_better": True, "scaling": "strong" if (strong or args.workload == "c4") else "weak",
            "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (seeded Philox streams; LL/STRESS presets of DESIGN.md §5)",
            "config": {"workload": DESCR[args.workload], "replicas_per_gpu": R, "requests_per_replica": N,
                       "requests_per_step": req_all, **({"share_of": pworld} if world == 1 and pworld > 1 else {}), "preset": "STRESS" if args.workload.startswith("c5") else "LL",
                       "l2": "flushed between timed steps (256 MiB write, untimed); inputs are < 1 MB",
                       "parallelism": f"dp{world} over replicas ({'seed-sharded climb' if args.workload == 'c4' else ('config-sharded: config c on rank c mod N, all seeds local' if strong else 'weak: full grid, per-rank seed block')})",
                       "exchange": exchange_desc,
                       "cuda_graph": ("ClimbGraph (one Alg. 1 step per replay)" if graph is not None else
                                      "SweepGraph (one sweep step per replay)" if sweep_graph is not None else None),
                       "launch": {"blocks_per_sm": info["blocks_per_sm"], "warps_per_block": info["warps_per_block"],
                                  "regs_per_thread": info["regs_per_thread"]}},
            "replica_segments_per_s": (req_all // N) * args.steps / t_total,
            "run_ms_per_step": 1000.0 * t_k1 / args.steps,
            "kernel_ms_per_step": {"simulate": 1000.0 * t_sim / args.steps, "k1g_generate": 1000.0 * t_gen / args.steps,
                                   "chain": 1000.0 * t_chain / args.steps, "k1b_select": 1000.0 * t_k1b / args.steps,
                                   "source": "CUDA events around each launch (slo_sim_profile) on the launching "
                                             "stream, " + ("the timed launches" if (graph is None and sweep_graph is None)
                                                           else "an eager replay of the graph's launches")},
            "work_per_step_per_gpu": {"philox_blocks": blocks, "batches": int(stats["batches"]),
                                      "member_steps": int(stats["member_steps"]),
                                      "decode_steps": int(stats["decode_steps"])},
            "roofline": roofline,
            "gpu_launches": launches_per_step * args.steps,
            **({"exchange_error": x_err} if world > 1 else {}),
            **({"pareto": pareto} if pareto is not None else {}),
            "e2e": e2e,
            "clocks": clk,
        }
        if world == 1 and not args.no_cpu_baseline:
            v, cores, reps, reqs, dt = cpu_oracle_sample(cfg, budget_s=args.cpu_budget)
            v1, reps1, reqs1, dt1 = cpu_oracle_1core(cfg, budget_s=max(3.0, args.cpu_budget / 2))
            line["cpu_baseline"] = {"value": v, "unit": "requests/s", "cores": cores, "kind": "oracle",
                                    "sample": f"{reps} replicas ({reqs} requests) of {args.workload.upper()} in "
                                              f"seed-major order, {dt:.1f} s on {cores} worker processes",
                                    "value_1core": v1,
                                    "sample_1core": f"{reps1} replicas ({reqs1} requests), same order, {dt1:.1f} s "
                                                    f"in one process (1 core)"}
        if args.workload == "c4" and graph is not None and world == 1:
            line["time_to_solution"] = climb_time_to_solution(S, cfg, seeds, graph)
        print(json.dumps(line))
    if world > 1:
        dist.barrier()                         # no rank still reads a peer window
        for xo in (xchg, graph.xchg if graph is not None else None):
            if xo is not None:
                xo.close()
    if graph is not None:
        graph.close()
    S.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
