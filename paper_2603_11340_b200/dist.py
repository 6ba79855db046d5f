"""Multi-GPU plumbing: one process per GPU, torch.distributed for the exchange.

Replicas are independent, so a sweep shards with no data-path collective; the one exchange the method
has is pooling the per-config aggregates (Eq. 1 pooled over seeds, R17) before the score and
the hill-climb argmax (Alg. 1) — an all-gather of 32-byte integer records over NCCL,
reduced on the device by K2b (`slo_aggregate_reduce`).  Integer sums make the pooled result independent
of rank order, so every rank holds bit-identical aggregates and takes the identical climb step.

Sharding rules:
  * sweeps (C2, C3, C5), default: config-sharded — config c on rank c mod world with all its
    seeds, one all-gather of the per-config aggregates assembles the grid (strong scaling: the BASELINE grid
    is split, unchanged); opt-in weak scaling — every rank runs the full config grid on its own seed block
    (seed offset rank * n_seeds), pooled aggregates then cover world * n_seeds seeds per config;
  * climb (C4): seed-sharded — the n_seeds seeds are split into contiguous per-rank blocks, so the pooled
    aggregate equals the single-GPU one exactly.
"""
from __future__ import annotations

from typing import List, Tuple

import torch
import torch.distributed as dist


def world() -> Tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def seed_block(n_seeds: int, rank: int, world_size: int) -> Tuple[int, int]:
    """Contiguous seed slice [lo, hi) of `rank` when n_seeds seeds are split over world_size ranks."""
    base, extra = divmod(n_seeds, world_size)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def config_shard(knobs: List, rank: int, world_size: int, pad=None) -> List:
    """Config-sharded sweep: config c goes to rank c mod world_size (round-robin balances the
    grid's heterogeneous costs), with all of its seeds, so per-config sums stay local.  With `pad` every rank's
    share is padded to ceil(n / world_size) records (an always-invalid record simulates nothing) so the
    aggregate all-gather has equal parts; the gathered table is rank-major: config c at row
    (c mod world_size) * per + c div world_size."""
    mine = list(knobs[rank::world_size])
    if pad is not None:
        per = -(-len(knobs) // world_size)
        mine += [pad] * (per - len(mine))
    return mine


def unshard_rows(n_cfg: int, world_size: int) -> List[int]:
    """Row of config c in the rank-major gathered table of config_shard(pad=...) shares."""
    per = -(-n_cfg // world_size)
    return [(c % world_size) * per + c // world_size for c in range(n_cfg)]


def sweep_seed_offset(n_seeds: int, rank: int, base_offset: int = 0) -> int:
    """Weak-scaled sweep: rank r simulates seeds [base + r n_seeds, base + (r+1) n_seeds)."""
    return base_offset + rank * n_seeds


def gather_aggregates(agg: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather per-config aggregates (uint8 [n_cfg, 32] slo_config_agg records) from every rank into a
    [world * n_cfg, 32] tensor in rank order (the layout slo_aggregate_reduce / slo_hillclimb_step take)."""
    _, w = world()
    if w == 1:
        return agg
    out = torch.empty((w * agg.shape[0], agg.shape[1]), dtype=agg.dtype, device=agg.device)
    dist.all_gather_into_tensor(out, agg.contiguous(), group=group)
    return out


def max_over_ranks(x: float, device=None) -> float:
    _, w = world()
    if w == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class PeerExchange:
    """NEXT-4: the aggregate exchange done by the aggregation kernel itself over NVLink peer memory.

    Every rank's K2x writes its per-config sums straight into every peer's window (CUDA IPC peer pointers)
    and publishes an epoch flag; K2w waits for all flags and sums the parts in rank order — the same integers
    as all-gather + K2b, with no NCCL call and no host round trip, so it can live inside the climb's CUDA
    graph.  Handles are swapped once through the process group (any backend)."""

    def __init__(self, sim, n_cfg: int, group=None):
        rank, w = world()
        if w < 2:
            raise ValueError("PeerExchange needs world_size >= 2")
        self.sim, self.n_cfg = sim, n_cfg
        self.x, handle = sim.exchange_create(w, rank, n_cfg)
        handles: List[bytes] = [b""] * w
        dist.all_gather_object(handles, handle, group=group)
        sim.exchange_open(self.x, b"".join(handles))
        dist.barrier(group=group)                 # every window is mapped before anyone pushes

    def pooled(self, detail: torch.Tensor, n_seeds: int, out: torch.Tensor, stream=None) -> torch.Tensor:
        return self.sim.aggregate_exchange(self.x, detail, n_seeds, out, stream=stream)

    def error(self) -> int:
        return self.sim.exchange_error(self.x)

    def close(self):
        if self.x is not None:
            self.sim.exchange_destroy(self.x)
            self.x = None


class SweepGraph:
    """One sweep step — K0/K1g/K1s (or K1/K1c)/K1b simulate and K2 aggregate — captured once in a CUDA graph
    on a handle of its own (the graph holds pointers into that handle's scratch) and replayed: a latency-bound
    launch (C1: one replica) then pays one graph launch instead of seven stream launches per step."""

    def __init__(self, sim, knobs: torch.Tensor, seeds: torch.Tensor, segment_len: int, warmup_len: int = 0,
                 slo_us: int = 1_200_000):
        self.sim = sim.twin()
        self.knobs, self.seeds = knobs, seeds
        self.n_cfg, self.n_seeds = knobs.shape[0], seeds.shape[0]
        self.args = (segment_len, warmup_len, slo_us)
        self.out = self.sim.alloc_outputs(self.n_cfg * self.n_seeds, detail=True, stats=True)
        self.agg = torch.empty((self.n_cfg, 32), dtype=torch.uint8, device=knobs.device)
        self.stream = torch.cuda.Stream(device=knobs.device)
        self.graph = None

    def _step(self):
        self.sim.run_batch(self.knobs, self.seeds, *self.args, out=self.out, stream=self.stream)
        self.sim.aggregate(self.out["detail"], self.n_cfg, self.n_seeds, out=self.agg, stream=self.stream)

    def capture(self):
        """Warm up (allocates the library's scratch), then capture one step."""
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):
            self._step()
        self.stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self._step()
        return self

    def close(self):
        self.graph = None
        self.sim.close()


def final_rerun(sim, cfg, state: torch.Tensor, seeds, out=None, stream=None) -> dict:
    """Alg. 1's last line ("Re-run one segment at K_best and report final metrics"; "re-measures it
    at the end"): simulate K_best — read straight from the device climb state (bytes 32..64 of slo_climb_state)
    — on `seeds` (a list or a device seeds tensor; a fresh seed block gives an independent segment) and return
    its per-seed p99 / goodput and the pooled aggregate ("agg"), on the device (asynchronous on `stream`; `out`
    from a previous call is reused)."""
    from . import sim as S
    kb = state.view(-1)[32:64].view(1, 32)
    st = seeds if isinstance(seeds, torch.Tensor) else S.seeds_tensor(seeds, device=state.device)
    out = sim.run_batch(kb, st, cfg.segment_len, cfg.warmup_len, cfg.slo_us, out=out, stream=stream)
    out["agg"] = sim.aggregate(out["detail"], 1, st.shape[0], out=out.get("agg"), stream=stream)
    return out


class ClimbGraph:
    """Alg. 1 with the whole step — K0/K1/K1b simulate, K2 aggregate, all-gather (N > 1), K3 climb — captured
    once in a CUDA graph and replayed (SV §8(f) NEXT-4): no host round trip between steps.  The candidate
    list and the climb state live in device buffers that the step rewrites in place."""

    def __init__(self, sim, cfg, seeds: List[int], n_cand: int = 32, sp=None, exchange: str = "nccl"):
        from . import sim as S
        # the graph holds pointers into its handle's scratch, so it gets a handle of its own: no other call can
        # regrow that scratch under it (the library also refuses any regrow of a captured handle)
        sim = sim.twin()
        self.sim, self.cfg = sim, cfg
        self.space = cfg.extra["space"]
        self.sp = dict(sp if sp is not None else cfg.extra["score"])
        K0 = cfg.knobs[0]
        self.n_cand, self.n_seeds = n_cand, len(seeds)
        self.cands = sim.candidates(self.space, K0, n_cand)
        self.state = sim.climb_state(K0)
        self.init_cands = self.cands.clone()
        self.init_state = self.state.clone()
        self.seeds = S.seeds_tensor(seeds, device=self.cands.device)
        self.out = sim.alloc_outputs(n_cand * len(seeds), detail=True, stats=True)
        self.agg = torch.empty((n_cand, 32), dtype=torch.uint8, device=self.cands.device)
        _, self.w = world()
        self.parts = (torch.empty((self.w * n_cand, 32), dtype=torch.uint8, device=self.cands.device)
                      if self.w > 1 else self.agg)
        # N > 1: "nccl" = K2 + NCCL all-gather + K3 summing the parts; "p2p" = PeerExchange (K2x + K2w)
        self.xchg = PeerExchange(sim, n_cand) if (self.w > 1 and exchange == "p2p") else None
        self.evaluated = torch.empty_like(self.cands)          # the step's candidates (K3 rewrites cands)
        self.scores = torch.empty(n_cand, dtype=torch.int64, device=self.cands.device)
        self.stream = torch.cuda.Stream(device=self.cands.device)
        self.graph = None

    def _step(self):
        c = self.cfg
        self.sim.run_batch(self.cands, self.seeds, c.segment_len, c.warmup_len, c.slo_us, out=self.out,
                           stream=self.stream)
        self.evaluated.copy_(self.cands)
        if self.xchg is not None:
            self.xchg.pooled(self.out["detail"], self.n_seeds, self.agg, stream=self.stream)
            self.sim.hillclimb_step(self.space, self.sp, self.cands, self.agg, 1, self.state, scores=self.scores,
                                    stream=self.stream)
            return
        self.sim.aggregate(self.out["detail"], self.n_cand, self.n_seeds, out=self.agg, stream=self.stream)
        if self.w > 1:
            dist.all_gather_into_tensor(self.parts, self.agg)
        self.sim.hillclimb_step(self.space, self.sp, self.cands, self.parts, self.w, self.state, scores=self.scores,
                                stream=self.stream)

    def capture(self):
        """Warm up (allocates the library's scratch), restore the initial state, capture one step."""
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):
            self._step()
        self.stream.synchronize()
        self.cands.copy_(self.init_cands)
        self.state.copy_(self.init_state)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self._step()
        return self

    def close(self):
        if self.xchg is not None:
            self.xchg.close()
            self.xchg = None
        self.graph = None
        self.sim.close()

    def run(self, steps: int):
        if self.graph is None:
            self.capture()
        for _ in range(steps):
            self.graph.replay()
        return self.state, self.cands

    def trajectory(self, steps: int, path=None) -> List[dict]:
        """Run `steps` climb steps from the current device state and return (and, with `path`, write as JSON
        lines — SPEC S:257/S:300 TuningTrajectory) one record per step: the evaluated candidates and their
        Eq. (3) scores, the argmax, whether K moved, the next K, the best-so-far and the EMA p99."""
        import json
        import numpy as np
        from . import sim as S
        from ._lib import CLIMB_DTYPE, KNOB_DTYPE
        if self.graph is None:
            self.capture()
        nb = self.state.numel()
        h_st = torch.empty((steps, nb), dtype=torch.uint8).pin_memory()
        h_ev = torch.empty((steps,) + tuple(self.evaluated.shape), dtype=torch.uint8).pin_memory()
        h_sc = torch.empty((steps, self.n_cand), dtype=torch.int64).pin_memory()
        st = self.stream
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            for i in range(steps):
                self.graph.replay()
                h_st[i].copy_(self.state.view(-1), non_blocking=True)
                h_ev[i].copy_(self.evaluated, non_blocking=True)
                h_sc[i].copy_(self.scores, non_blocking=True)
        st.synchronize()
        recs = []
        for i in range(steps):
            s = h_st[i].numpy().view(CLIMB_DTYPE)[0]
            ks = S.unpack_knobs(h_ev[i].numpy().view(KNOB_DTYPE))
            sc = h_sc[i].numpy().tolist()
            valid = [j for j, k in enumerate(ks) if k["conc"] > 0]
            recs.append({"step": int(s["step"]), "current": ks[0],
                         "candidates": [ks[j] for j in valid], "scores_micro": [sc[j] for j in valid],
                         "argmax": int(s["argmax"]), "moved": bool(s["moved"]),
                         "next": S.unpack_knobs(np.array([s["K"]]))[0],
                         "best": S.unpack_knobs(np.array([s["K_best"]]))[0], "best_score_micro": int(s["S_best_micro"]),
                         "ema_p99_us": int(s["ema_p99_us"]) if int(s["has_ema"]) else None})
        if path is not None:
            with open(path, "w") as fh:
                for r in recs:
                    fh.write(json.dumps(r) + "\n")
        return recs

    def run_host(self, steps: int, h_cands: torch.Tensor, h_state: torch.Tensor, h_traj: torch.Tensor):
        """End-to-end use from host memory: copy the starting candidates and climb state in (pinned host ->
        device), replay `steps` climb steps and read every step's climb state back into h_traj[step]
        (pinned uint8 [steps, 104]) — the trajectory a caller observes.  Synchronous."""
        if self.graph is None:
            self.capture()
        st = self.stream
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            self.cands.copy_(h_cands, non_blocking=True)
            self.state.copy_(h_state, non_blocking=True)
            for i in range(steps):
                self.graph.replay()
                h_traj[i].copy_(self.state.view(-1), non_blocking=True)
        st.synchronize()
        return h_traj


class LookaheadClimbGraph:
    """Alg. 1 two steps per round (SV §8(f) NEXT-4 neighbour-of-neighbour lookahead, slo_lookahead_*): a round
    simulates U(K) = {K} u N(K) u N(N(K)) minus what the previous round measured (the cache), then takes two
    steps from the table.  Same trajectory as ClimbGraph; the whole round — prepare, K0/K1/K1b over the
    SLO_LOOKAHEAD_CAP-record list (invalid padding records cost nothing), K2, all-gather (N > 1, seed-sharded),
    two steps — is one CUDA graph."""

    CAP = 320                                             # SLO_LOOKAHEAD_CAP
    TABLE_BYTES = 34576                                   # SLO_LOOKAHEAD_TABLE_BYTES

    def __init__(self, sim, cfg, seeds: List[int], n_cand: int = 32, sp=None):
        from . import sim as S
        sim = sim.twin()                                   # the graph holds this handle's scratch
        self.sim, self.cfg = sim, cfg
        self.space = cfg.extra["space"]
        self.sp = dict(sp if sp is not None else cfg.extra["score"])
        dev = torch.device("cuda", sim.device)
        self.n_cand, self.n_seeds = n_cand, len(seeds)
        self.state = sim.climb_state(cfg.knobs[0])
        self.init_state = self.state.clone()
        self.table = torch.zeros(self.TABLE_BYTES, dtype=torch.uint8, device=dev)
        self.sim_list = torch.zeros((self.CAP, 32), dtype=torch.uint8, device=dev)
        self.seeds = S.seeds_tensor(seeds, device=dev)
        self.out = sim.alloc_outputs(self.CAP * len(seeds), detail=True, stats=True)
        self.agg = torch.empty((self.CAP, 32), dtype=torch.uint8, device=dev)
        _, self.w = world()
        self.parts = (torch.empty((self.w * self.CAP, 32), dtype=torch.uint8, device=dev) if self.w > 1 else self.agg)
        self.traj = torch.empty((2, self.state.numel()), dtype=torch.uint8, device=dev)
        self.stream = torch.cuda.Stream(device=dev)
        self.graph = None

    def _round(self, host_gather: bool = False):
        c, st = self.cfg, self.stream
        self.sim.lookahead_prepare(self.space, self.state, self.table, self.sim_list, stream=st)
        # only the table's n_sim records are simulated (its 3rd word): the padding costs nothing
        self.sim.run_batch(self.sim_list, self.seeds, c.segment_len, c.warmup_len, c.slo_us, out=self.out, stream=st,
                           live_configs_ptr=self.table.data_ptr() + 8)
        self.sim.aggregate(self.out["detail"], self.CAP, self.n_seeds, out=self.agg, stream=st)
        if self.w > 1 and host_gather:                     # eager over a host backend (gloo): stage through host
            st.synchronize()
            parts = torch.empty(tuple(self.parts.shape), dtype=torch.uint8)
            dist.all_gather_into_tensor(parts, self.agg.cpu())
            self.parts.copy_(parts)
        elif self.w > 1:
            dist.all_gather_into_tensor(self.parts, self.agg)
        self.sim.lookahead_step(self.space, self.sp, self.table, self.parts, self.w, self.n_cand, self.state,
                                self.traj, stream=st)

    def reset(self):
        self.state.copy_(self.init_state)
        self.table.zero_()

    def capture(self):
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):
            self._round()
        self.stream.synchronize()
        self.reset()
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self._round()
        return self

    def close(self):
        self.graph = None
        self.sim.close()

    def run(self, rounds: int):
        if self.graph is None:
            self.capture()
        for _ in range(rounds):
            self.graph.replay()
        return self.state

    def run_eager(self, rounds: int) -> torch.Tensor:
        """The rounds without a graph (a multi-rank run over a host backend such as gloo, whose collectives a CUDA
        graph cannot capture); returns the state after every step, uint8 [2 rounds, 104] (host)."""
        host = self.w > 1 and dist.get_backend() != "nccl"
        h = torch.empty((rounds, 2, self.state.numel()), dtype=torch.uint8)
        with torch.cuda.stream(self.stream):
            for i in range(rounds):
                self._round(host_gather=host)
                h[i].copy_(self.traj.cpu())
        self.stream.synchronize()
        self.check()
        return h.view(2 * rounds, -1)

    def states(self, rounds: int) -> torch.Tensor:
        """Replay `rounds` rounds and return the climb state after every step: uint8 [2 rounds, 104] (host)."""
        if self.graph is None:
            self.capture()
        h = torch.empty((rounds, 2, self.state.numel()), dtype=torch.uint8).pin_memory()
        st = self.stream
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            for i in range(rounds):
                self.graph.replay()
                h[i].copy_(self.traj, non_blocking=True)
        st.synchronize()
        self.check()
        return h.view(2 * rounds, -1)

    def check(self) -> None:
        """Raise if a round's U(K) exceeded the table's capacity (the table's 4th word; not reachable with the
        built-in stencils: tests/test_lookahead_cpu.py bounds |U| by 272)."""
        over = int(self.table[12:16].view(torch.int32).item())
        if over:
            raise RuntimeError(f"lookahead: |U(K)| = {over} exceeds the capacity {self.CAP}")

    def simulated(self) -> int:
        """Records the last round simulated (the rest came from the cache)."""
        return int(self.table[8:12].view(torch.int32).item())


def hillclimb(sim, cfg, steps: int, seeds: List[int], n_cand: int = 32, stream=None):
    """Device-resident Alg. 1 over `steps` iterations on this rank's seed slice; returns the final state.

    Each step: K1 over [K, neighbours] x seeds -> K2 per-config sums -> all-gather over ranks -> K3 climb
    step (score, argmax, move, best-so-far, next candidates).  Nothing returns to the host between steps."""
    from . import sim as S
    space, sp = cfg.extra["space"], cfg.extra["score"]
    K0 = cfg.knobs[0]
    cands = sim.candidates(space, K0, n_cand)
    state = sim.climb_state(K0)
    seeds_t = S.seeds_tensor(seeds, device=cands.device)
    out = sim.alloc_outputs(n_cand * len(seeds), detail=True)
    agg = torch.empty((n_cand, 32), dtype=torch.uint8, device=cands.device)
    _, w = world()
    for _ in range(steps):
        sim.run_batch(cands, seeds_t, cfg.segment_len, cfg.warmup_len, cfg.slo_us, out=out, stream=stream)
        sim.aggregate(out["detail"], n_cand, len(seeds), out=agg, stream=stream)
        parts = gather_aggregates(agg)
        sim.hillclimb_step(space, sp, cands, parts, w, state, stream=stream)
    return state, cands
