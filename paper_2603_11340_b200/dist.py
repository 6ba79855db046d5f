"""Multi-GPU plumbing: one process per GPU, torch.distributed for the exchange.

Replicas are independent, so a sweep shards with no data-path collective; the one exchange the method
has is pooling the per-config aggregates (Eq. 1 pooled over seeds, R17) before the score and
the hill-climb argmax (Alg. 1) — an all-gather of 32-byte integer records over NCCL,
reduced on the device by K2b (`slo_aggregate_reduce`).  Integer sums make the pooled result independent
of rank order, so every rank holds bit-identical aggregates and takes the identical climb step.

Sharding rules:
  * sweeps (C2, C3, C5): weak scaling — every rank runs the full config grid on its own seed block
    (seed offset rank * n_seeds); pooled aggregates then cover world * n_seeds seeds per config;
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
