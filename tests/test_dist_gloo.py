"""Multi-process (world size 2, gloo, CPU) checks of the N>1 host logic: seed sharding, the all-gather layout
of per-config aggregates, and that every rank takes the identical climb decision from pooled aggregates
equal to the single-process ones.  The per-replica results come from the oracle here (no
GPU); on B200 the same records come from K1/K2 and the reduction runs in K2b/K3."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_11340_b200 import inputs
from paper_2603_11340_b200.dist import gather_aggregates, seed_block

AGG = np.dtype([("sum_p99_us", "<u8"), ("sum_slo_met", "<u8"), ("sum_window_us", "<u8"),
                ("n_seeds", "<u4"), ("flags", "<u4")])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_seed_blocks_partition():
    for n in (1, 5, 128, 129):
        for w in (1, 2, 3, 8):
            blocks = [seed_block(n, r, w) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


def _agg_records(orc, cfg, cands, seeds, N):
    from oracle import climb
    recs = np.zeros(len(cands), AGG)
    aggs = []
    for ci, k in enumerate(cands):
        a = climb.aggregate([orc.run(cfg.workloads, k, s, N) for s in seeds])
        aggs.append(a)
        for f in AGG.names:
            recs[ci][f] = a[f]
    return recs, aggs


def _worker(rank, world_size, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    try:
        import oracle
        from oracle import climb
        cfg = inputs.config_c4(n_seeds=6, segment_len=300)
        space, sp = cfg.extra["space"], cfg.extra["score"]
        seeds = cfg.seeds()
        lo, hi = seed_block(len(seeds), rank, world_size)
        st = climb.initial_state(cfg.knobs[0])
        traj = []
        for _ in range(2):
            cands = [st["K"]] + climb.neighbours(space, st["K"])
            recs, _ = _agg_records(oracle, cfg, cands, seeds[lo:hi], cfg.segment_len)
            local = torch.from_numpy(recs.view(np.uint8).reshape(len(cands), 32).copy())
            parts = gather_aggregates(local)                       # [world * n_cand, 32] in rank order
            arr = parts.numpy().view(AGG).reshape(world_size, len(cands))
            pooled = []
            for ci in range(len(cands)):
                d = {f: int(sum(int(arr[r][ci][f]) for r in range(world_size))) for f in AGG.names if f != "flags"}
                d["flags"] = int(np.bitwise_or.reduce([int(arr[r][ci]["flags"]) for r in range(world_size)]))
                pooled.append(d)
            st, moved, idx, scores = climb.step(st, cands, pooled, sp)
            traj.append((moved, idx, scores, dict(st["K"])))
        q.put((rank, traj))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_pooled_climb_matches_single_process():
    import oracle
    from oracle import climb
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1]                                        # identical decisions on every rank
    # single-process reference over all seeds
    cfg = inputs.config_c4(n_seeds=6, segment_len=300)
    space, sp = cfg.extra["space"], cfg.extra["score"]
    st = climb.initial_state(cfg.knobs[0])
    for step in range(2):
        cands = [st["K"]] + climb.neighbours(space, st["K"])
        _, aggs = _agg_records(oracle, cfg, cands, cfg.seeds(), cfg.segment_len)
        st, moved, idx, scores = climb.step(st, cands, aggs, sp)
        assert (moved, idx, scores, dict(st["K"])) == res[0][step]


def test_config_shard_partition():
    from paper_2603_11340_b200.dist import config_shard, unshard_rows
    for n in (1, 7, 512, 1000):
        for w in (1, 2, 3, 8):
            shares = [config_shard(list(range(n)), r, w, pad=-1) for r in range(w)]
            per = -(-n // w)
            assert all(len(s) == per for s in shares)
            table = [x for s in shares for x in s]                 # the rank-major all-gather
            rows = unshard_rows(n, w)
            assert [table[rows[c]] for c in range(n)] == list(range(n))
            assert sorted(x for x in table if x >= 0) == list(range(n))


def _sweep_worker(rank, world_size, port, q):
    """Config-sharded sweep: config c on rank c mod world with all its seeds; the one exchange
    is an all-gather of the per-config aggregates (padding records are invalid and simulate nothing)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    try:
        import oracle
        from paper_2603_11340_b200.dist import config_shard
        cfg = inputs.config_c2(n_seeds=3, segment_len=200)
        knobs = cfg.knobs[::37]                                       # 14 configs: uneven over 2 and 3 ranks
        mine = config_shard(knobs, rank, world_size, pad=inputs.PAD_KNOBS)
        recs, _ = _agg_records(oracle, cfg, mine, cfg.seeds(), cfg.segment_len)
        local = torch.from_numpy(recs.view(np.uint8).reshape(len(mine), 32).copy())
        parts = gather_aggregates(local)
        q.put((rank, parts.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world_size", [2, 3])
def test_config_sharded_sweep_matches_single_process(world_size):
    import oracle
    from paper_2603_11340_b200.dist import unshard_rows
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sweep_worker, args=(r, world_size, port, q)) for r in range(world_size)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(set(res.values())) == 1                              # every rank holds the same table
    cfg = inputs.config_c2(n_seeds=3, segment_len=200)
    knobs = cfg.knobs[::37]
    table = np.frombuffer(res[0], dtype=AGG)
    rows = unshard_rows(len(knobs), world_size)
    ref, _ = _agg_records(oracle, cfg, knobs, cfg.seeds(), cfg.segment_len)
    assert table[rows].tobytes() == ref.tobytes()                  # = the single-process grid, config order
    pad_rows = sorted(set(range(len(table))) - set(rows))
    assert all(int(table[r]["flags"]) & 1 for r in pad_rows)      # padding: invalid, no work
