"""Worker for tests/test_gpu_exchange.py (not collected): one rank of the NEXT-4 peer exchange.

Launched by torchrun with 2 ranks sharing GPU 0 (the only GPU of a test box): each rank simulates its seed
slice of a small C4 climb and runs Alg. 1 steps through dist.ClimbGraph(exchange="p2p") — K2x pushes the
per-config sums into both ranks' windows through CUDA IPC peer pointers, K2w waits for the epoch flags and
sums.  Rank 0 writes the pooled aggregates of one standalone exchange and the final climb state to the
JSON file named by argv[1]."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    out_path, steps = sys.argv[1], int(sys.argv[2])
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    from paper_2603_11340_b200 import dist as D
    from paper_2603_11340_b200 import inputs, sim
    cfg = inputs.config_c4(n_seeds=8, segment_len=400)
    lo, hi = D.seed_block(cfg.n_seeds, rank, world)
    seeds = cfg.seeds()[lo:hi]
    s = sim.Simulator(cfg.workloads, device=0)
    # one standalone exchange of the first step's aggregates
    cands = s.candidates(cfg.extra["space"], cfg.knobs[0], 32)
    out = s.run_batch(cands, sim.seeds_tensor(seeds), cfg.segment_len)
    x = D.PeerExchange(s, 32)
    pooled = torch.empty((32, 32), dtype=torch.uint8, device="cuda")
    x.pooled(out["detail"], len(seeds), pooled)
    torch.cuda.synchronize()
    err0 = x.error()
    x.close()
    # the graph-captured climb with the p2p exchange
    g = D.ClimbGraph(s, cfg, seeds, exchange="p2p").capture()
    st, cands = g.run(steps)
    torch.cuda.synchronize()
    err1 = g.xchg.error()
    dist.barrier()
    if rank == 0:
        json.dump({"pooled": pooled.cpu().numpy().tobytes().hex(), "state": st.cpu().numpy().tobytes().hex(),
                   "cands": cands.cpu().numpy().tobytes().hex(), "err": [err0, err1]}, open(out_path, "w"))
    dist.barrier()
    g.xchg.close()
    s.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
