"""Worker for tests/test_gpu_lookahead.py (not collected): one rank of a seed-sharded lookahead climb.

Launched by torchrun with 2 ranks (gloo) sharing GPU 0: each rank simulates its seed slice of every round's
records, the per-rank aggregates are all-gathered and summed by K3L-step, and both ranks take the same two steps
per round.  Rank 0 writes the climb state after every step (hex) to the JSON file named by argv[1]."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    out_path, rounds = sys.argv[1], int(sys.argv[2])
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    from paper_2603_11340_b200 import dist as D
    from paper_2603_11340_b200 import inputs, sim
    cfg = inputs.config_c4(n_seeds=8, segment_len=400)
    lo, hi = D.seed_block(cfg.n_seeds, rank, world)
    s = sim.Simulator(cfg.workloads, device=0)
    la = D.LookaheadClimbGraph(s, cfg, cfg.seeds()[lo:hi], n_cand=32)
    traj = la.run_eager(rounds)
    dist.barrier()
    if rank == 0:
        with open(out_path, "w") as fh:
            json.dump({"states": [traj[i].numpy().tobytes().hex() for i in range(traj.shape[0])]}, fh)
    la.close()
    s.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
