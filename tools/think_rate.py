"""Throughput of the think-time closed loops against zero think time on C2's knob grid."""
import torch, sys
sys.path.insert(0, ".")
from paper_2603_11340_b200 import inputs, sim
for cont in (0, 1):
    for think in (None, 300_000):
        w = inputs.preset_closed(think_us=think)
        if cont:
            w = inputs.continuous(w)
        ks = [inputs.knobs(conc=c, max_num_seqs=b, draft_len=g, spec_on=int(g > 0), accept_q16=32768)
              for c in range(1, 17) for b in range(2, 17, 2) for g in (0, 4, 8, 16)]
        seeds = inputs.seeds(64, 0)
        s = sim.Simulator([w], device=0)
        kt, st = sim.knobs_tensor(ks), sim.seeds_tensor(seeds)
        for _ in range(2):
            s.run_batch(kt, st, 10_000)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            s.run_batch(kt, st, 10_000)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"batching={'continuous' if cont else 'static'} think={think}: {ms:.1f} ms/step, "
              f"{len(ks) * len(seeds) * 10_000 / ms * 1e3:.3e} simulated req/s")
        s.close()
