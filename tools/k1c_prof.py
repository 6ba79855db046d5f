"""K1c pass statistics on the C2-cont grid (profiling build: tools/build_variant.sh prof -DSLO_K1C_PROF)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_11340_b200 import inputs, sim, _lib

cfg = inputs.config_c2_cont()
S = sim.Simulator(cfg.workloads, device=0)
dev = torch.device("cuda", 0)
seeds = sim.seeds_tensor(cfg.seeds(), device=dev)
L = _lib.lib()
buf = (ctypes.c_ulonglong * 16)()
names = ["warp trips", "group trips (active)", "need_s groups", "prefill groups", "decode groups", "sum K",
         "K by completion", "K by prefill", "noise refills (warp)", "finishers", "warp trips w/ prefill region",
         "warp trips w/ decode region", "warp trips w/ finish region", "sum nrun (decode groups)",
         "K == 2G", "active groups per warp trip (sum)"]
for sub, ks in (("all", cfg.knobs), ("C>=3", [k for k in cfg.knobs if k["conc"] >= 3])):
    kt = sim.knobs_tensor(ks, device=dev)
    out = S.alloc_outputs(len(ks) * cfg.n_seeds)
    L.slo_debug_k1c_prof(buf, 1)
    S.run_batch(kt, seeds, cfg.segment_len, out=out)
    torch.cuda.synchronize()
    L.slo_debug_k1c_prof(buf, 1)
    v = list(buf)
    print("==", sub, len(ks) * cfg.n_seeds, "replicas")
    for n, x in zip(names, v):
        print(f"  {n:36s} {x:16,d}")
    print(f"  mean K {v[5] / max(v[4], 1):.2f}, decode groups / warp trip {v[4] / max(v[11], 1):.2f}, "
          f"active groups / warp trip {v[15] / max(v[0], 1):.2f}, mean nrun {v[13] / max(v[4], 1):.2f}")
