"""NEXT-4 peer exchange (include/slo_sim.h slo_exchange_*) on the device.

Two ranks share the test box's one GPU (the mechanism — CUDA IPC peer pointers, P2P stores, release/acquire
epoch flags, double-buffered windows — is the same as across NVLink); their pooled aggregates and the climb
they drive must equal, bit for bit, the single-process result over all seeds."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_peer_exchange_two_ranks_matches_single_process(tmp_path):
    import __graft_entry__
    __graft_entry__.build()
    from paper_2603_11340_b200 import inputs, sim
    from paper_2603_11340_b200.dist import hillclimb
    steps = 4
    out = tmp_path / "rank0.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tests", "exchange_worker.py"),
           str(out), str(steps)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=420)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    got = json.load(open(out))
    assert got["err"] == [0, 0]
    cfg = inputs.config_c4(n_seeds=8, segment_len=400)
    s = sim.Simulator(cfg.workloads, device=0)
    cands = s.candidates(cfg.extra["space"], cfg.knobs[0], 32)
    o = s.run_batch(cands, sim.seeds_tensor(cfg.seeds()), cfg.segment_len)
    agg = s.aggregate(o["detail"], 32, cfg.n_seeds)
    torch.cuda.synchronize()
    assert agg.cpu().numpy().tobytes().hex() == got["pooled"]
    st, c = hillclimb(s, cfg, steps, cfg.seeds())
    torch.cuda.synchronize()
    assert st.cpu().numpy().tobytes().hex() == got["state"]
    assert c.cpu().numpy().tobytes().hex() == got["cands"]
    s.close()
