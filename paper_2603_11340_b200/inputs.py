"""Seeded synthetic input generators — shared by the CUDA path, the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no Philox, no transforms, no event rules, no scoring):
it only produces plain-integer descriptions of workloads, knob records, seeds and config
grids.  Both sides marshal these into their own structs.

Shapes follow the paper's workloads:
* LL: TinyLlama-on-vLLM-like single replayed prompt, 64-token output cap, steady load;
* SIM: the simulator's "large prompt, moderate output" log-normal lengths;
* STRESS: means scaled 1.5x plus a burstier (MMPP-2) arrival process (BJ config 5).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, asdict
from typing import Dict, List, Sequence

U64 = (1 << 64) - 1
NO_ARRIVALS = U64          # mean_gap_q16 sentinel: a state without arrivals (on/off "off")

KNOB_FIELDS = ("conc", "max_num_seqs", "draft_len", "spec_on", "draft_width", "workload",
               "rate_scale_q8", "accept_q16", "max_wait_us")


# --------------------------------------------------------------------------------------------
# seeds
# --------------------------------------------------------------------------------------------
def splitmix64(x: int) -> int:
    """SplitMix64 finaliser (Steele et al.), used only to spread replica seeds."""
    x = (x + 0x9E3779B97F4A7C15) & U64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & U64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & U64
    return z ^ (z >> 31)


def seeds(n: int, offset: int = 0) -> List[int]:
    """seed_s = SplitMix64(0x5EED0000 + s) for s in [offset, offset + n)."""
    return [splitmix64(0x5EED0000 + s) for s in range(offset, offset + n)]


# --------------------------------------------------------------------------------------------
# length tables ("prompt and output lengths follow log-normal distributions")
# --------------------------------------------------------------------------------------------
def _phi(z: float) -> float:
    return 0.5 * math.erfc(-z / math.sqrt(2.0))


def lognormal_table(mu: float, sigma: float, lo: int, hi: int) -> Dict:
    """Integer CDF table for round(LogNormal(mu, sigma)) clamped to [lo, hi].

    Mass of value v = log-normal mass on [v - 1/2, v + 1/2); the end bins absorb the tails.
    Returns {"lo": lo, "cw": [cut points]} with len(cw) = (#values - 1); the sampled length for a
    uniform u32 word u is lo + #{l : cw[l] <= u}.  Cut points that would reach 2^32 are dropped
    (those values are unreachable).
    """
    assert 1 <= lo <= hi
    if sigma == 0.0:
        v = min(hi, max(lo, int(round(math.exp(mu)))))
        return {"lo": v, "cw": []}
    cw = []
    for v in range(lo, hi):
        cdf = _phi((math.log(v + 0.5) - mu) / sigma)
        c = int(round(cdf * 2.0 ** 32))
        if c >= 1 << 32:
            break
        if cw and c < cw[-1]:
            c = cw[-1]
        cw.append(c)
    return {"lo": lo, "cw": cw}


def point_mass(v: int) -> Dict:
    return {"lo": int(v), "cw": []}


# --------------------------------------------------------------------------------------------
# workloads
# --------------------------------------------------------------------------------------------
def mean_gap_q16(rate_per_s: float) -> int:
    """Mean inter-arrival gap in Q48.16 microseconds for a rate in requests/s."""
    return int(round(1e6 / rate_per_s * 65536.0))


LL_TIMING = dict(pre_base_us=2000, pre_tok_us=60, dec_base_us=7000, dec_seq_us=200,
                 dr_base_us=1500, dr_seq_us=50, ver_base_us=8000, ver_seq_us=300, ver_tok_us=20,
                 noise_step_ppm=338)

SIM_TIMING = dict(pre_base_us=0, pre_tok_us=125, dec_base_us=4000, dec_seq_us=400,
                  dr_base_us=1000, dr_seq_us=0, ver_base_us=6000, ver_seq_us=500, ver_tok_us=0,
                  noise_step_ppm=338)


def workload(kind=0, rate=10.0, prompt=None, output=None, timing=None, stream_id=0,
             start_state=0, rate_hi=None, rate_lo=None, sojourn_us=(2_000_000, 2_000_000)) -> Dict:
    if kind == 0:
        gaps = [mean_gap_q16(rate), mean_gap_q16(rate)]
    else:
        gaps = [mean_gap_q16(rate_hi) if rate_hi else NO_ARRIVALS,
                mean_gap_q16(rate_lo) if rate_lo else NO_ARRIVALS]
    return {
        "arrivals": {"kind": kind, "start_state": start_state, "mean_gap_q16": gaps,
                     "mean_sojourn_us": [int(sojourn_us[0]), int(sojourn_us[1])]},
        "prompt": prompt if prompt is not None else point_mass(40),
        "output": output if output is not None else lognormal_table(math.log(80.0), 0.4, 1, 64),
        "timing": dict(timing if timing is not None else LL_TIMING),
        "stream_id": int(stream_id),
        "batching": 0,
    }


def preset_ll(rate=10.0, stream_id=0) -> Dict:
    """LL: Poisson `rate` req/s, prompt 40 tokens, output min(64, round(LN(ln 80, 0.4)))."""
    return workload(kind=0, rate=rate, prompt=point_mass(40),
                    output=lognormal_table(math.log(80.0), 0.4, 1, 64),
                    timing=LL_TIMING, stream_id=stream_id)


def preset_sim(rate=12.0, stream_id=0) -> Dict:
    """SIM: S:397 defaults — prompt mean 512 (sigma .6, [16,4096]), output mean 64 (sigma .6, [1,512])."""
    s = 0.6
    return workload(kind=0, rate=rate,
                    prompt=lognormal_table(math.log(512.0) - s * s / 2, s, 16, 4096),
                    output=lognormal_table(math.log(64.0) - s * s / 2, s, 1, 512),
                    timing=SIM_TIMING, stream_id=stream_id)


def preset_closed(stream_id=0, think_us=None) -> Dict:
    """CLOSED: the paper's live client: a single replayed prompt, 64-token output cap and a
    closed loop of `conc` users with zero think time (arrival kind 3); latency from issue.
    With `think_us` (mean, microseconds; 0 allowed) every user thinks an exponential time between a
    completion and its next request (arrival kind 4; static or continuous batching)."""
    w = preset_ll(stream_id=stream_id)
    w["arrivals"]["kind"] = 3
    if think_us is not None:
        w["arrivals"]["kind"] = 4
        w["arrivals"]["mean_gap_q16"] = [int(round(think_us * 65536)), NO_ARRIVALS]
    return w


def continuous(w: Dict) -> Dict:
    """The same workload served with continuous (iteration-level, vLLM-style) batching."""
    w = dict(w)
    w["batching"] = 1
    return w


def preset_stress(rate=10.0, stream_id=0, kind=1) -> Dict:
    """STRESS: LL lengths x1.5, MMPP-2 with lambda_H = 1.8 rate, lambda_L = 0.2 rate, 2 s sojourns."""
    return workload(kind=kind, prompt=point_mass(60),
                    output=lognormal_table(math.log(120.0), 0.4, 1, 96),
                    timing=LL_TIMING, stream_id=stream_id,
                    rate_hi=1.8 * rate, rate_lo=0.2 * rate)


# --------------------------------------------------------------------------------------------
# knob records
# --------------------------------------------------------------------------------------------
def knobs(conc=8, max_num_seqs=8, draft_len=0, spec_on=0, draft_width=1, workload=0,
          rate_scale_q8=256, accept_q16=32768, max_wait_us=0) -> Dict:
    return dict(conc=conc, max_num_seqs=max_num_seqs, draft_len=draft_len, spec_on=spec_on,
                draft_width=draft_width, workload=workload, rate_scale_q8=rate_scale_q8,
                accept_q16=accept_q16, max_wait_us=max_wait_us)


def q16(x: float) -> int:
    return int(round(x * 65536.0))


PAD_KNOBS = knobs(conc=0)          # an always-invalid record (used to pad candidate lists)


# --------------------------------------------------------------------------------------------
# BASELINE.json configs
# --------------------------------------------------------------------------------------------
@dataclass
class Config:
    name: str
    workloads: List[Dict]
    knobs: List[Dict]
    n_seeds: int
    segment_len: int
    warmup_len: int = 0
    slo_us: int = 1_200_000
    seed_offset: int = 0
    extra: Dict = field(default_factory=dict)

    @property
    def replicas(self) -> int:
        return len(self.knobs) * self.n_seeds

    @property
    def requests(self) -> int:
        return self.replicas * (self.segment_len + self.warmup_len)

    def seeds(self) -> List[int]:
        return seeds(self.n_seeds, self.seed_offset)


def config_c1() -> Config:
    """C1: single replica, C=8, B=16, no speculation, Poisson 10 req/s, 2,000 requests, SLO 1.2 s."""
    return Config("C1", [preset_ll()], [knobs(conc=8, max_num_seqs=16)], 1, 2000)


def config_c2(n_seeds=64, segment_len=10_000) -> Config:
    """C2: 16 concurrency x 8 batch limits x 4 speculation settings x 64 seeds, 10k requests."""
    ks = []
    for c in range(1, 17):
        for b in range(2, 17, 2):
            for (on, g) in ((0, 0), (1, 4), (1, 8), (1, 16)):
                ks.append(knobs(conc=c, max_num_seqs=b, draft_len=g, spec_on=on, accept_q16=q16(0.5)))
    return Config("C2", [preset_ll()], ks, n_seeds, segment_len)


def config_c2_cont(n_seeds=64, segment_len=10_000) -> Config:
    """C2's knob grid with continuous (iteration-level) batching (SV §8(f) NEXT-2)."""
    c = config_c2(n_seeds, segment_len)
    return Config("C2-cont", [continuous(preset_ll())], c.knobs, n_seeds, segment_len)


def config_c3(n_seeds=256, segment_len=10_000) -> Config:
    """C3: draft length 0-8 x acceptance .3-.9, C = B = 8 (K0), 256 seeds."""
    ks = []
    for g in range(0, 9):
        for a in (0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9):
            ks.append(knobs(conc=8, max_num_seqs=8, draft_len=g, spec_on=1 if g else 0,
                            accept_q16=q16(a)))
    return Config("C3", [preset_ll()], ks, n_seeds, segment_len)


def config_c5(n_seeds=16, segment_len=2000, limit=None, stride=1) -> Config:
    """C5: STRESS grid 25 C x 25 B x 8 gamma x 5 alpha x 40 rate levels (2..80 req/s) = 10^6 configs.
    `stride` keeps every stride-th config of the full grid (a sample spanning every knob), `limit` the first
    `limit` configs after striding."""
    ks = []
    idx = -1
    gam = (0, 1, 2, 3, 4, 6, 8, 12)
    alph = (0.3, 0.45, 0.6, 0.75, 0.9)
    rates = [2.0 + i * (78.0 / 39.0) for i in range(40)]
    for c in range(1, 26):
        for b in range(1, 26):
            for g in gam:
                for a in alph:
                    for r in rates:
                        idx += 1
                        if idx % stride:
                            continue
                        ks.append(knobs(conc=c, max_num_seqs=b, draft_len=g, spec_on=1 if g else 0,
                                        accept_q16=q16(a), rate_scale_q8=max(1, int(round(r / 10.0 * 256)))))
                        if limit is not None and len(ks) >= limit:
                            return Config("C5", [preset_stress()], ks, n_seeds, segment_len)
    return Config("C5", [preset_stress()], ks, n_seeds, segment_len)


# hill-climb spaces (P:142 live space; S:56/S:83 sim space), dims: conc, max_num_seqs, draft_len,
# draft_width, max_wait_us
SPACE_LIVE = dict(stencil=0, lo=[2, 4, 0, 1, 0], hi=[16, 16, 16, 4, 50_000], step=[2, 3, 4, 1, 10_000])
SPACE_SIM = dict(stencil=1, lo=[1, 1, 2, 1, 0], hi=[32, 32, 16, 4, 50_000], step=[2, 4, 2, 1, 10_000])
SPACE_WIDE32 = dict(stencil=2, lo=[1, 1, 0, 1, 0], hi=[32, 32, 16, 4, 50_000], step=[2, 3, 4, 1, 10_000])

K0 = knobs(conc=8, max_num_seqs=8, draft_len=8, spec_on=1, accept_q16=q16(0.5))   # Alg. 1 init

SCORE_DEFAULTS = dict(lambda_milli=5000, w_conc_micro=10_000, w_max_micro=10_000, w_spec_micro=20_000,
                      delta_micro=20_000, slo_us=1_200_000, strict_alg1=1, viol_mult=1, k_max=16,
                      w_W_micro=0, w_k_micro=0, ema_beta_q16=0)
# the paper's simulator controller: 10 lambda violation term,
# draft/verifier cost, EMA(beta = 0.5) of the current point's p99
SCORE_SIM = dict(SCORE_DEFAULTS, viol_mult=10, w_W_micro=20_000, w_k_micro=5_000, ema_beta_q16=32768)


def config_c4(n_seeds=128, segment_len=5000) -> Config:
    """C4: hill-climb, 32 candidates (wide-32 stencil) x 128 seeds per step, 5k-request segments."""
    return Config("C4", [preset_ll()], [dict(K0)], n_seeds, segment_len,
                  extra=dict(space=SPACE_WIDE32, score=SCORE_DEFAULTS, n_cand=32))


def random_knobs(rng, n_wl=1, spec=True, max_wait=True) -> Dict:
    """A random valid knob record (for parity sampling)."""
    g = rng.randrange(0, 17) if spec else 0
    return knobs(conc=rng.randrange(1, 33), max_num_seqs=rng.randrange(1, 33), draft_len=g,
                 spec_on=rng.randrange(0, 2) if g else rng.randrange(0, 2), draft_width=rng.randrange(1, 5),
                 workload=rng.randrange(0, n_wl), rate_scale_q8=rng.randrange(32, 1024),
                 accept_q16=rng.choice([0, 65536, rng.randrange(0, 65537)]),
                 max_wait_us=rng.choice([0, 0, rng.randrange(0, 50_001)]) if max_wait else 0)
