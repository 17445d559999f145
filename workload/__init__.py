"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no forward math, no scheduling
rule).  It only draws the inputs both sides consume, so that the oracle
(`oracle/`) and the product path (`paper_2506_10470_b200/`) never share code
beyond it:

* model shapes of the BASELINE.json configs (SURVEY.md §8 shape table),
* request sets with ShareGPT-like length mixes (§4.1 "filter
  input sentences with a length of less than 1024 tokens"; SPEC.md:43 lognormal
  stand-in, clamped not rejected SPEC.md:60),
* output-length predictions from a percentile-bucket stand-in for the BERT
  classifier (§3.3 "[P0, P25) to [P99, +)", "average value of the
  category"; adjacent-bucket error 0.45 -> accuracy ~0.55),
* a synthetic, frozen profile table (decode-step ns per batch size, prefill ns
  per token count) used by the scheduler-parity tests.

Weights are not drawn here: both sides implement the counter-based splitmix64
recipe of SURVEY.md §8(c) F9 independently (oracle/weights.py, csrc init kernel).
"""
from __future__ import annotations

from dataclasses import dataclass, field, asdict
from typing import List, Optional

import numpy as np


# --------------------------------------------------------------------------
# Model shapes (Table 2 for 13B / 70B)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class ModelShape:
    name: str
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    d_ffn: int
    vocab: int
    rope_theta: float = 10000.0
    rms_eps: float = 1e-5
    max_seq_len: int = 4096

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    def with_layers(self, n: int) -> "ModelShape":
        d = asdict(self)
        d["n_layers"] = n
        d["name"] = f"{self.name}-L{n}"
        return ModelShape(**d)


SHAPES = {
    # C1: tiny Llama-style (BASELINE.json configs[0]); F=256 is SURVEY's proposal.
    "tiny": ModelShape("tiny", 2, 64, 4, 4, 256, 256, max_seq_len=512),
    # C1 GQA variant used by the oracle pins and GPU parity (H/Hkv = 2).
    "tiny_gqa": ModelShape("tiny_gqa", 2, 64, 4, 2, 256, 256, max_seq_len=512),
    # C2 Llama-2-7B
    "llama2_7b": ModelShape("llama2_7b", 32, 4096, 32, 32, 11008, 32000),
    # C3 Llama-2-13B
    "llama2_13b": ModelShape("llama2_13b", 40, 5120, 40, 40, 13824, 32000),
    # C4 OPT-30B-shaped, SwiGLU param-matched F (SURVEY.md §8 proposal)
    "opt30b_shaped": ModelShape("opt30b_shaped", 48, 7168, 56, 56, 19200, 50272),
    # C5 Llama-2-70B, GQA 64/8
    "llama2_70b": ModelShape("llama2_70b", 80, 8192, 64, 8, 28672, 32000),
}


# --------------------------------------------------------------------------
# Requests
# --------------------------------------------------------------------------
@dataclass
class Request:
    rid: int
    prompt: np.ndarray          # int32 token ids, uniform in [0, V)
    max_new_tokens: int         # ground-truth stop length N (EOS disabled)
    predicted_len: int          # P, predicted output length (>= 1)


@dataclass
class Workload:
    requests: List[Request]
    seed: int
    recipe: dict = field(default_factory=dict)

    @property
    def prompt_lens(self) -> np.ndarray:
        return np.array([len(r.prompt) for r in self.requests], dtype=np.int64)

    @property
    def output_lens(self) -> np.ndarray:
        return np.array([r.max_new_tokens for r in self.requests], dtype=np.int64)


def _lognormal_lengths(rng: np.random.Generator, n: int, mu: float, sigma: float,
                       lo: int, hi: int) -> np.ndarray:
    """clip(rint(lognormal(mu, sigma)), lo, hi) -- SPEC.md:43, clamped."""
    x = rng.lognormal(mean=mu, sigma=sigma, size=n)
    return np.clip(np.rint(x), lo, hi).astype(np.int64)


def fit_buckets(train_out: np.ndarray, percentiles=(25, 50, 75, 90, 95, 99)):
    """Nearest-rank percentile boundaries + per-bucket means.

    Buckets are [P0,P25), [P25,P50), ..., [P99, +inf).
    Returns (boundaries, means) with len(means) == len(boundaries) + 1.
    """
    s = np.sort(np.asarray(train_out, dtype=np.int64))
    n = len(s)
    bnd = []
    for p in percentiles:
        k = max(1, int(np.ceil(p / 100.0 * n)))   # nearest rank (1-based)
        bnd.append(int(s[k - 1]))
    bnd = np.array(bnd, dtype=np.int64)
    idx = np.searchsorted(bnd, s, side="right")
    means = []
    for b in range(len(bnd) + 1):
        m = s[idx == b]
        if len(m) == 0:  # empty bucket (ties in the data): borrow the boundary
            m = np.array([bnd[min(b, len(bnd) - 1)]])
        means.append(int(max(1, round(float(m.mean())))))
    return bnd, np.array(means, dtype=np.int64)


def bucket_predict(true_out: np.ndarray, bnd: np.ndarray, means: np.ndarray,
                   rng: np.random.Generator, adjacent_error: float) -> np.ndarray:
    """Bucket-mean predictor with adjacent-bucket misclassification."""
    b = np.searchsorted(bnd, true_out, side="right")
    flip = rng.random(len(b)) < adjacent_error
    step = np.where(rng.random(len(b)) < 0.5, -1, 1)
    b2 = np.clip(b + np.where(flip, step, 0), 0, len(means) - 1)
    return np.maximum(means[b2], 1)


def generate_workload(n: int, vocab: int, seed: int, *, in_mu=5.0, in_sigma=1.0,
                      out_mu=4.5, out_sigma=1.0, in_max=1023, out_max=1024,
                      predictor: str = "bucket", adjacent_error: float = 0.45,
                      fixed_in: Optional[int] = None, fixed_out: Optional[int] = None,
                      uniform_in: Optional[tuple] = None,
                      uniform_out: Optional[tuple] = None) -> Workload:
    """ShareGPT-shaped request set (SURVEY.md §8(d) "Synthetic inputs").

    predictor: "oracle" (P = N, exactness runs), "bucket" (bucket means with
    adjacent-bucket error), or "noisy" (N x lognormal(0, 0.3)).
    """
    rng = np.random.default_rng(seed)
    if fixed_in is not None:
        lin = np.full(n, fixed_in, dtype=np.int64)
    elif uniform_in is not None:
        lin = rng.integers(uniform_in[0], uniform_in[1] + 1, size=n).astype(np.int64)
    else:
        lin = _lognormal_lengths(rng, n, in_mu, in_sigma, 1, in_max)
    if fixed_out is not None:
        lout = np.full(n, fixed_out, dtype=np.int64)
    elif uniform_out is not None:
        lout = rng.integers(uniform_out[0], uniform_out[1] + 1, size=n).astype(np.int64)
    else:
        lout = _lognormal_lengths(rng, n, out_mu, out_sigma, 1, out_max)
    prompts = [rng.integers(0, vocab, size=int(L)).astype(np.int32) for L in lin]
    if predictor == "oracle":
        pred = lout.copy()
    elif predictor == "bucket":
        trng = np.random.default_rng(seed + 1_000_003)
        train = _lognormal_lengths(trng, 4096, out_mu, out_sigma, 1, out_max)
        bnd, means = fit_buckets(train)
        pred = bucket_predict(lout, bnd, means, np.random.default_rng(seed + 7), adjacent_error)
    elif predictor == "noisy":
        nrng = np.random.default_rng(seed + 11)
        pred = np.maximum(1, np.rint(lout * nrng.lognormal(0.0, 0.3, size=n))).astype(np.int64)
    else:
        raise ValueError(predictor)
    reqs = [Request(i, prompts[i], int(lout[i]), int(max(1, pred[i]))) for i in range(n)]
    recipe = dict(n=n, vocab=vocab, seed=seed, in_mu=in_mu, in_sigma=in_sigma, out_mu=out_mu,
                  out_sigma=out_sigma, in_max=in_max, out_max=out_max, predictor=predictor,
                  adjacent_error=adjacent_error, fixed_in=fixed_in, fixed_out=fixed_out,
                  uniform_in=uniform_in, uniform_out=uniform_out)
    return Workload(reqs, seed, recipe)


def config_workload(name: str) -> Workload:
    """The request sets of BASELINE.json configs."""
    if name == "C1":      # 8 requests, prompt 16 / output 16
        return generate_workload(8, 256, 0, fixed_in=16, fixed_out=16, predictor="oracle")
    if name == "C2":
        return generate_workload(256, 32000, 2)
    if name == "C3":
        return generate_workload(1024, 32000, 3)
    if name == "C4":
        return generate_workload(2048, 50272, 4, out_mu=6.2, out_sigma=0.6, out_max=2048)
    if name == "C5":
        return generate_workload(4096, 32000, 5)
    raise KeyError(name)


def random_tiny_workload(seed: int, vocab: int = 256, n_max: int = 12, len_max: int = 40):
    """C1a-style random tiny workloads for scheduler parity."""
    rng = np.random.default_rng(10_000 + seed)
    n = int(rng.integers(1, n_max + 1))
    return generate_workload(n, vocab, seed, uniform_in=(1, len_max), uniform_out=(1, len_max),
                             predictor=("oracle" if seed % 3 == 0 else "noisy"))


# --------------------------------------------------------------------------
# Synthetic frozen profile table (input data for scheduler parity tests)
# --------------------------------------------------------------------------
def synthetic_profile(b_max: int, k_max: int, dec_base_ns=2_000_000, dec_per_req_ns=10_000,
                      pre_base_ns=500_000, pre_per_tok_ns=9_000, knee: int = 0):
    """Dense int64 tables Tdec[1..b_max], Tpre[1..k_max] (index 0 unused = 0).

    Tdec[b] = base + per_req*b (SURVEY.md §8(c) pins' toy table), optionally with
    a flat memory-bound plateau below `knee` so Achieved(b) saturates.
    """
    b = np.arange(b_max + 1, dtype=np.int64)
    tdec = dec_base_ns + dec_per_req_ns * np.maximum(b, knee)
    tdec[0] = 0
    k = np.arange(k_max + 1, dtype=np.int64)
    tpre = pre_base_ns + pre_per_tok_ns * k
    tpre[0] = 0
    return tdec.astype(np.int64), tpre.astype(np.int64)


def write_profile_csv(path: str, tdec: np.ndarray, tpre: np.ndarray) -> None:
    """CSV: lines `D,b,ns` and `P,k,ns` (the format td_profile writes)."""
    with open(path, "w") as f:
        for b in range(1, len(tdec)):
            f.write(f"D,{b},{int(tdec[b])}\n")
        for k in range(1, len(tpre)):
            f.write(f"P,{k},{int(tpre[k])}\n")


def read_profile_csv(path: str):
    d, p = {}, {}
    with open(path) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            kind, i, ns = line.split(",")
            (d if kind == "D" else p)[int(i)] = int(ns)
    tdec = np.zeros(max(d) + 1, dtype=np.int64)
    tpre = np.zeros(max(p) + 1, dtype=np.int64)
    for b, v in d.items():
        tdec[b] = v
    for k, v in p.items():
        tpre[k] = v
    return tdec, tpre
