"""F9 weight recipe, oracle side -- TEST INFRASTRUCTURE ONLY.

Random-init weights (BASELINE.json north_star: "random-init weights") are drawn
from a counter-based generator so that oracle and GPU hold bit-identical bf16
values without sharing code:

    u = (splitmix64(seed ^ (tensor_id << 40) ^ i) >> 40) * 2^-24,   i = row-major
        index in the logical [out, in] matrix (or [d] vector)
    projection:  w = bf16_rne( fp32( sqrt_f32(3/fan_in) * (2u-1) ) )
    norm gain:   g = bf16_rne( fp32( 1 + fp32(0.1 * (2u-1)) ) )
    embedding:   e = bf16_rne( 2u-1 )

All fp32 steps are single IEEE roundings (no fused multiply-add).
Tensor ids: embed 0; layer l: 1+9l + {0 g1, 1 Wq, 2 Wk, 3 Wv, 4 Wo, 5 g2,
6 Wg, 7 Wu, 8 Wd}; final norm 1+9L; LM head 2+9L.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
DEFAULT_SEED = 0x5EED_7D


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser (Steele/Lea/Flood), uint64 with wrap-around."""
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform01(seed: int, tensor_id: int, n: int, start: int = 0) -> np.ndarray:
    """u in [0,1) with 24 random bits, as float32 (exact)."""
    i = np.arange(start, start + n, dtype=np.uint64)
    key = np.uint64(seed) ^ (np.uint64(tensor_id) << np.uint64(40))
    h = splitmix64(key ^ i)
    k = (h >> np.uint64(40)).astype(np.float32)          # < 2^24, exact in fp32
    return k * np.float32(2.0 ** -24)


def bf16_rne(x: np.ndarray) -> np.ndarray:
    """Round float32 -> bfloat16 (nearest-even); returned as float32 values."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)) << np.uint64(16)
    return r.astype(np.uint32).view(np.float32)


def proj_weight(seed: int, tensor_id: int, n_out: int, fan_in: int) -> np.ndarray:
    u = uniform01(seed, tensor_id, n_out * fan_in)
    s = np.sqrt(np.float32(3.0) / np.float32(fan_in), dtype=np.float32)
    v = (np.float32(2.0) * u - np.float32(1.0)).astype(np.float32)   # exact
    w = (s * v).astype(np.float32)
    return bf16_rne(w).reshape(n_out, fan_in)


def norm_gain(seed: int, tensor_id: int, n: int) -> np.ndarray:
    u = uniform01(seed, tensor_id, n)
    v = (np.float32(2.0) * u - np.float32(1.0)).astype(np.float32)
    t = (np.float32(0.1) * v).astype(np.float32)
    return bf16_rne((np.float32(1.0) + t).astype(np.float32))


def embedding(seed: int, vocab: int, d: int) -> np.ndarray:
    u = uniform01(seed, 0, vocab * d)
    v = (np.float32(2.0) * u - np.float32(1.0)).astype(np.float32)
    return bf16_rne(v).reshape(vocab, d)


def tensor_id(layer: int, which: str, n_layers: int) -> int:
    order = ["g1", "wq", "wk", "wv", "wo", "g2", "wg", "wu", "wd"]
    if which == "embed":
        return 0
    if which == "gf":
        return 1 + 9 * n_layers
    if which == "lm":
        return 2 + 9 * n_layers
    return 1 + 9 * layer + order.index(which)


class OracleWeights:
    """All weights of a shape as float64 arrays (values exactly the bf16 ones).

    Generated lazily per layer so that 7B/70B-shaped single layers fit in RAM.
    """

    def __init__(self, shape, seed: int = DEFAULT_SEED):
        self.shape = shape
        self.seed = seed
        self._layers = {}
        self._embed = None
        self._gf = None
        self._lm = None

    def embed(self) -> np.ndarray:
        if self._embed is None:
            self._embed = embedding(self.seed, self.shape.vocab, self.shape.d_model).astype(np.float64)
        return self._embed

    def final_norm(self) -> np.ndarray:
        if self._gf is None:
            self._gf = norm_gain(self.seed, tensor_id(0, "gf", self.shape.n_layers),
                                 self.shape.d_model).astype(np.float64)
        return self._gf

    def lm_head(self) -> np.ndarray:
        if self._lm is None:
            s = self.shape
            self._lm = proj_weight(self.seed, tensor_id(0, "lm", s.n_layers), s.vocab,
                                   s.d_model).astype(np.float64)
        return self._lm

    def layer(self, l: int) -> dict:
        if l not in self._layers:
            s = self.shape
            hd = s.head_dim
            L = s.n_layers
            tid = lambda w: tensor_id(l, w, L)
            self._layers[l] = {
                "g1": norm_gain(self.seed, tid("g1"), s.d_model).astype(np.float64),
                "wq": proj_weight(self.seed, tid("wq"), s.n_heads * hd, s.d_model).astype(np.float64),
                "wk": proj_weight(self.seed, tid("wk"), s.n_kv_heads * hd, s.d_model).astype(np.float64),
                "wv": proj_weight(self.seed, tid("wv"), s.n_kv_heads * hd, s.d_model).astype(np.float64),
                "wo": proj_weight(self.seed, tid("wo"), s.d_model, s.n_heads * hd).astype(np.float64),
                "g2": norm_gain(self.seed, tid("g2"), s.d_model).astype(np.float64),
                "wg": proj_weight(self.seed, tid("wg"), s.d_ffn, s.d_model).astype(np.float64),
                "wu": proj_weight(self.seed, tid("wu"), s.d_ffn, s.d_model).astype(np.float64),
                "wd": proj_weight(self.seed, tid("wd"), s.d_model, s.d_ffn).astype(np.float64),
            }
        return self._layers[l]

    def drop_layer(self, l: int) -> None:
        self._layers.pop(l, None)
