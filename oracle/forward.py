"""Forward oracle -- TEST INFRASTRUCTURE ONLY.

What TD-Pipe computes: TD-Pipe changes *when* work runs, never *what* is
computed, so each request's output is the plain per-request greedy decode of
its prompt (§2.1: prefill "processes these tokens
concurrently to generate a new token", then "each step of the decode phase only
processes one new token").  The oracle is that definition written out, one
request at a time, in float64, with contiguous KV (F6) -- batch-, stage- and
phase-invariant by construction.

Model: Llama-style pre-norm decoder (the paper's Llama2 / Qwen2.5 models,
PAPER.md:506-508 Table 2):
  F1  x0 = E[tok]
  F2  per layer: a = RMSNorm(x; g1); q,k,v = a Wq^T, a Wk^T, a Wv^T (no bias);
      rotate-half RoPE at absolute 0-based position p with theta_i =
      10000^(-2i/hd); causal softmax(q k^T / sqrt(hd)) v with GQA head map
      h -> h // (H/Hkv); x += o Wo^T; m = RMSNorm(x; g2);
      x += (silu(m Wg^T) * (m Wu^T)) Wd^T
  F3  logits = RMSNorm(x; gf) Wlm^T  (untied)
  F4  greedy argmax, ties -> lowest index
  F5  logits of position t predict token t+1; prefill = last prompt position.
"""
from __future__ import annotations

import numpy as np


def rmsnorm(x: np.ndarray, g: np.ndarray, eps: float) -> np.ndarray:
    """RMSNorm(x) = x / sqrt(mean(x^2) + eps) * g   (F2)."""
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * g


def rope(x: np.ndarray, pos: np.ndarray, theta: float) -> np.ndarray:
    """Rotate-half RoPE (F2).  x: [T, nh, hd]; pos: [T] absolute positions.

    (x_i, x_{i+hd/2}) -> (x_i cos(p th_i) - x_{i+hd/2} sin(p th_i),
                          x_{i+hd/2} cos(p th_i) + x_i sin(p th_i)),
    th_i = theta^(-2i/hd), i < hd/2.
    """
    hd = x.shape[-1]
    half = hd // 2
    i = np.arange(half, dtype=np.float64)
    inv = theta ** (-2.0 * i / hd)
    ang = pos.astype(np.float64)[:, None] * inv[None, :]        # [T, half]
    c = np.cos(ang)[:, None, :]
    s = np.sin(ang)[:, None, :]
    x1 = x[..., :half]
    x2 = x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def causal_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray,
                     q_pos: np.ndarray, k_pos: np.ndarray) -> np.ndarray:
    """softmax(q k^T / sqrt(hd) + causal) v with GQA map h -> h // (H/Hkv).

    q: [Tq, H, hd]; k, v: [Tk, Hkv, hd]; query at q_pos attends keys with
    k_pos <= q_pos.  Returns [Tq, H, hd].
    """
    Tq, H, hd = q.shape
    Hkv = k.shape[1]
    G = H // Hkv
    out = np.empty_like(q)
    mask = k_pos[None, :] <= q_pos[:, None]                      # [Tq, Tk]
    scale = 1.0 / np.sqrt(hd)
    for h in range(H):
        kh = k[:, h // G, :]
        vh = v[:, h // G, :]
        s = (q[:, h, :] @ kh.T) * scale
        s = np.where(mask, s, -np.inf)
        s = s - s.max(axis=1, keepdims=True)
        p = np.exp(s)
        p = p / p.sum(axis=1, keepdims=True)
        out[:, h, :] = p @ vh
    return out


def silu(x: np.ndarray) -> np.ndarray:
    return x / (1.0 + np.exp(-x))


def layer_forward(x: np.ndarray, w: dict, shape, pos: np.ndarray) -> np.ndarray:
    """One decoder layer over a whole (prefix of a) request, F2.  x: [T, d]."""
    s = shape
    hd = s.head_dim
    T = x.shape[0]
    a = rmsnorm(x, w["g1"], s.rms_eps)
    q = (a @ w["wq"].T).reshape(T, s.n_heads, hd)
    k = (a @ w["wk"].T).reshape(T, s.n_kv_heads, hd)
    v = (a @ w["wv"].T).reshape(T, s.n_kv_heads, hd)
    q = rope(q, pos, s.rope_theta)
    k = rope(k, pos, s.rope_theta)
    o = causal_attention(q, k, v, pos, pos).reshape(T, s.n_heads * hd)
    x = x + o @ w["wo"].T
    m = rmsnorm(x, w["g2"], s.rms_eps)
    h = silu(m @ w["wg"].T) * (m @ w["wu"].T)
    return x + h @ w["wd"].T


def embed(weights, tokens: np.ndarray) -> np.ndarray:
    """F1: x0 = E[tok] (float64)."""
    return weights.embed()[np.asarray(tokens, dtype=np.int64)]


def logits_from_hidden(weights, x: np.ndarray) -> np.ndarray:
    """F3: logits = RMSNorm(x; gf) Wlm^T."""
    return rmsnorm(x, weights.final_norm(), weights.shape.rms_eps) @ weights.lm_head().T


def forward_hidden(weights, tokens: np.ndarray, layers=None, x0=None) -> np.ndarray:
    """Run `layers` (default: all) over the full causal sequence; returns x."""
    s = weights.shape
    T = len(tokens) if x0 is None else x0.shape[0]
    pos = np.arange(T, dtype=np.int64)
    x = embed(weights, tokens) if x0 is None else np.asarray(x0, dtype=np.float64)
    for l in (range(s.n_layers) if layers is None else layers):
        x = layer_forward(x, weights.layer(l), s, pos)
    return x


def sequence_logits(weights, tokens: np.ndarray) -> np.ndarray:
    """Logits at every position of `tokens` (causal): [T, V] (F3, F5)."""
    return logits_from_hidden(weights, forward_hidden(weights, tokens))


def greedy_argmax(logits: np.ndarray) -> np.ndarray:
    """F4: argmax with ties -> lowest index (numpy argmax semantics)."""
    return np.argmax(logits, axis=-1)


def greedy_generate(weights, prompt: np.ndarray, n_new: int):
    """Plain per-request greedy decode: returns (tokens, logits).

    Step j feeds the whole prefix again (no cache) -- the definition, slow.
    """
    toks = list(np.asarray(prompt, dtype=np.int64))
    out, lg = [], []
    for _ in range(n_new):
        l = sequence_logits(weights, np.array(toks))[-1]
        t = int(greedy_argmax(l))
        lg.append(l)
        out.append(t)
        toks.append(t)
    return np.array(out, dtype=np.int64), np.stack(lg) if lg else np.zeros((0, weights.shape.vocab))


def teacher_forced_logits(weights, prompt: np.ndarray, generated: np.ndarray) -> np.ndarray:
    """Logits that produced each generated token, given the GPU's own tokens (F8).

    Row j = logits at position len(prompt)-1+j of prompt ++ generated.
    """
    seq = np.concatenate([np.asarray(prompt, np.int64), np.asarray(generated, np.int64)])
    n = len(generated)
    if n == 0:
        return np.zeros((0, weights.shape.vocab))
    lg = sequence_logits(weights, seq[: len(prompt) + n - 1])
    return lg[len(prompt) - 1:]


def max_abs_rel(g: np.ndarray, o: np.ndarray) -> np.ndarray:
    """F8 row metric: max_i |g_i - o_i| / max(max_i |o_i|, 1e-6), per row."""
    g = np.atleast_2d(np.asarray(g, np.float64))
    o = np.atleast_2d(np.asarray(o, np.float64))
    return np.abs(g - o).max(axis=-1) / np.maximum(np.abs(o).max(axis=-1), 1e-6)


# ------------------------------------------------------------------------
# Stage view (PP layer partition): for td_stage_forward parity
# ------------------------------------------------------------------------
def partition_layers(n_layers: int, n_stages: int):
    """Balanced contiguous split, remainder to earlier stages."""
    if not 1 <= n_stages <= n_layers:
        raise ValueError("n_stages must be in [1, n_layers] (SPEC.md:118)")
    q, r = divmod(n_layers, n_stages)
    out, start = [], 0
    for s in range(n_stages):
        c = q + (1 if s < r else 0)
        out.append(range(start, start + c))
        start += c
    return out


def kv_bytes_per_token(n_layers: int, d_model: int, n_heads: int, n_kv_heads: int,
                       dtype_bytes: int = 2) -> int:
    """2 (K,V) x layers x (d x Hkv/H) x dtype bytes."""
    return 2 * n_layers * (d_model * n_kv_heads // n_heads) * dtype_bytes
