"""KV-cached forward -- TEST INFRASTRUCTURE ONLY.

The same definition as oracle/forward.py (F1-F5), computed the way F6 states
it: one request at a time with a contiguous per-request KV cache, so that a
decode step processes only its new token (§2.1: "each step of
the decode phase only processes one new token").  A decode step over several
requests stacks their single new rows for the row-independent projections
(norm, QKV, O, SwiGLU MLP, LM head act on each row separately) and attends
every request to its OWN cache only -- nothing crosses requests.

Pinned in tests/test_oracle_cached.py against the cache-less definition
(forward.sequence_logits) at every position (fp64: <= 1e-12 relative), so it
can stand in for it where the cache-less form is quadratic: the CPU timing
baseline of bench.py (SURVEY.md §8(d) "Oracle timing", numpy fp32) and long
teacher-forced references.  Shares no code with the CUDA path.
"""
from __future__ import annotations

import numpy as np

from oracle.forward import causal_attention, rmsnorm, rope, silu


class Cache:
    """Contiguous K/V of one request: per layer [T, Hkv, hd] (F6)."""

    def __init__(self, n_layers: int):
        self.k = [None] * n_layers
        self.v = [None] * n_layers
        self.T = 0


def _weights(W, l, dtype):
    key = ("_cached_dtype_layer", l, np.dtype(dtype).str)
    store = W.__dict__.setdefault("_cast", {})
    if key not in store:
        store[key] = {k: v.astype(dtype) for k, v in W.layer(l).items()}
    return store[key]


def _global(W, name, dtype):
    store = W.__dict__.setdefault("_cast", {})
    key = (name, np.dtype(dtype).str)
    if key not in store:
        store[key] = {"embed": W.embed, "gf": W.final_norm, "lm": W.lm_head}[name]().astype(dtype)
    return store[key]


def _layer_rows(x, w, s, pos, caches, seg):
    """One decoder layer (F2) for the new rows x [T, d] of several requests:
    rows seg[i]:seg[i+1] belong to caches[i] at absolute positions pos[...]."""
    hd = s.head_dim
    T = x.shape[0]
    a = rmsnorm(x, w["g1"], s.rms_eps)
    q = (a @ w["wq"].T).reshape(T, s.n_heads, hd)
    k = (a @ w["wk"].T).reshape(T, s.n_kv_heads, hd)
    v = (a @ w["wv"].T).reshape(T, s.n_kv_heads, hd)
    q = rope(q, pos, s.rope_theta).astype(x.dtype)
    k = rope(k, pos, s.rope_theta).astype(x.dtype)
    o = np.empty_like(q)
    for i, (c, l_) in enumerate(caches):
        r0, r1 = seg[i], seg[i + 1]
        kc = k[r0:r1] if c.k[l_] is None else np.concatenate([c.k[l_], k[r0:r1]])
        vc = v[r0:r1] if c.v[l_] is None else np.concatenate([c.v[l_], v[r0:r1]])
        c.k[l_], c.v[l_] = kc, vc
        kpos = np.arange(kc.shape[0], dtype=np.int64)
        o[r0:r1] = causal_attention(q[r0:r1], kc, vc, pos[r0:r1], kpos)
    x = x + o.reshape(T, s.n_heads * hd) @ w["wo"].T
    m = rmsnorm(x, w["g2"], s.rms_eps)
    h = silu(m @ w["wg"].T) * (m @ w["wu"].T)
    return x + h @ w["wd"].T


def forward_rows(W, caches, tokens_per_req, layers=None, dtype=np.float64, last_only=True):
    """Process the new tokens of several requests through `layers` (default
    all) with their caches; returns logits of each request's last new token
    ([n, V]) -- or of every new row when last_only is False ([T, V])."""
    s = W.shape
    layers = range(s.n_layers) if layers is None else layers
    seg = [0]
    pos = []
    for c, toks in zip(caches, tokens_per_req):
        pos.extend(range(c.T, c.T + len(toks)))
        seg.append(seg[-1] + len(toks))
    pos = np.asarray(pos, dtype=np.int64)
    E = _global(W, "embed", dtype)
    x = E[np.concatenate([np.asarray(t, np.int64) for t in tokens_per_req])]
    for l in layers:
        x = _layer_rows(x, _weights(W, l, dtype), s, pos, [(c, l) for c in caches], seg)
    for c, toks in zip(caches, tokens_per_req):
        c.T += len(toks)
    rows = np.asarray(seg[1:]) - 1 if last_only else np.arange(seg[-1])
    return rmsnorm(x[rows], _global(W, "gf", dtype), s.rms_eps) @ _global(W, "lm", dtype).T


def greedy_generate_cached(W, prompt, n_new: int, dtype=np.float64):
    """Per-request greedy decode with a KV cache: returns
    (tokens, logits) like forward.greedy_generate."""
    c = Cache(W.shape.n_layers)
    lg = forward_rows(W, [c], [np.asarray(prompt, np.int64)], dtype=dtype)[0]
    out, lgs = [], []
    for _ in range(n_new):
        t = int(np.argmax(lg))
        out.append(t)
        lgs.append(lg)
        if len(out) == n_new:
            break
        lg = forward_rows(W, [c], [[t]], dtype=dtype)[0]
    return np.array(out, dtype=np.int64), np.stack(lgs) if lgs else np.zeros((0, W.shape.vocab))
