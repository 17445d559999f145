"""Pins for the forward oracle -- CPU only.

Each test checks the oracle against something other than itself: a library
routine (HF LlamaForCausalLM, torch's bf16 cast), published generator test
vectors, closed forms and invariants, or numbers printed in the paper.
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import forward as F
from oracle import weights as Wt
from workload import SHAPES, ModelShape

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


# ----------------------------------------------------------------- F9 weights
def test_splitmix64_reference_vectors():
    g = np.uint64(0x9E3779B97F4A7C15)
    with np.errstate(over="ignore"):
        xs = np.array([0, g, g * np.uint64(2)], dtype=np.uint64)
    got = [format(int(v), "016x") for v in Wt.splitmix64(xs)]
    assert got == GOLD["splitmix64"]["outputs_hex"]


def test_bf16_rne_matches_torch_cast():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(100000).astype(np.float32),
                        # exact ties: low 16 bits == 0x8000 with odd / even upper halves
                        np.array([0x3F808000, 0x3F818000, 0xBF808000, 0x40490000], np.uint32).view(np.float32)])
    ours = Wt.bf16_rne(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(ours.view(np.uint32), ref.view(np.uint32))


def test_weight_statistics():
    w = Wt.proj_weight(Wt.DEFAULT_SEED, 2, 256, 1024).astype(np.float64)
    assert abs(w.std() * np.sqrt(1024) - 1.0) < 0.02          # U(+-sqrt(3/fan_in)) -> std 1/sqrt(fan_in)
    assert abs(w.mean()) < 3e-3
    g = Wt.norm_gain(Wt.DEFAULT_SEED, 1, 4096)
    assert g.min() >= 0.9 - 1e-2 and g.max() <= 1.1 + 1e-2
    e = Wt.embedding(Wt.DEFAULT_SEED, 64, 64)
    assert e.min() >= -1 and e.max() <= 1
    # different tensor ids / indices are decorrelated
    a = Wt.uniform01(1, 3, 10000)
    b = Wt.uniform01(1, 4, 10000)
    assert abs(np.corrcoef(a, b)[0, 1]) < 0.05


# ----------------------------------------------------------------- closed forms
def test_rmsnorm_constant_vector():
    d = 64
    g = np.linspace(0.5, 1.5, d)
    for c in (-3.0, 0.25, 7.0):
        x = np.full((1, d), c)
        got = F.rmsnorm(x, g, 1e-5)
        want = np.sign(c) * g / np.sqrt(1.0 + 1e-5 / c ** 2)
        np.testing.assert_allclose(got[0], want, rtol=1e-13)


def test_rope_invariants():
    rng = np.random.default_rng(1)
    hd = 16
    x = rng.standard_normal((5, 3, hd))
    # p = 0 -> identity
    np.testing.assert_allclose(F.rope(x, np.zeros(5, np.int64), 1e4), x, atol=0)
    # rotations preserve every (i, i+hd/2) pair norm
    pos = np.array([1, 7, 100, 1000, 3000])
    y = F.rope(x, pos, 1e4)
    h = hd // 2
    np.testing.assert_allclose(x[..., :h] ** 2 + x[..., h:] ** 2, y[..., :h] ** 2 + y[..., h:] ** 2, rtol=1e-12)
    # q(m).k(n) depends only on m - n
    q = rng.standard_normal((1, 1, hd))
    k = rng.standard_normal((1, 1, hd))
    dots = []
    for m, n in [(5, 2), (105, 102), (2003, 2000)]:
        qm = F.rope(q, np.array([m]), 1e4)
        kn = F.rope(k, np.array([n]), 1e4)
        dots.append(float((qm * kn).sum()))
    np.testing.assert_allclose(dots, dots[0], rtol=1e-9)
    # position 1, i = 0 is a rotation by exactly 1 radian (theta_0 = 1)
    e = np.zeros((1, 1, hd)); e[0, 0, 0] = 1.0
    r = F.rope(e, np.array([1]), 1e4)
    assert abs(r[0, 0, 0] - np.cos(1.0)) < 1e-15 and abs(r[0, 0, h] - np.sin(1.0)) < 1e-15


def test_attention_special_cases():
    rng = np.random.default_rng(2)
    H, Hkv, hd = 4, 2, 8
    v = rng.standard_normal((6, Hkv, hd))
    k = rng.standard_normal((6, Hkv, hd))
    # a single visible key -> output = v0 of the mapped kv head (GQA map h // (H/Hkv))
    q = rng.standard_normal((1, H, hd))
    o = F.causal_attention(q, k[:1], v[:1], np.array([0]), np.array([0]))
    for h in range(H):
        np.testing.assert_allclose(o[0, h], v[0, h // 2], rtol=1e-14)
    # q = 0 -> uniform weights -> mean of the visible values
    q0 = np.zeros((6, H, hd))
    pos = np.arange(6)
    o = F.causal_attention(q0, k, v, pos, pos)
    for t in range(6):
        for h in range(H):
            np.testing.assert_allclose(o[t, h], v[: t + 1, h // 2].mean(axis=0), rtol=1e-12)


# ------------------------------------------------------------ library routine
def _hf_model(shape: ModelShape, W: Wt.OracleWeights):
    from transformers import LlamaConfig, LlamaForCausalLM
    cfg = LlamaConfig(vocab_size=shape.vocab, hidden_size=shape.d_model,
                      intermediate_size=shape.d_ffn, num_hidden_layers=shape.n_layers,
                      num_attention_heads=shape.n_heads, num_key_value_heads=shape.n_kv_heads,
                      rms_norm_eps=shape.rms_eps, max_position_embeddings=shape.max_seq_len,
                      tie_word_embeddings=False, attention_bias=False, mlp_bias=False)
    cfg.rope_parameters = {"rope_theta": shape.rope_theta, "rope_type": "default"}
    m = LlamaForCausalLM(cfg).to(torch.float64).eval()
    sd = {"model.embed_tokens.weight": W.embed(), "model.norm.weight": W.final_norm(),
          "lm_head.weight": W.lm_head()}
    for l in range(shape.n_layers):
        w = W.layer(l)
        p = f"model.layers.{l}."
        sd.update({p + "input_layernorm.weight": w["g1"], p + "post_attention_layernorm.weight": w["g2"],
                   p + "self_attn.q_proj.weight": w["wq"], p + "self_attn.k_proj.weight": w["wk"],
                   p + "self_attn.v_proj.weight": w["wv"], p + "self_attn.o_proj.weight": w["wo"],
                   p + "mlp.gate_proj.weight": w["wg"], p + "mlp.up_proj.weight": w["wu"],
                   p + "mlp.down_proj.weight": w["wd"]})
    missing, unexpected = m.load_state_dict({k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in sd.items()},
                                            strict=False)
    assert not unexpected and all("rotary" in k for k in missing), (missing, unexpected)
    return m


@pytest.mark.parametrize("name", ["tiny", "tiny_gqa"])
def test_forward_matches_hf_llama(name):
    shape = SHAPES[name]
    W = Wt.OracleWeights(shape)
    rng = np.random.default_rng(3)
    toks = rng.integers(0, shape.vocab, size=37)
    ours = F.sequence_logits(W, toks)
    m = _hf_model(shape, W)
    with torch.no_grad():
        ref = m(torch.from_numpy(toks)[None]).logits[0].numpy()
    # HF builds cos/sin in fp32 internally -> ~1e-7 relative
    rel = F.max_abs_rel(ours, ref)
    assert rel.max() < 2e-6, rel.max()
    assert np.array_equal(F.greedy_argmax(ours), ref.argmax(-1))


def test_greedy_decode_is_prefix_consistent():
    """F5/F6: token j of a greedy decode = argmax of the causal logits of the prefix,
    so teacher forcing on the oracle's own tokens reproduces its logits."""
    shape = SHAPES["tiny_gqa"]
    W = Wt.OracleWeights(shape)
    prompt = np.random.default_rng(4).integers(0, shape.vocab, size=9)
    toks, lg = F.greedy_generate(W, prompt, 6)
    tf = F.teacher_forced_logits(W, prompt, toks)
    np.testing.assert_allclose(tf, lg, rtol=1e-12, atol=1e-12)
    assert np.array_equal(F.greedy_argmax(tf), toks)


def test_pipeline_stage_split_equals_full_forward():
    """A pipelined run must equal a single-stage run (north_star): running the
    layer partition stage by stage and handing x over equals the full forward."""
    shape = SHAPES["tiny"].with_layers(5)
    W = Wt.OracleWeights(shape)
    toks = np.random.default_rng(5).integers(0, shape.vocab, size=11)
    full = F.forward_hidden(W, toks)
    x = None
    for rng_ in F.partition_layers(shape.n_layers, 3):
        x = F.forward_hidden(W, toks, layers=rng_, x0=x) if x is not None else F.forward_hidden(W, toks, layers=rng_)
    np.testing.assert_array_equal(x, full)


# ---------------------------------------------------------------- paper numbers
def test_kv_arithmetic_paper():
    g = GOLD["kv_llama30b"]
    b = F.kv_bytes_per_token(g["n_layers"], g["d_model"], g["n_heads"], g["n_kv_heads"])
    assert b == g["bytes_per_token"]
    assert round(b / 2 ** 20, 2) == g["mb_per_token"]
    tot = g["n_requests"] * g["avg_len"] * b / 2 ** 30
    assert abs(tot - g["total_gib_approx"]) / g["total_gib_approx"] < 0.01
    g7 = GOLD["kv_llama70b_gqa"]
    assert F.kv_bytes_per_token(g7["n_layers"], g7["d_model"], g7["n_heads"], g7["n_kv_heads"]) == g7["bytes_per_token"]


def test_partition_examples():
    for L, S, want in GOLD["partition"]["cases"]:
        assert [len(r) for r in F.partition_layers(L, S)] == want
    with pytest.raises(ValueError):
        F.partition_layers(4, 5)
