"""Pins of oracle/cached.py (the F6 KV-cached form) against the cache-less
definition oracle/forward.py: equal logits at every position (fp64, up to
rounding order), equal greedy tokens, and batching several requests' decode
rows changes nothing (rows never mix across requests)."""
import numpy as np
import pytest

from oracle import cached as Cc
from oracle import forward as F
from oracle.weights import OracleWeights
from workload import SHAPES


@pytest.mark.parametrize("name", ["tiny", "tiny_gqa"])
def test_cached_prefill_and_decode_equal_definition(name):
    W = OracleWeights(SHAPES[name])
    rng = np.random.default_rng(3)
    seq = rng.integers(0, 256, size=30)
    ref = F.sequence_logits(W, seq)                      # [30, V], cache-less
    c = Cc.Cache(W.shape.n_layers)
    got = [Cc.forward_rows(W, [c], [seq[:20]], last_only=False)]
    for t in seq[20:]:
        got.append(Cc.forward_rows(W, [c], [[t]]))
    got = np.concatenate(got)
    assert got.shape == ref.shape
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12 * np.abs(ref).max())


def test_batched_rows_equal_one_request_at_a_time():
    W = OracleWeights(SHAPES["tiny_gqa"])
    rng = np.random.default_rng(4)
    prompts = [rng.integers(0, 256, size=L) for L in (5, 17, 1)]
    solo, batch = [], [Cc.Cache(2) for _ in prompts]
    for p in prompts:
        c = Cc.Cache(2)
        Cc.forward_rows(W, [c], [p])
        solo.append((c, Cc.forward_rows(W, [c], [[7]])[0]))
    Cc.forward_rows(W, batch, prompts)
    lg = Cc.forward_rows(W, batch, [[7]] * 3)
    for i in range(3):
        np.testing.assert_allclose(lg[i], solo[i][1], rtol=0, atol=1e-12)
        assert batch[i].T == len(prompts[i]) + 1


def test_greedy_generate_cached_equals_definition():
    W = OracleWeights(SHAPES["tiny"])
    p = np.random.default_rng(5).integers(0, 256, size=9)
    t1, l1 = F.greedy_generate(W, p, 12)
    t2, l2 = Cc.greedy_generate_cached(W, p, 12)
    assert np.array_equal(t1, t2)
    np.testing.assert_allclose(l2, l1, rtol=0, atol=1e-12 * np.abs(l1).max())


def test_fp32_mode_within_fp32_rounding():
    W = OracleWeights(SHAPES["tiny"])
    seq = np.random.default_rng(6).integers(0, 256, size=24)
    ref = F.sequence_logits(W, seq)[-1]
    c = Cc.Cache(2)
    got = Cc.forward_rows(W, [c], [seq], dtype=np.float32)[0]
    assert got.dtype == np.float32
    assert F.max_abs_rel(got, ref).max() < 1e-5
