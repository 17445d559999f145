"""Kernel-level GPU checks: the tcgen05/TMA GEMMs (decode swap-AB with split-K,
persistent token-major prefill) vs an fp64 product of the same bf16 operands
(the plain definition of a matmul)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2506_10470_b200.tdpipe import td_test_gemm  # noqa: E402


def _bf16(rng, shape, scale=1.0):
    x = (rng.standard_normal(shape) * scale).astype(np.float32)
    b = torch.from_numpy(x).to(torch.bfloat16)
    return b.view(torch.int16).numpy().view(np.uint16), b.to(torch.float64).numpy()


@pytest.mark.parametrize("T,N,K", [(1, 128, 64), (7, 192, 128), (32, 256, 256), (64, 384, 512), (100, 128, 1024),
                                   (128, 512, 4096), (200, 640, 320), (256, 1024, 4096), (300, 256, 576),
                                   (2048, 1024, 1024), (513, 4096, 128)])
@pytest.mark.parametrize("impl,splits", [(0, 1), (0, 3), (2, 1), (2, 2)])
def test_gemm_vs_fp64(T, N, K, impl, splits):
    rng = np.random.default_rng(T * 7 + N + K)
    Ab, Af = _bf16(rng, (T, K))
    Wb, Wf = _bf16(rng, (N, K), 1.0 / np.sqrt(K))
    out = td_test_gemm(Ab, Wb, impl=impl, splits=splits)
    ref = Af @ Wf.T
    err = np.abs(out - ref).max() / max(np.abs(ref).max(), 1e-6)
    assert err < 2e-5, err     # fp32 accumulation of exact bf16 products


@pytest.mark.parametrize("T,N,K,splits", [(129, 256, 1024, 2), (256, 1024, 4096, 3), (300, 640, 576, 2),
                                          (512, 4096, 2048, 4), (200, 384, 512, 8), (256, 8192, 1024, 1),
                                          (2048, 4096, 512, 1), (1900, 3200, 256, 2), (640, 12288, 192, 3)])
def test_gemm_token_major_split_k_vs_fp64(T, N, K, splits):
    """The persistent token-major tcgen05 kernel with split-K (impl 4): every
    split writes an fp32 partial tile, reduced in split order -- the engine's
    path for 129..512-token decode micro-batches; 128-feature tiles when the
    256-feature tiles fill < 96 SMs, 256 otherwise (the last three cases);
    bitwise repeatable."""
    rng = np.random.default_rng(T * 13 + N + K + splits)
    Ab, Af = _bf16(rng, (T, K))
    Wb, Wf = _bf16(rng, (N, K), 1.0 / np.sqrt(K))
    ref = Af @ Wf.T
    out = td_test_gemm(Ab, Wb, impl=4, splits=splits)
    err = np.abs(out - ref).max() / max(np.abs(ref).max(), 1e-6)
    assert err < 2e-5, err
    assert np.array_equal(td_test_gemm(Ab, Wb, impl=4, splits=splits), out)


@pytest.mark.parametrize("T,N,K", [(1, 128, 64), (4, 256, 64), (7, 256, 256), (32, 4096, 4096), (8, 4096, 11008),
                                   (33, 1024, 1024), (64, 8192, 1024), (100, 512, 4096), (128, 22016, 4096)])
def test_chain_gemm_vs_fp64(T, N, K):
    """The persistent decode chain (impl 5): a GEMM op split stream-K style into
    (CTA, weight tile) segments, each tile reduced in CTA order by the CTA that
    completes it (ticket) into a zeroed residual --
    the engine's path for decode micro-batches of <= 128 tokens; bitwise
    repeatable."""
    rng = np.random.default_rng(T * 11 + N + K)
    Ab, Af = _bf16(rng, (T, K))
    Wb, Wf = _bf16(rng, (N, K), 1.0 / np.sqrt(K))
    out = td_test_gemm(Ab, Wb, impl=5)
    ref = Af @ Wf.T
    err = np.abs(out - ref).max() / max(np.abs(ref).max(), 1e-6)
    assert err < 2e-5, err
    assert np.array_equal(td_test_gemm(Ab, Wb, impl=5), out)


def _bits_to_f64(b):
    return torch.from_numpy(b.view(np.int16)).view(torch.bfloat16).to(torch.float64).numpy()


@pytest.mark.parametrize("T,d,F", [(1, 128, 256), (4, 256, 512), (9, 1024, 2816), (40, 512, 1536), (128, 1024, 1024)])
def test_chain_mlp_vs_fp64(T, d, F):
    """Decode chain on one MLP block with its split RMSNorm (prep: a = bf16(x0*g)
    and sums of squares | gate/up GEMM, tile reductions scale by 1/rms and apply
    SwiGLU | down GEMM, tile reductions add into the residual; grid barriers
    between) vs the plain definition in fp64.  a and h are checked to 1 bf16
    ulp; the residual is recomputed from the kernel's own h, so its fp32
    tolerance is tight."""
    from paper_2506_10470_b200.tdpipe import td_test_chain_mlp
    rng = np.random.default_rng(T + d + F)
    x0 = rng.standard_normal((T, d)).astype(np.float32)
    gb, gf = _bf16(rng, (d,), 0.5)
    gb = gb.copy()
    Wgub, Wguf = _bf16(rng, (2 * F, d), 1.0 / np.sqrt(d))
    Wdb, Wdf = _bf16(rng, (d, F), 1.0 / np.sqrt(F))
    a, h, x = td_test_chain_mlp(x0, gb, Wgub, Wdb)
    xr = x0.astype(np.float64)
    a_k = _bits_to_f64(a)
    a_ref = xr * gf
    assert np.abs(a_k - a_ref).max() <= 2 ** -8 * np.abs(a_ref).max()
    inv = 1.0 / np.sqrt((xr * xr).mean(axis=1, keepdims=True) + 1e-5)
    gu = (a_k @ Wguf.T) * inv
    g_, u_ = gu[:, 0::2], gu[:, 1::2]
    h_ref = g_ / (1 + np.exp(-g_)) * u_
    h_k = _bits_to_f64(h)
    assert np.abs(h_k - h_ref).max() <= 2 ** -7 * np.abs(h_ref).max() + 1e-6
    x_ref = xr + h_k @ Wdf.T
    assert np.abs(x - x_ref).max() <= 2e-5 * np.abs(x_ref).max()
    a2, h2, x2 = td_test_chain_mlp(x0, gb, Wgub, Wdb)
    assert np.array_equal(x2, x) and np.array_equal(a2, a) and np.array_equal(h2, h)

