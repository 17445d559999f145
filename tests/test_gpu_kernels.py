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
