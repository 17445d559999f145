"""Kernel-level GPU checks: the tcgen05/TMA GEMM and the mma.sync baseline vs
an fp64 product of the same bf16 operands (plain definition of a matmul)."""
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
@pytest.mark.parametrize("impl,splits", [(0, 1), (0, 3), (2, 1), (2, 2), (1, 1)])
def test_gemm_vs_fp64(T, N, K, impl, splits):
    rng = np.random.default_rng(T * 7 + N + K)
    Ab, Af = _bf16(rng, (T, K))
    Wb, Wf = _bf16(rng, (N, K), 1.0 / np.sqrt(K))
    out = td_test_gemm(Ab, Wb, impl=impl, splits=splits)
    ref = Af @ Wf.T
    err = np.abs(out - ref).max() / max(np.abs(ref).max(), 1e-6)
    assert err < 2e-5, err     # fp32 accumulation of exact bf16 products


@pytest.mark.parametrize("T,N,K", [(1, 128, 64), (7, 192, 128), (8, 256, 128), (32, 256, 256), (33, 384, 512),
                                   (64, 4096, 4096), (100, 128, 1024), (128, 512, 4096), (5, 12288, 4096),
                                   (16, 4096, 11008), (3, 22016, 4096), (128, 1536, 512)])
def test_gemm_stream_k_vs_fp64(T, N, K):
    """Stream-K decode GEMM (impl 3): ranges cut tiles into 1..many
    contributors (U < 148 gives one k-block per CTA); partial sums are combined
    by the last arriving contributor, in contributor order -- so whichever CTA
    arrives last, the result is bitwise the same (checked over repeated calls)."""
    rng = np.random.default_rng(T * 11 + N + K)
    Ab, Af = _bf16(rng, (T, K))
    Wb, Wf = _bf16(rng, (N, K), 1.0 / np.sqrt(K))
    ref = Af @ Wf.T
    out = td_test_gemm(Ab, Wb, impl=3)
    err = np.abs(out - ref).max() / max(np.abs(ref).max(), 1e-6)
    assert err < 2e-5, err
    for _ in range(3):
        assert np.array_equal(td_test_gemm(Ab, Wb, impl=3), out)
