// gemm_mma.cu -- C[M,N] = A[M,K] . W[N,K]^T with fused epilogues.
//
// Baseline tensor-core GEMM (mma.sync m16n8k16 bf16, fp32 accumulate,
// cp.async 3-stage pipeline, XOR-swizzled smem, ldmatrix).  It is the
// correctness reference path and the decode path for small M; the tcgen05/TMEM
// kernel (gemm_tc.cu) replaces it for large GEMMs.
//
// Fused epilogues:
//   kEpiQKV    a3: RoPE (rotate-half, pairs stored interleaved so a thread's
//              (c0,c1) column pair IS the rotation pair) + q store + paged K/V write
//   kEpiResid  a6/a9: fp32 residual += acc (each element owned by one CTA: deterministic)
//   kEpiSwiGLU a8: gate/up rows interleaved -> h = silu(g) * u
//   kEpiF32    a11: LM-head logits
// The K-reduction order of every output element is independent of its row
// position and of M, so results are batch-invariant.
#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"

namespace tdp {

namespace {
constexpr int BM = 128, BN = 128, BK = 64, STAGES = 3, NT = 256;
constexpr int TILE_BYTES = BM * BK * 2;   // 16 KB per operand per stage

TDP_DEV int swz(int r, int c) { return r * 8 + (c ^ (r & 7)); }   // 16-byte chunk index

TDP_DEV void ldmatrix_x4(uint32_t* r, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}

TDP_DEV void mma16816(float* c, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__global__ void __launch_bounds__(NT, 2)
gemm_mma_kernel(const bf16* __restrict__ A, const bf16* __restrict__ W, int M, int N, int K, EpiParams ep) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * TILE_BYTES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;          // 2 x 4 warps, warp tile 64 x 32
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
  const int KT = K / BK;

  auto load_stage = [&](int s, int kt) {
    const int k0 = kt * BK;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int id = tid + i * NT;
      const int r = id >> 3, c = id & 7;
      const int gm = m0 + r;
      const bf16* ga = A + (int64_t)(gm < M ? gm : 0) * K + k0 + c * 8;
      cp_async16(sA + s * TILE_BYTES + swz(r, c) * 16, ga, gm < M);
      const int gn = n0 + r;
      const bf16* gb = W + (int64_t)(gn < N ? gn : 0) * K + k0 + c * 8;
      cp_async16(sB + s * TILE_BYTES + swz(r, c) * 16, gb, gn < N);
    }
  };

  float acc[4][4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.f;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_async_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nk = kt + STAGES - 1;
    if (nk < KT) load_stage(nk % STAGES, nk);
    cp_async_commit();
    const uint32_t baseA = smem_u32(sA + (kt % STAGES) * TILE_BYTES);
    const uint32_t baseB = smem_u32(sB + (kt % STAGES) * TILE_BYTES);
#pragma unroll
    for (int kk = 0; kk < BK / 16; ++kk) {
      uint32_t af[4][4], bfr[2][4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int r = wm * 64 + mi * 16 + (lane & 15);
        const int c = kk * 2 + (lane >> 4);
        ldmatrix_x4(af[mi], baseA + swz(r, c) * 16);
      }
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) {
        const int r = wn * 32 + nj * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int c = kk * 2 + ((lane >> 3) & 1);
        ldmatrix_x4(bfr[nj], baseB + swz(r, c) * 16);
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) mma16816(acc[mi][ni], af[mi], &bfr[ni >> 1][(ni & 1) * 2]);
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int m = m0 + wm * 64 + mi * 16 + (lane >> 2);
      const int n = n0 + wn * 32 + ni * 8 + 2 * (lane & 3);
      epilogue_pair(ep, M, N, m, n, acc[mi][ni][0], acc[mi][ni][1]);
      epilogue_pair(ep, M, N, m + 8, n, acc[mi][ni][2], acc[mi][ni][3]);
    }
}
}  // namespace

void launch_gemm(const bf16* A, const bf16* W, int M, int N, int K, const EpiParams& ep, cudaStream_t st) {
  if (M <= 0) return;
  static bool attr = false;
  const int smem = 2 * STAGES * TILE_BYTES;
  if (!attr) {
    cudaFuncSetAttribute(gemm_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM);
  gemm_mma_kernel<<<grid, NT, smem, st>>>(A, W, M, N, K, ep);
}

}  // namespace tdp
