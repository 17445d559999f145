// epilogue.cuh -- fused GEMM epilogues shared by the mma.sync and tcgen05 GEMMs
// and the split-K reduction.  (m, n) = (token row, output feature); n is even
// and (v0, v1) are the values of features n and n+1:
//   kEpiQKV    RoPE on the interleaved (i, i+hd/2) pair + q store / paged K,V write
//   kEpiResid  fp32 residual += (deterministic: one owner per element)
//   kEpiSwiGLU gate/up interleaved rows: h[m][n/2] = silu(g) * u
//   kEpiF32 / kEpiBF16 plain stores
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace tdp {

TDP_DEV float silu(float g) { return g / (1.0f + __expf(-g)); }

TDP_DEV void epilogue_pair(const EpiParams& ep, int M, int N, int m, int n, float v0, float v1) {
  if (m >= M || n >= N) return;
  switch (ep.mode) {
    case kEpiF32: {
      *reinterpret_cast<float2*>(ep.out_f32 + (int64_t)m * ep.ldo + n) = make_float2(v0, v1);
      break;
    }
    case kEpiResid: {
      float2* p = reinterpret_cast<float2*>(ep.out_f32 + (int64_t)m * ep.ldo + n);
      float2 x = *p;
      x.x += v0;
      x.y += v1;
      *p = x;
      break;
    }
    case kEpiSwiGLU: {
      ep.out_bf16[(int64_t)m * (N >> 1) + (n >> 1)] = __float2bfloat16_rn(silu(v0) * v1);
      break;
    }
    case kEpiBF16: {
      *reinterpret_cast<uint32_t*>(ep.out_bf16 + (int64_t)m * ep.ldo + n) = pack_bf16x2(v0, v1);
      break;
    }
    case kEpiQKV: {
      const int hd = ep.hd;
      const int qcols = ep.H * hd, kcols = ep.Hkv * hd;
      if (n < qcols + kcols) {
        const int i = (n % hd) >> 1;
        const float2 cs = *reinterpret_cast<const float2*>(ep.rope_cs + ((int64_t)ep.pos[m] * (hd >> 1) + i) * 2);
        const float r0 = v0 * cs.x - v1 * cs.y;
        const float r1 = v1 * cs.x + v0 * cs.y;
        if (n < qcols) {
          *reinterpret_cast<uint32_t*>(ep.out_bf16 + (int64_t)m * qcols + n) = pack_bf16x2(r0, r1);
        } else {
          const int kn = n - qcols, kh = kn / hd, j = kn % hd;
          const int s = ep.slot[m];
          const int64_t off = ((((int64_t)(s >> 4) * 2 + 0) * ep.Hkv + kh) * kBlock + (s & 15)) * hd + j;
          *reinterpret_cast<uint32_t*>(ep.kcache + off) = pack_bf16x2(r0, r1);
        }
      } else {
        const int vn = n - qcols - kcols, vh = vn / hd, j = vn % hd;
        const int s = ep.slot[m];
        const int64_t off = ((((int64_t)(s >> 4) * 2 + 1) * ep.Hkv + vh) * kBlock + (s & 15)) * hd + j;
        *reinterpret_cast<uint32_t*>(ep.kcache + off) = pack_bf16x2(v0, v1);
      }
      break;
    }
  }
}

}  // namespace tdp
