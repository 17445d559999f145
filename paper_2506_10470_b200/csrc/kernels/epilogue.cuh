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

// Swap-AB tcgen05 epilogue for one 32-token chunk: this lane owns output
// feature f and holds its accumulators for tokens t0 .. t0+31 in r[].  Per-token
// metadata (position, KV slot) is loaded once per chunk by lane j for token
// t0+j and broadcast with shuffles; all other loads of a chunk are issued
// before any store, so the chunk costs one memory latency instead of 32.
// Every lane executes the shuffles (no divergence around them).
TDP_DEV void epilogue_chunk(const EpiParams& ep, int T, int Nf, int f, int t0, const uint32_t* r) {
  const int lane = threadIdx.x & 31;
  const bool even = (lane & 1) == 0;
  const bool fok = f < Nf;
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  switch (ep.mode) {
    case kEpiF32: {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (t0 + j < T && fok) ep.out_f32[(int64_t)(t0 + j) * ep.ldo + f] = v[j];
      break;
    }
    case kEpiResid: {
      float xo[32];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        xo[j] = (t0 + j < T && fok) ? ep.out_f32[(int64_t)(t0 + j) * ep.ldo + f] : 0.f;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (t0 + j < T && fok) ep.out_f32[(int64_t)(t0 + j) * ep.ldo + f] = xo[j] + v[j];
      break;
    }
    case kEpiSwiGLU: {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float u = __shfl_xor_sync(0xffffffffu, v[j], 1);
        if (even && t0 + j < T && fok) ep.out_bf16[(int64_t)(t0 + j) * (Nf >> 1) + (f >> 1)] = __float2bfloat16_rn(silu(v[j]) * u);
      }
      break;
    }
    case kEpiBF16: {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (t0 + j < T && fok) ep.out_bf16[(int64_t)(t0 + j) * ep.ldo + f] = __float2bfloat16_rn(v[j]);
      break;
    }
    case kEpiQKV: {
      const int hd = ep.hd, half = hd >> 1;
      const int qcols = ep.H * hd, kcols = ep.Hkv * hd;
      const int tl = t0 + lane;
      const int my_pos = tl < T ? ep.pos[tl] : 0;
      const int my_slot = tl < T ? ep.slot[tl] : 0;
      const bool rot = f < qcols + kcols;
      const int i = (f % hd) >> 1;
      float2 cs[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int pj = __shfl_sync(0xffffffffu, my_pos, j);
        cs[j] = (rot && fok && t0 + j < T) ? *reinterpret_cast<const float2*>(ep.rope_cs + ((int64_t)pj * half + i) * 2)
                                           : make_float2(1.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float pv = __shfl_xor_sync(0xffffffffu, v[j], 1);
        const int sj = __shfl_sync(0xffffffffu, my_slot, j);
        const int t = t0 + j;
        if (t >= T || !fok) continue;
        // rotate-half pair (x_e, x_o) = (lane even, lane odd)
        const float out = !rot ? v[j] : (even ? v[j] * cs[j].x - pv * cs[j].y : v[j] * cs[j].x + pv * cs[j].y);
        const bf16 ob = __float2bfloat16_rn(out);
        if (f < qcols) {
          ep.out_bf16[(int64_t)t * qcols + f] = ob;
        } else if (f < qcols + kcols) {
          const int kn = f - qcols;
          ep.kcache[((((int64_t)(sj >> 4) * 2 + 0) * ep.Hkv + kn / hd) * kBlock + (sj & 15)) * hd + kn % hd] = ob;
        } else {
          const int vn = f - qcols - kcols;
          ep.kcache[((((int64_t)(sj >> 4) * 2 + 1) * ep.Hkv + vn / hd) * kBlock + (sj & 15)) * hd + vn % hd] = ob;
        }
      }
      break;
    }
  }
}

// Token-major tcgen05 epilogue (prefill GEMM): this thread owns token t and
// holds features f0 .. f0+31 in v[] (consecutive TMEM columns), so RoPE pairs
// (2i, 2i+1) and gate/up pairs are adjacent registers and every global access
// is a 16-byte vector.  pos / slot are this token's position and KV slot.
TDP_DEV void store_bf16x16(bf16* dst, const float* v) {
  uint4 a, b;
  a.x = pack_bf16x2(v[0], v[1]);
  a.y = pack_bf16x2(v[2], v[3]);
  a.z = pack_bf16x2(v[4], v[5]);
  a.w = pack_bf16x2(v[6], v[7]);
  b.x = pack_bf16x2(v[8], v[9]);
  b.y = pack_bf16x2(v[10], v[11]);
  b.z = pack_bf16x2(v[12], v[13]);
  b.w = pack_bf16x2(v[14], v[15]);
  reinterpret_cast<uint4*>(dst)[0] = a;
  reinterpret_cast<uint4*>(dst)[1] = b;
}

TDP_DEV void epilogue_row(const EpiParams& ep, int Nf, int t, int f0, float* v, int pos, int slot) {
  const bool full = f0 + 32 <= Nf;
  switch (ep.mode) {
    case kEpiF32: {
      float* o = ep.out_f32 + (int64_t)t * ep.ldo + f0;
      if (full) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      } else {
        for (int j = 0; j < 32; ++j)
          if (f0 + j < Nf) o[j] = v[j];
      }
      break;
    }
    case kEpiResid: {
      float* o = ep.out_f32 + (int64_t)t * ep.ldo + f0;
      if (full) {
        float4 x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = reinterpret_cast<const float4*>(o)[j];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          reinterpret_cast<float4*>(o)[j] =
              make_float4(x[j].x + v[4 * j], x[j].y + v[4 * j + 1], x[j].z + v[4 * j + 2], x[j].w + v[4 * j + 3]);
      } else {
        for (int j = 0; j < 32; ++j)
          if (f0 + j < Nf) o[j] += v[j];
      }
      break;
    }
    case kEpiSwiGLU: {
      float h[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) h[j] = silu(v[2 * j]) * v[2 * j + 1];
      bf16* o = ep.out_bf16 + (int64_t)t * (Nf >> 1) + (f0 >> 1);
      if (full) {
        store_bf16x16(o, h);
      } else {
        for (int j = 0; j < 16; ++j)
          if (f0 + 2 * j < Nf) o[j] = __float2bfloat16_rn(h[j]);
      }
      break;
    }
    case kEpiBF16: {
      bf16* o = ep.out_bf16 + (int64_t)t * ep.ldo + f0;
      if (full) {
        store_bf16x16(o, v);
        store_bf16x16(o + 16, v + 16);
      } else {
        for (int j = 0; j < 32; ++j)
          if (f0 + j < Nf) o[j] = __float2bfloat16_rn(v[j]);
      }
      break;
    }
    case kEpiQKV: {
      const int hd = ep.hd, half = hd >> 1;
      const int qcols = ep.H * hd, kcols = ep.Hkv * hd;
#pragma unroll
      for (int g = 0; g < 2; ++g) {           // 16-feature groups (a group never spans two heads)
        const int f = f0 + 16 * g;
        if (f >= Nf) break;
        float* w = v + 16 * g;
        if (f < qcols + kcols) {              // rotate-half pairs (2i, 2i+1) at absolute position pos
          const int i0 = (f % hd) >> 1;
          const float4* cs = reinterpret_cast<const float4*>(ep.rope_cs + ((int64_t)pos * half + i0) * 2);
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            const float4 c2 = cs[p];          // (cos, sin) of pairs 2p and 2p+1
            const float e0 = w[4 * p], o0 = w[4 * p + 1], e1 = w[4 * p + 2], o1 = w[4 * p + 3];
            w[4 * p] = e0 * c2.x - o0 * c2.y;
            w[4 * p + 1] = o0 * c2.x + e0 * c2.y;
            w[4 * p + 2] = e1 * c2.z - o1 * c2.w;
            w[4 * p + 3] = o1 * c2.z + e1 * c2.w;
          }
        }
        bf16* dst;
        if (f < qcols) {
          dst = ep.out_bf16 + (int64_t)t * qcols + f;
        } else {
          const bool isk = f < qcols + kcols;
          const int kn = f - (isk ? qcols : qcols + kcols);
          dst = ep.kcache + ((((int64_t)(slot >> 4) * 2 + (isk ? 0 : 1)) * ep.Hkv + kn / hd) * kBlock + (slot & 15)) * hd +
                kn % hd;
        }
        store_bf16x16(dst, w);
      }
      break;
    }
  }
}

}  // namespace tdp
