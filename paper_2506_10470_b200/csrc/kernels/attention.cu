// attention.cu -- paged decode attention (split-KV) and varlen causal prefill
// attention over the paged KV cache.
//
// KV pool layout per layer: [block][K|V][Hkv][16 tokens][hd] bf16, so one
// (block, kv-head) K or V page is 16*hd*2 contiguous bytes (4 KB at hd=128).
// q/k rotate-half pairs are stored interleaved ((i, i+hd/2) -> (2i, 2i+1));
// dot products are invariant under that common permutation, v/o are logical.
//
// Decode: HBM-streaming, one CTA per (split, kv-head, sequence); a kv page is
// read once for all G = H/Hkv query heads (GQA).  LPT = hd/8 lanes cooperate
// on one token (16-byte loads), U tokens in flight per thread-group, online
// softmax in fp32 (exp2 with log2e-prescaled scores), warp-shuffle merges.
// Splits are fixed 512-token chunks of each sequence's own context, merged in
// split order -> results do not depend on batch composition.
#include <float.h>
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace tdp {

constexpr int kSplit = 512;
constexpr float kLog2e = 1.4426950408889634f;

struct SoftmaxState {
  float m, l;
};

template <int HD, int G>
__global__ void __launch_bounds__(128)
decode_attn_kernel(DecodeAttnParams p) {
  constexpr int LPT = HD / 8;          // lanes per token
  constexpr int TPW = 32 / LPT;        // tokens per warp per step
  constexpr int NW = 4;
  constexpr int U = 4;                 // tokens in flight per thread group
  const int seq = blockIdx.z, kh = blockIdx.y, split = blockIdx.x;
  const int ctx = p.ctx[seq];
  const int n_splits = (ctx + kSplit - 1) / kSplit;
  if (split >= n_splits) return;
  const int t_begin = split * kSplit;
  const int t_end = min(ctx, t_begin + kSplit);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tg = lane / LPT, sub = lane % LPT;
  const int H = p.H;
  const float scale = rsqrtf((float)HD) * kLog2e;

  float q[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const uint4 u = *reinterpret_cast<const uint4*>(p.q + ((int64_t)seq * H + kh * G + g) * HD + sub * 8);
    bf16x8_to_f32(u, q[g]);
#pragma unroll
    for (int i = 0; i < 8; ++i) q[g][i] *= scale;
  }
  float m[G], l[G], acc[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[g][i] = 0.f;
  }
  const int32_t* bt = p.bt + (int64_t)seq * p.maxblk;
  const int64_t head_stride = (int64_t)kBlock * HD;           // one (blk, kv, head) page
  for (int base = t_begin; base < t_end; base += NW * TPW * U) {
    uint4 kr[U], vr[U];
    bool valid[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = base + (u * NW + warp) * TPW + tg;
      valid[u] = t < t_end;
      const int tt = valid[u] ? t : t_begin;
      const int blk = bt[tt >> 4];
      const int64_t kbase = (((int64_t)blk * 2) * p.Hkv + kh) * head_stride + (tt & 15) * HD + sub * 8;
      kr[u] = ld_nc_v4(p.kv + kbase);
      vr[u] = ld_nc_v4(p.kv + kbase + (int64_t)p.Hkv * head_stride);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float kf[8], vf[8];
      bf16x8_to_f32(kr[u], kf);
      bf16x8_to_f32(vr[u], vf);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) s = fmaf(q[g][i], kf[i], s);
#pragma unroll
        for (int o = LPT / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (valid[u]) {
          const float mn = fmaxf(m[g], s);
          const float corr = exp2f(m[g] - mn);
          const float pr = exp2f(s - mn);
          l[g] = l[g] * corr + pr;
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[g][i] = fmaf(pr, vf[i], acc[g][i] * corr);
          m[g] = mn;
        }
      }
    }
  }
  // merge thread groups within the warp (lanes with equal `sub`)
#pragma unroll
  for (int o = LPT; o < 32; o <<= 1) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m[g], o);
      const float l2 = __shfl_xor_sync(0xffffffffu, l[g], o);
      const float mn = fmaxf(m[g], m2);
      const float c1 = mn == -INFINITY ? 0.f : exp2f(m[g] - mn);
      const float c2 = mn == -INFINITY ? 0.f : exp2f(m2 - mn);
      l[g] = l[g] * c1 + l2 * c2;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float a2 = __shfl_xor_sync(0xffffffffu, acc[g][i], o);
        acc[g][i] = acc[g][i] * c1 + a2 * c2;
      }
      m[g] = mn;
    }
  }
  __shared__ float sm[NW][G][2];
  __shared__ float sacc[NW][G][HD];
  if (tg == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (sub == 0) { sm[warp][g][0] = m[g]; sm[warp][g][1] = l[g]; }
#pragma unroll
      for (int i = 0; i < 8; ++i) sacc[warp][g][sub * 8 + i] = acc[g][i];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < G * HD; e += blockDim.x) {
    const int g = e / HD, dim = e % HD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; ++w) M = fmaxf(M, sm[w][g][0]);
    float L = 0.f, A = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const float c = M == -INFINITY ? 0.f : exp2f(sm[w][g][0] - M);
      L += sm[w][g][1] * c;
      A += sacc[w][g][dim] * c;
    }
    const int h = kh * G + g;
    if (n_splits == 1) {
      p.o[((int64_t)seq * H + h) * HD + dim] = __float2bfloat16_rn(A / L);
    } else {
      float* part = p.part + (((int64_t)seq * H + h) * p.max_splits + split) * (HD + 2);
      part[2 + dim] = A;
      if (dim == 0) { part[0] = M; part[1] = L; }
    }
  }
}

__global__ void decode_combine_kernel(DecodeAttnParams p, int hd) {
  const int seq = blockIdx.y, h = blockIdx.x;
  const int ctx = p.ctx[seq];
  const int n_splits = (ctx + kSplit - 1) / kSplit;
  if (n_splits <= 1) return;
  const float* part = p.part + ((int64_t)seq * p.H + h) * p.max_splits * (hd + 2);
  float M = -INFINITY;
  for (int s = 0; s < n_splits; ++s) M = fmaxf(M, part[s * (hd + 2)]);
  for (int dim = threadIdx.x; dim < hd; dim += blockDim.x) {
    float L = 0.f, A = 0.f;
    for (int s = 0; s < n_splits; ++s) {
      const float* ps = part + s * (hd + 2);
      const float c = exp2f(ps[0] - M);
      L += ps[1] * c;
      A += ps[2 + dim] * c;
    }
    p.o[((int64_t)seq * p.H + h) * hd + dim] = __float2bfloat16_rn(A / L);
  }
}

template <int HD>
static void launch_decode_hd(const DecodeAttnParams& p, cudaStream_t st) {
  const int G = p.H / p.Hkv;
  dim3 grid(p.max_splits, p.Hkv, p.n);
  switch (G) {
    case 1: decode_attn_kernel<HD, 1><<<grid, 128, 0, st>>>(p); break;
    case 2: decode_attn_kernel<HD, 2><<<grid, 128, 0, st>>>(p); break;
    case 4: decode_attn_kernel<HD, 4><<<grid, 128, 0, st>>>(p); break;
    case 8: decode_attn_kernel<HD, 8><<<grid, 128, 0, st>>>(p); break;
    default: return;
  }
  if (p.max_splits > 1) decode_combine_kernel<<<dim3(p.H, p.n), 128, 0, st>>>(p, HD);
}

void launch_decode_attn(const DecodeAttnParams& p, cudaStream_t st) {
  if (p.n <= 0) return;
  switch (p.hd) {
    case 16: launch_decode_hd<16>(p, st); break;
    case 32: launch_decode_hd<32>(p, st); break;
    case 64: launch_decode_hd<64>(p, st); break;
    case 128: launch_decode_hd<128>(p, st); break;
  }
}

// ------------------------------------------------------------------ prefill
// One warp per (query token, head): lane-per-key scores over 32-key chunks,
// online softmax, lane-owned output dims.  Keys = positions 0..pos of the
// token's own sequence, read from the paged cache (written by the QKV epilogue
// of this micro-batch).
template <int HD>
__global__ void __launch_bounds__(128) prefill_attn_kernel(PrefillAttnParams p) {
  constexpr int DPL = HD >= 32 ? HD / 32 : 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x;
  const int h = blockIdx.y * 4 + warp;
  if (h >= p.H) return;
  const int G = p.H / p.Hkv;
  const int kh = h / G;
  const int seq = p.tok_seq[t];
  const int pos = p.tok_pos[t];
  const int32_t* bt = p.bt + (int64_t)seq * p.maxblk;
  __shared__ float qs[4][HD];
  const float scale = rsqrtf((float)HD) * kLog2e;
  for (int d = lane; d < HD; d += 32)
    qs[warp][d] = __bfloat162float(p.q[((int64_t)t * p.H + h) * HD + d]) * scale;
  __syncwarp();
  const int64_t head_stride = (int64_t)kBlock * HD;
  float m = -INFINITY, l = 0.f, acc[DPL];
#pragma unroll
  for (int i = 0; i < DPL; ++i) acc[i] = 0.f;
  for (int base = 0; base <= pos; base += 32) {
    const int j = base + lane;
    float s = -INFINITY;
    if (j <= pos) {
      const int blk = bt[j >> 4];
      const bf16* kp = p.kv + (((int64_t)blk * 2) * p.Hkv + kh) * head_stride + (j & 15) * HD;
      float dot = 0.f;
#pragma unroll
      for (int c = 0; c < HD / 8; ++c) {
        float kf[8];
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(kp + c * 8), kf);
#pragma unroll
        for (int i = 0; i < 8; ++i) dot = fmaf(qs[warp][c * 8 + i], kf[i], dot);
      }
      s = dot;
    }
    const float cmax = warp_max(s);
    const float mn = fmaxf(m, cmax);
    const float corr = exp2f(m - mn);     // m = -inf on the first chunk -> 0
    const float pr = (j <= pos) ? exp2f(s - mn) : 0.f;
    l = l * corr + warp_sum(pr);
#pragma unroll
    for (int i = 0; i < DPL; ++i) acc[i] *= corr;
    const int nk = min(32, pos - base + 1);
    for (int k = 0; k < nk; ++k) {
      const float pk = __shfl_sync(0xffffffffu, pr, k);
      const int jj = base + k;
      const int blk = bt[jj >> 4];
      const bf16* vp = p.kv + (((int64_t)blk * 2 + 1) * p.Hkv + kh) * head_stride + (jj & 15) * HD;
#pragma unroll
      for (int i = 0; i < DPL; ++i) {
        const int d = lane + 32 * i;
        if (d < HD) acc[i] = fmaf(pk, __bfloat162float(vp[d]), acc[i]);
      }
    }
    m = mn;
  }
#pragma unroll
  for (int i = 0; i < DPL; ++i) {
    const int d = lane + 32 * i;
    if (d < HD) p.o[((int64_t)t * p.H + h) * HD + d] = __float2bfloat16_rn(acc[i] / l);
  }
}

void launch_prefill_attn(const PrefillAttnParams& p, cudaStream_t st) {
  if (p.T <= 0) return;
  dim3 grid(p.T, (p.H + 3) / 4);
  switch (p.hd) {
    case 16: prefill_attn_kernel<16><<<grid, 128, 0, st>>>(p); break;
    case 32: prefill_attn_kernel<32><<<grid, 128, 0, st>>>(p); break;
    case 64: prefill_attn_kernel<64><<<grid, 128, 0, st>>>(p); break;
    case 128: prefill_attn_kernel<128><<<grid, 128, 0, st>>>(p); break;
  }
}

}  // namespace tdp
