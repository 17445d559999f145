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
// Splits are fixed-size chunks of each sequence's own context (128..512
// tokens, chosen per micro-batch so that the grid fills the GPU), merged in
// split order.
#include <float.h>
#include <math.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace tdp {

constexpr float kLog2e = 1.4426950408889634f;

struct SoftmaxState {
  float m, l;
};

// Combine the per-thread online-softmax states of one CTA (lanes, then warps)
// and write the result: o directly for a single segment, else the segment's
// partial (m, l, acc) -- the last segment of (seq, kh) to arrive merges all
// partials in segment order (deterministic; no separate combine launch).
template <int HD, int G>
__device__ __forceinline__ void attn_finish(const DecodeAttnParams& p, int seq, int kh, int split, int n_splits,
                                            float (&m)[G], float (&l)[G], float (&acc)[G][8]) {
  constexpr int LPT = HD / 8;
  constexpr int NW = 4;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tg = lane / LPT, sub = lane % LPT;
  const int H = p.H;
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
  __syncthreads();   // the previous segment of this CTA is done with sm / sacc
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
      __stcg(part + 2 + dim, A);
      if (dim == 0) {
        __stcg(part, M);
        __stcg(part + 1, L);
      }
    }
  }
  if (n_splits == 1) return;
  // the last split CTA of this (sequence, kv head) merges all splits in split
  // order (deterministic) -- no separate combine launch
  __shared__ int s_last;
  // barrier, then one cumulative fence + ticket by thread 0 (the grid-sync
  // pattern): the CTA's partial stores are ordered before the ticket
  // (measured 0.5 % faster than a fence in every thread)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&p.counters[seq * p.Hkv + kh], 1) == n_splits - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int e = threadIdx.x; e < G * HD; e += blockDim.x) {
    const int g = e / HD, dim = e % HD;
    const int h = kh * G + g;
    const float* part = p.part + ((int64_t)seq * H + h) * p.max_splits * (HD + 2);
    // up to 8 splits' partials are loaded at once (one L2 round trip per 8
    // splits instead of two dependent loads per split), then combined in
    // split order; with <= 8 splits the arithmetic is the two-pass
    // global-max form exactly
    float M = -INFINITY, L = 0.f, A = 0.f;
    for (int s0 = 0; s0 < n_splits; s0 += 8) {
      float mv[8], lv[8], av[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const bool ok = s0 + j < n_splits;
        const float* ps = part + (s0 + j) * (HD + 2);
        mv[j] = ok ? __ldcg(ps) : -INFINITY;
        lv[j] = ok ? __ldcg(ps + 1) : 0.f;
        av[j] = ok ? __ldcg(ps + 2 + dim) : 0.f;
      }
      float mn = M;
#pragma unroll
      for (int j = 0; j < 8; ++j) mn = fmaxf(mn, mv[j]);
      if (M != -INFINITY) {
        const float c0 = exp2f(M - mn);
        L *= c0;
        A *= c0;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float c = mv[j] == -INFINITY ? 0.f : exp2f(mv[j] - mn);
        L += lv[j] * c;
        A += av[j] * c;
      }
      M = mn;
    }
    p.o[((int64_t)seq * H + h) * HD + dim] = __float2bfloat16_rn(A / L);
  }
  if (threadIdx.x == 0) p.counters[seq * p.Hkv + kh] = 0;
}


// One CTA attends (sequence seq, kv head kh) over context tokens
// [t_begin, t_end): segment `split` of `n_splits`.  With n_splits == 1 it writes
// o; otherwise it writes the segment's partial (m, l, acc) and the last
// segment to finish merges all of them in segment order.
template <int HD, int G>
__device__ __forceinline__ void attend_range(const DecodeAttnParams& p, int seq, int kh, int t_begin, int t_end,
                                             int split, int n_splits, int newest) {
  constexpr int LPT = HD / 8;          // lanes per token
  constexpr int TPW = 32 / LPT;        // tokens per warp per step
  constexpr int NW = 4;
  constexpr int U = 4;                 // tokens in flight per thread group
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tg = lane / LPT, sub = lane % LPT;
  const int H = p.H;
  const float scale = rsqrtf((float)HD) * kLog2e;

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
  constexpr int STEP = NW * TPW * U;
  // software pipeline (G <= 2): the next step's K/V loads are in flight while
  // this step's softmax runs (two steps of 16-byte loads per thread)
  constexpr bool PF = G <= 2;
  uint4 kr[U], vr[U], kn[U], vn[U];
  bool valid[U], vnx[U];
  // K/V are read once per layer: evict-first, so they do not push
  // activations, split-K partials or metadata out of L2
  const uint64_t kvpol = l2_evict_first_policy();
  auto issue = [&](int base, uint4* K, uint4* Vv, bool* ok) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = base + (u * NW + warp) * TPW + tg;
      ok[u] = t < t_end;
      const int tt = ok[u] ? t : t_begin;
      const int blk = bt[tt >> 4];
      const int64_t kb = (((int64_t)blk * 2) * p.Hkv + kh) * head_stride + (tt & 15) * HD + sub * 8;
      K[u] = ld_nc_v4_ef(p.kv + kb, kvpol);
      Vv[u] = ld_nc_v4_ef(p.kv + kb + (int64_t)p.Hkv * head_stride, kvpol);
    }
  };
  // The first step's K/V loads go out before the PDL wait: every context
  // token except the newest was written by earlier steps, so they overlap the
  // tail of the QKV kernel.  After the wait, the thread holding the newest
  // token (written by that kernel) reloads it through L2 (ld.cg: the
  // pre-wait load may have left a stale line in L1), and q is read.
  const bool fused = p.qkv_ws != nullptr;
  // fused mode: the newest token's k / v do not exist yet (they are in the
  // QKV partials); it is left out of the streamed range and added last
  const bool has_new = fused && newest >= t_begin && newest < t_end;
  if (has_new) t_end = newest;
  issue(t_begin, kr, vr, valid);
  pdl_wait();
  __shared__ __align__(16) bf16 s_qkv[(G + 2) * HD];
  if (fused) {
    // the QKV split-K epilogue, done cooperatively (all loads in flight at
    // once): q of the G heads of kv head kh, plus k / v of the newest token
    // when this CTA holds it; sum in split order, RoPE at position ctx-1 on
    // the interleaved (i, i+hd/2) pairs, bf16 -- as splitk_reduce_kernel
    const int npairs = (G + (has_new ? 2 : 0)) * (HD / 2);
    for (int pi = threadIdx.x; pi < npairs; pi += NW * 32) {
      const int e = pi * 2;
      int f;
      bool rope = true;
      if (e < G * HD) f = kh * G * HD + e;
      else if (e < (G + 1) * HD) f = (H + kh) * HD + (e - G * HD);
      else { f = (H + p.Hkv + kh) * HD + (e - (G + 1) * HD); rope = false; }
      float2 pr[8];
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2)
        if (s2 < p.qkv_splits)
          pr[s2] = __ldcg(reinterpret_cast<const float2*>(p.qkv_ws + ((int64_t)s2 * p.n + seq) * p.nqkv + f));
      const float2 cs = rope ? *reinterpret_cast<const float2*>(p.rope_cs + ((int64_t)newest * (HD >> 1) + ((f % HD) >> 1)) * 2)
                             : make_float2(1.f, 0.f);
      float v0 = 0.f, v1 = 0.f;
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2)
        if (s2 < p.qkv_splits) { v0 += pr[s2].x; v1 += pr[s2].y; }
      for (int s2 = 8; s2 < p.qkv_splits; ++s2) {
        const float2 q2 = __ldcg(reinterpret_cast<const float2*>(p.qkv_ws + ((int64_t)s2 * p.n + seq) * p.nqkv + f));
        v0 += q2.x;
        v1 += q2.y;
      }
      float r0 = v0, r1 = v1;
      if (rope) {
        r0 = v0 * cs.x - v1 * cs.y;
        r1 = v1 * cs.x + v0 * cs.y;
      }
      *reinterpret_cast<uint32_t*>(s_qkv + e) = pack_bf16x2(r0, r1);
    }
    __syncthreads();
    if (has_new && warp == 0 && tg == 0) {   // the new token's K / V into the paged cache
      const int64_t kb = (((int64_t)bt[newest >> 4] * 2) * p.Hkv + kh) * head_stride + (newest & 15) * HD + sub * 8;
      bf16* kvw = const_cast<bf16*>(p.kv);
      *reinterpret_cast<uint4*>(kvw + kb) = *reinterpret_cast<const uint4*>(s_qkv + G * HD + sub * 8);
      *reinterpret_cast<uint4*>(kvw + kb + (int64_t)p.Hkv * head_stride) =
          *reinterpret_cast<const uint4*>(s_qkv + (G + 1) * HD + sub * 8);
    }
  } else {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = t_begin + (u * NW + warp) * TPW + tg;
      if (t == newest) {
        const int64_t kb = (((int64_t)bt[t >> 4] * 2) * p.Hkv + kh) * head_stride + (t & 15) * HD + sub * 8;
        kr[u] = __ldcg(reinterpret_cast<const uint4*>(p.kv + kb));
        vr[u] = __ldcg(reinterpret_cast<const uint4*>(p.kv + kb + (int64_t)p.Hkv * head_stride));
      }
    }
  }
  float q[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const uint4 u = fused ? *reinterpret_cast<const uint4*>(s_qkv + g * HD + sub * 8)
                          : *reinterpret_cast<const uint4*>(p.q + ((int64_t)seq * H + kh * G + g) * HD + sub * 8);
    bf16x8_to_f32(u, q[g]);
#pragma unroll
    for (int i = 0; i < 8; ++i) q[g][i] *= scale;
  }
  for (int base = t_begin; base < t_end; base += STEP) {
    if (PF && base + STEP < t_end) issue(base + STEP, kn, vn, vnx);
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
    if (base + STEP < t_end) {
      if (PF) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          kr[u] = kn[u];
          vr[u] = vn[u];
          valid[u] = vnx[u];
        }
      } else {
        issue(base + STEP, kr, vr, valid);
      }
    }
  }
  if (has_new && warp == 0) {   // fused mode: the newest token, by thread group 0 of warp 0
    float kf[8], vf[8];
    bf16x8_to_f32(*reinterpret_cast<const uint4*>(s_qkv + G * HD + sub * 8), kf);
    bf16x8_to_f32(*reinterpret_cast<const uint4*>(s_qkv + (G + 1) * HD + sub * 8), vf);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float sc = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) sc = fmaf(q[g][i], kf[i], sc);
#pragma unroll
      for (int o = LPT / 2; o > 0; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
      if (tg == 0) {
        const float mn = fmaxf(m[g], sc);
        const float corr = exp2f(m[g] - mn);
        const float pr = exp2f(sc - mn);
        l[g] = l[g] * corr + pr;
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[g][i] = fmaf(pr, vf[i], acc[g][i] * corr);
        m[g] = mn;
      }
    }
  }
  attn_finish<HD, G>(p, seq, kh, split, n_splits, m, l, acc);
}

#ifndef TDP_ATTN_MINB
#define TDP_ATTN_MINB 5   // resident CTAs per SM for G = 1 (MHA): 96 registers, no spills; 6 spills (measured)
#endif
template <int HD, int G>
__global__ void __launch_bounds__(128, G == 1 ? TDP_ATTN_MINB : 1)
decode_attn_kernel(DecodeAttnParams p) {
  pdl_trigger_tail(G == 1 ? TDP_ATTN_MINB : G <= 4 ? 3 : 2);   // resident CTAs per SM (registers)
  // ctx / block tables are host-uploaded metadata (complete before the
  // previous kernel ran): read before the PDL wait, which attend_range takes
  const int seq = blockIdx.z, kh = blockIdx.y, split = blockIdx.x;
  const int ctx = p.ctx[seq];
  const int len = p.split_tokens;
  const int n_splits = (ctx + len - 1) / len;
  if (split >= n_splits) {
    pdl_wait();
    return;
  }
  const int t_begin = split * len;
  attend_range<HD, G>(p, seq, kh, t_begin, min(ctx, t_begin + len), split, n_splits, ctx - 1);
}

// ---------------------------------------------------------------- decode v2
// Page-streaming variant: a producer warp copies whole K and V pages (16 tokens
// x hd, contiguous in the paged pool) into an R-slot shared-memory ring with
// cp.async.bulk + mbarrier transaction counts; 4 consumer warps each own every
// 4th page and compute scores / online softmax / PV from shared memory.  The
// in-flight bytes live in smem rather than registers, so a few CTAs per SM keep
// enough of HBM busy even for small batches with long contexts.
namespace {
TDP_DEV void dmbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
TDP_DEV void dmbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(smem_u32(b)), "r"(parity) : "memory");
}
TDP_DEV void dmbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
TDP_DEV void dmbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
TDP_DEV void dbulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
}  // namespace

template <int HD, int G, int RW>
__global__ void __launch_bounds__(160)
decode_attn_v2_kernel(DecodeAttnParams p) {
  constexpr int LPT = HD / 8, TPW = 32 / LPT, NWC = 4;
  constexpr int R = NWC * RW;                      // ring slots (RW per consumer warp)
  constexpr int PAGE = kBlock * HD * 2;            // bytes of one K (or V) page
  extern __shared__ __align__(128) uint8_t dsm[];
  uint8_t* ring = dsm;                             // R x (K page, V page)
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm + R * 2 * PAGE);
  uint64_t* empty = full + R;
  float* sm = reinterpret_cast<float*>(empty + R);            // [NWC][G][2]
  float* sacc = sm + NWC * G * 2;                             // [NWC][G][HD]
  __shared__ int s_last;

  pdl_trigger();
  const int seq = blockIdx.z, kh = blockIdx.y, split = blockIdx.x;
  const int ctx = p.ctx[seq];
  const int n_splits = (ctx + p.split_tokens - 1) / p.split_tokens;
  if (split >= n_splits) return;
  const int t_begin = split * p.split_tokens;
  const int t_end = min(ctx, t_begin + p.split_tokens);
  const int pg0 = t_begin >> 4, npg = ((t_end + 15) >> 4) - pg0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = p.H;
  if (threadIdx.x == 0) {
    for (int i = 0; i < R; ++i) {
      dmbar_init(&full[i], 1);
      dmbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  const int32_t* bt = p.bt + (int64_t)seq * p.maxblk;
  const int64_t head_stride = (int64_t)kBlock * HD;

  if (warp == NWC) {   // producer
    if (lane == 0) {
      // page i belongs to consumer warp i % NWC, which owns slots
      // [w*RW, (w+1)*RW) and consumes them strictly in order (one consumer per
      // barrier: a parity wait can never be two phases ahead)
      for (int i = 0; i < npg; ++i) {
        const int w = i % NWC, j = i / NWC;
        const int s = w * RW + j % RW;
        if (j >= RW) dmbar_wait(&empty[s], ((j / RW) & 1) ^ 1);
        const int blk = bt[pg0 + i];
        const bf16* kp = p.kv + (((int64_t)blk * 2) * p.Hkv + kh) * head_stride;
        dmbar_expect(&full[s], 2 * PAGE);
        dbulk(ring + s * 2 * PAGE, kp, PAGE, &full[s]);
        dbulk(ring + s * 2 * PAGE + PAGE, kp + (int64_t)p.Hkv * head_stride, PAGE, &full[s]);
      }
    }
  } else {
    const int tg = lane / LPT, sub = lane % LPT;
    const float scale = rsqrtf((float)HD) * kLog2e;
    float q[G][8], m[G], l[G], acc[G][8];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint4 u = *reinterpret_cast<const uint4*>(p.q + ((int64_t)seq * H + kh * G + g) * HD + sub * 8);
      bf16x8_to_f32(u, q[g]);
#pragma unroll
      for (int i = 0; i < 8; ++i) q[g][i] *= scale;
      m[g] = -INFINITY;
      l[g] = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[g][i] = 0.f;
    }
    for (int i = warp; i < npg; i += NWC) {
      const int j = i / NWC;
      const int s = warp * RW + j % RW;
      dmbar_wait(&full[s], (j / RW) & 1);
      const uint8_t* kpg = ring + s * 2 * PAGE;
      const uint8_t* vpg = kpg + PAGE;
      const int tbase = (pg0 + i) << 4;
#pragma unroll
      for (int it = 0; it < kBlock / TPW; ++it) {
        const int r = it * TPW + tg;                 // token row inside the page
        const bool valid = tbase + r < t_end;
        float kf[8], vf[8];
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(kpg + (r * HD + sub * 8) * 2), kf);
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(vpg + (r * HD + sub * 8) * 2), vf);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          float sc = 0.f;
#pragma unroll
          for (int k = 0; k < 8; ++k) sc = fmaf(q[g][k], kf[k], sc);
#pragma unroll
          for (int o = LPT / 2; o > 0; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
          if (valid) {
            const float mn = fmaxf(m[g], sc);
            const float corr = exp2f(m[g] - mn);
            const float pr = exp2f(sc - mn);
            l[g] = l[g] * corr + pr;
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[g][k] = fmaf(pr, vf[k], acc[g][k] * corr);
            m[g] = mn;
          }
        }
      }
      __syncwarp();
      if (lane == 0) dmbar_arrive(&empty[s]);
    }
    // merge the token groups of the warp, then the warps through smem
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
        for (int k = 0; k < 8; ++k) {
          const float a2 = __shfl_xor_sync(0xffffffffu, acc[g][k], o);
          acc[g][k] = acc[g][k] * c1 + a2 * c2;
        }
        m[g] = mn;
      }
    }
    if (tg == 0) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (sub == 0) {
          sm[(warp * G + g) * 2] = m[g];
          sm[(warp * G + g) * 2 + 1] = l[g];
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) sacc[(warp * G + g) * HD + sub * 8 + k] = acc[g][k];
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < G * HD; e += blockDim.x) {
    const int g = e / HD, dim = e % HD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < NWC; ++w) M = fmaxf(M, sm[(w * G + g) * 2]);
    float L = 0.f, A = 0.f;
#pragma unroll
    for (int w = 0; w < NWC; ++w) {
      const float c = M == -INFINITY ? 0.f : exp2f(sm[(w * G + g) * 2] - M);
      L += sm[(w * G + g) * 2 + 1] * c;
      A += sacc[(w * G + g) * HD + dim] * c;
    }
    const int h = kh * G + g;
    if (n_splits == 1) {
      p.o[((int64_t)seq * H + h) * HD + dim] = __float2bfloat16_rn(A / L);
    } else {
      float* part = p.part + (((int64_t)seq * H + h) * p.max_splits + split) * (HD + 2);
      __stcg(part + 2 + dim, A);
      if (dim == 0) {
        __stcg(part, M);
        __stcg(part + 1, L);
      }
    }
  }
  if (n_splits == 1) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&p.counters[seq * p.Hkv + kh], 1) == n_splits - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int e = threadIdx.x; e < G * HD; e += blockDim.x) {
    const int g = e / HD, dim = e % HD;
    const int h = kh * G + g;
    const float* part = p.part + ((int64_t)seq * H + h) * p.max_splits * (HD + 2);
    float M = -INFINITY;
    for (int s2 = 0; s2 < n_splits; ++s2) M = fmaxf(M, __ldcg(part + s2 * (HD + 2)));
    float L = 0.f, A = 0.f;
    for (int s2 = 0; s2 < n_splits; ++s2) {
      const float* ps = part + s2 * (HD + 2);
      const float c = exp2f(__ldcg(ps) - M);
      L += __ldcg(ps + 1) * c;
      A += __ldcg(ps + 2 + dim) * c;
    }
    p.o[((int64_t)seq * H + h) * HD + dim] = __float2bfloat16_rn(A / L);
  }
  if (threadIdx.x == 0) p.counters[seq * p.Hkv + kh] = 0;
}

template <int HD, int G>
static void launch_v2(const DecodeAttnParams& p, cudaStream_t st) {
  constexpr int RW = 2;
  constexpr int R = 4 * RW;
  constexpr int smem = R * 2 * kBlock * HD * 2 + R * 16 + 4 * G * 2 * 4 + 4 * G * HD * 4 + 64;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(decode_attn_v2_kernel<HD, G, RW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  launch_k(decode_attn_v2_kernel<HD, G, RW>, dim3(p.max_splits, p.Hkv, p.n), dim3(160), smem, st, p);
}

static bool v2_enabled() {   // TDPIPE_ATTN_V2=1: smem page-ring kernel (measured slower; A/B only)
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("TDPIPE_ATTN_V2");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  return on == 1;
}

template <int HD>
static void launch_decode_hd(const DecodeAttnParams& p, cudaStream_t st) {
  const int G = p.H / p.Hkv;
  if (v2_enabled() && !p.qkv_ws) {
    switch (G) {
      case 1: launch_v2<HD, 1>(p, st); return;
      case 2: launch_v2<HD, 2>(p, st); return;
      case 4: launch_v2<HD, 4>(p, st); return;
      case 8: launch_v2<HD, 8>(p, st); return;
      default: return;
    }
  }
  dim3 grid(p.max_splits, p.Hkv, p.n);
  switch (G) {
    case 1: launch_k(decode_attn_kernel<HD, 1>, grid, dim3(128), 0, st, p); break;
    case 2: launch_k(decode_attn_kernel<HD, 2>, grid, dim3(128), 0, st, p); break;
    case 4: launch_k(decode_attn_kernel<HD, 4>, grid, dim3(128), 0, st, p); break;
    case 8: launch_k(decode_attn_kernel<HD, 8>, grid, dim3(128), 0, st, p); break;
    default: return;
  }

}

void plan_decode_attn(DecodeAttnParams& p, const int* ctx) {
  // split size: the largest of 512/256/128 context tokens that still yields
  // >= 8 CTAs per SM over the batch's actual context lengths (short CTAs of
  // similar size balance the wave tail; >= 128 tokens amortise a CTA); the
  // page-ring kernel keeps 6 pages in flight per CTA, so it wants fewer,
  // longer CTAs: one resident wave of ~4 per SM
  const bool v2 = v2_enabled();
  // A/B knobs: CTA target per SM, largest split (tokens, power of two >= 128)
  static const int tgt_env = std::getenv("TDPIPE_ATTN_TARGET") ? std::atoi(std::getenv("TDPIPE_ATTN_TARGET")) : 0;
  static const int max_env = std::getenv("TDPIPE_ATTN_MAXSPLIT") ? std::atoi(std::getenv("TDPIPE_ATTN_MAXSPLIT")) : 0;
  const int64_t target = (int64_t)(tgt_env > 0 ? tgt_env : (v2 ? 4 : 8)) * 148;
  int split = max_env >= kAttnMinSplit ? max_env : 512, max_ctx = 1;
  for (int i = 0; i < p.n; ++i) max_ctx = std::max(max_ctx, ctx[i]);
  for (;;) {
    int64_t ctas = 0;
    for (int i = 0; i < p.n; ++i) ctas += (ctx[i] + split - 1) / split;
    if (ctas * p.Hkv >= target || split <= (v2 ? 256 : kAttnMinSplit)) break;
    split >>= 1;
  }
  // Small batches: the grid is only Hkv x n x splits CTAs (GQA: few kv
  // heads).  While that is below one CTA per SM, halve the
  // split (down to 32 tokens) as long as a sequence keeps <= 8 splits (one
  // merge round trip) and the workspace holds the partials.  Measured on
  // Llama-2-70B heads (profiles/r1/attn_sweep_gqa8_small.txt): 1.6x at
  // n <= 4 x 256 tokens (MHA, Llama-2-7B heads: 1.1-1.3x at n <= 2 x 256);
  // more splits than 8, or splitting a grid that already has >= 1 CTA per
  // SM, was slower.
  const int G = p.H / p.Hkv;
  if (!v2 && split == kAttnMinSplit) {
    for (;;) {
      int64_t ctas = 0;
      for (int i = 0; i < p.n; ++i) ctas += (ctx[i] + split - 1) / split;
      const int nsplit = split / 2;
      const int64_t nsplits = (max_ctx + nsplit - 1) / nsplit;
      if (ctas * p.Hkv >= 148 || nsplit < kAttnMinSplitGQA || nsplits > 8) break;
      if ((int64_t)p.n * nsplits > p.part_cap) break;
      split = nsplit;
    }
  }
  p.split_tokens = split;
  p.max_splits = (max_ctx + split - 1) / split;
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
// Varlen causal flash attention on tensor cores (mma.sync m16n8k16 bf16, fp32
// softmax), K/V read from the paged cache the QKV epilogue just wrote.  Grid:
// (64-query tile, sequence, head); 4 warps x 16 query rows; 64-key tiles
// double-buffered with cp.async; S = Q K^T and O += P V with P kept in
// registers (accumulator layout == A-fragment layout).  Prefill is < 1% of the
// prefill FLOPs at ShareGPT lengths, so mma.sync suffices.
namespace {
TDP_DEV void ldsm_x4(uint32_t* r, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
TDP_DEV void ldsm_x4_t(uint32_t* r, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
TDP_DEV void mma_bf16(float* c, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
template <int HD>
TDP_DEV int fswz(int r, int c) {   // 16-byte chunk index inside a [64][HD] bf16 tile
  constexpr int CH = HD / 8;
  int pc;
  if constexpr (CH >= 8) pc = c ^ (r & 7);
  else if constexpr (CH == 4) pc = c ^ ((r >> 1) & 3);
  else pc = c ^ ((r >> 2) & 1);
  return r * CH + pc;
}
}  // namespace

template <int HD>
__global__ void __launch_bounds__(128) flash_prefill_kernel(PrefillAttnParams p) {
  constexpr int BQ = 64, BKV = 64, CH = HD / 8;
  constexpr int TILE = BQ * HD * 2;
  extern __shared__ __align__(128) uint8_t fsm[];
  uint8_t* sQ = fsm;
  uint8_t* sK = fsm + TILE;          // 2 stages
  uint8_t* sV = fsm + 3 * TILE;      // 2 stages
  pdl_trigger_tail(2);
  pdl_wait();
  const int qt = blockIdx.x, seq = blockIdx.y, h = blockIdx.z;
  const int L = p.seq_ctx[seq];                  // keys: positions 0 .. L-1
  const int qs = p.seq_qstart ? p.seq_qstart[seq] : 0;
  const int nq = L - qs;                         // queries: positions qs .. L-1
  const int q0 = qt * BQ;                        // (query indices relative to qs)
  if (q0 >= nq) return;
  const int row0 = p.seq_last[seq] - nq + 1;    // token row of query 0
  const int G = p.H / p.Hkv, kh = h / G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int32_t* bt = p.bt + (int64_t)seq * p.maxblk;
  const int64_t head_stride = (int64_t)kBlock * HD;

  // Q tile
  for (int i = tid; i < BQ * CH; i += 128) {
    const int r = i / CH, c = i % CH;
    const int q = q0 + r;
    const bf16* src = p.q + ((int64_t)(row0 + (q < nq ? q : 0)) * p.H + h) * HD + c * 8;
    cp_async16(sQ + fswz<HD>(r, c) * 16, src, q < nq);
  }
  auto load_kv = [&](int stage, int k0) {
    for (int i = tid; i < BKV * CH; i += 128) {
      const int r = i / CH, c = i % CH;
      const int j = k0 + r;
      const bool ok = j < L;
      const int jj = ok ? j : 0;
      const int64_t base = (((int64_t)bt[jj >> 4] * 2) * p.Hkv + kh) * head_stride + (jj & 15) * HD + c * 8;
      cp_async16(sK + stage * TILE + fswz<HD>(r, c) * 16, p.kv + base, ok);
      cp_async16(sV + stage * TILE + fswz<HD>(r, c) * 16, p.kv + base + (int64_t)p.Hkv * head_stride, ok);
    }
  };
  const int last_q = qs + min(q0 + BQ, nq) - 1;   // absolute position of the tile's last query
  const int n_kt = last_q / BKV + 1;
  load_kv(0, 0);
  cp_async_commit();

  const float sl2 = rsqrtf((float)HD) * kLog2e;
  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  uint32_t qf[HD / 16][4];
  const int g = lane >> 2, tq = lane & 3;
  const int qr0 = q0 + warp * 16 + g;     // this thread's two queries (relative): qr0, qr0 + 8

  for (int kt = 0; kt < n_kt; ++kt) {
    if (kt + 1 < n_kt) load_kv((kt + 1) & 1, (kt + 1) * BKV);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        ldsm_x4(qf[kk], smem_u32(sQ + fswz<HD>(warp * 16 + (lane & 15), kk * 2 + (lane >> 4)) * 16));
    }
    const uint8_t* K = sK + (kt & 1) * TILE;
    const uint8_t* V = sV + (kt & 1) * TILE;
    float s[BKV / 8][4];
#pragma unroll
    for (int i = 0; i < BKV / 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
      for (int nb = 0; nb < BKV / 16; ++nb) {
        uint32_t b[4];
        const int r = nb * 16 + (lane & 7) + ((lane >> 4) << 3);
        ldsm_x4(b, smem_u32(K + fswz<HD>(r, kk * 2 + ((lane >> 3) & 1)) * 16));
        mma_bf16(s[2 * nb], qf[kk], b);
        mma_bf16(s[2 * nb + 1], qf[kk], b + 2);
      }
    }
    // scale, causal + length mask, online softmax (rows qr0 and qr0 + 8)
    const int k0 = kt * BKV;
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int ni = 0; ni < BKV / 8; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = k0 + ni * 8 + 2 * tq + (e & 1);
        const int qp = qs + qr0 + (e >> 1) * 8;   // absolute query position (causal bound)
        const float v = (key <= qp && key < L) ? s[ni][e] * sl2 : -INFINITY;
        s[ni][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
    float corr[2];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      mx[rr] = fmaxf(mx[rr], __shfl_xor_sync(0xffffffffu, mx[rr], 1));
      mx[rr] = fmaxf(mx[rr], __shfl_xor_sync(0xffffffffu, mx[rr], 2));
      const float mn = fmaxf(m_r[rr], mx[rr]);
      corr[rr] = mn == -INFINITY ? 1.f : exp2f(m_r[rr] - mn);
      m_r[rr] = mn;
    }
    float rs[2] = {0.f, 0.f};
#pragma unroll
    for (int ni = 0; ni < BKV / 8; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float mm = m_r[e >> 1];
        const float pv = mm == -INFINITY ? 0.f : exp2f(s[ni][e] - mm);
        s[ni][e] = pv;
        rs[e >> 1] += pv;
      }
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      rs[rr] += __shfl_xor_sync(0xffffffffu, rs[rr], 1);
      rs[rr] += __shfl_xor_sync(0xffffffffu, rs[rr], 2);
      l_r[rr] = l_r[rr] * corr[rr] + rs[rr];
    }
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      o[i][0] *= corr[0];
      o[i][1] *= corr[0];
      o[i][2] *= corr[1];
      o[i][3] *= corr[1];
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < BKV / 16; ++kk) {
      uint32_t a[4];
      a[0] = pack_bf16x2(s[2 * kk][0], s[2 * kk][1]);
      a[1] = pack_bf16x2(s[2 * kk][2], s[2 * kk][3]);
      a[2] = pack_bf16x2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      a[3] = pack_bf16x2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int dn = 0; dn < HD / 16; ++dn) {
        uint32_t b[4];
        const int r = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
        ldsm_x4_t(b, smem_u32(V + fswz<HD>(r, dn * 2 + (lane >> 4)) * 16));
        mma_bf16(o[2 * dn], a, b);
        mma_bf16(o[2 * dn + 1], a, b + 2);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int q = qr0 + rr * 8;
    if (q >= nq) continue;
    const float inv = 1.f / l_r[rr];
    bf16* dst = p.o + ((int64_t)(row0 + q) * p.H + h) * HD;
#pragma unroll
    for (int ni = 0; ni < HD / 8; ++ni)
      *reinterpret_cast<uint32_t*>(dst + ni * 8 + 2 * tq) = pack_bf16x2(o[ni][2 * rr] * inv, o[ni][2 * rr + 1] * inv);
  }
}

template <int HD>
static void launch_flash(const PrefillAttnParams& p, cudaStream_t st) {
  constexpr int smem = 5 * 64 * HD * 2;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(flash_prefill_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid((p.max_len + 63) / 64, p.n_seqs, p.H);
  launch_k(flash_prefill_kernel<HD>, grid, dim3(128), smem, st, p);
}

void launch_prefill_attn(const PrefillAttnParams& p, cudaStream_t st) {
  if (p.T <= 0) return;
  switch (p.hd) {
    case 16: launch_flash<16>(p, st); break;
    case 32: launch_flash<32>(p, st); break;
    case 64: launch_flash<64>(p, st); break;
    case 128: launch_flash<128>(p, st); break;
  }
}

}  // namespace tdp
