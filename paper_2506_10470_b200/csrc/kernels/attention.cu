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

#include <cudaTypedefs.h>

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

// ------------------------------------------------------ decode, tensor cores
// GQA decode attention on tensor cores (G = H/Hkv query heads share each K/V
// page; Table 2's 32B / 70B models are GQA).  One CTA per
// (split, kv head, sequence), as the SIMT kernel, but:
//  * a producer warp streams the split's 16-token K and V pages with TMA
//    (cp.async.bulk.tensor, 128B-swizzled 64-column boxes, L2 evict-first)
//    into an R-slot shared-memory ring (mbarrier transaction counts), so a CTA
//    keeps R x 8 KB in flight without holding it in registers;
//  * 4 consumer warps each take every 4th page (slot = page mod R, R a
//    multiple of 4: one consumer per slot, never two phases ahead) and compute
//    transposed tiles on mma.sync m16n8k16 (bf16 in, fp32 accumulate):
//      S^T[16 tokens x 8 heads]  = K[16 x hd] . Q^T[hd x 8]       (8 HMMA)
//      O^T[hd x 8 heads]        += V^T[hd x 16] . P^T[16 x 8]      (8 HMMA)
//    with the G <= 8 heads as the n = 8 dimension (no padding for G = 8);
//    K is the row-major A operand (ldmatrix), V^T comes from ldmatrix.trans,
//    and P^T is the exp2'd S^T accumulator transposed in registers with
//    movmatrix (the C layout of S^T is the B layout of P^T after an 8x8
//    transpose), so P never touches shared memory;
//  * online softmax per head (a column of S^T): column max over the 16 tokens
//    with 3 shuffles, per-thread partial sums reduced once at the end;
//  * warps merge through shared memory, then the split merge of the SIMT
//    kernel (partials in split order, last CTA merges).
// q comes from the QKV GEMM's epilogue (or its split-K reduce), which has also
// written the newest token's K / V into the cache: the kernel never runs in the
// SIMT kernel's fused-QKV mode (launch_decode_attn falls back if asked to).
namespace {
TDP_DEV void tc_mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
TDP_DEV void tc_mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(smem_u32(b)), "r"(parity) : "memory");
}
#ifdef TDP_TC_PROF
// measurement build only: cycles per wait site summed over lane 0 of every warp
__device__ unsigned long long g_tc_prof[16];
#define TC_PW(k, ...)                       \
  do {                                      \
    const long long t0_ = clock64();        \
    __VA_ARGS__;                            \
    prof[k] += clock64() - t0_;             \
  } while (0)
#else
#define TC_PW(k, ...) __VA_ARGS__
#endif
TDP_DEV void tc_mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
TDP_DEV void tc_mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
TDP_DEV void tma_load_4d_ef(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3, uint64_t* bar,
                            uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, "
      "%4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
TDP_DEV void ldsm4(uint32_t* r, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
TDP_DEV void ldsm4_t(uint32_t* r, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
TDP_DEV uint32_t movm_t(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
  return d;
}
TDP_DEV void hmma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// byte offset of (row r, 16-byte chunk ch) in a page staged as hd/64 boxes of
// [16 rows][128 B] with the 128B swizzle (chunk ^ (row & 7))
// a page staged by ONE 4-D box (64 columns x hd/64 halves x 16 rows): 128-B row
// segments ordered (row, half), 128B swizzle on the segment index
template <int NB>
TDP_DEV uint32_t page_off(int r, int ch) {
  const int seg = r * NB + (ch >> 3);
  return (uint32_t)(seg * 128 + (((ch & 7) ^ (seg & 7)) << 4));
}
}  // namespace

// n contiguous floats from shared memory (16-byte aligned for n % 4 == 0, else 8)
template <int N>
TDP_DEV void ld_vec(float (&v)[N], const float* src) {
  if constexpr (N % 4 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 4) {
      const float4 t = *reinterpret_cast<const float4*>(src + i);
      v[i] = t.x; v[i + 1] = t.y; v[i + 2] = t.z; v[i + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      const float2 t = *reinterpret_cast<const float2*>(src + i);
      v[i] = t.x; v[i + 1] = t.y;
    }
  }
}
// n floats -> n contiguous bf16 (round to nearest), one store of 2n bytes
template <int N>
TDP_DEV void st_bf16_vec(bf16* dst, const float (&r)[N]) {
  if constexpr (N == 2) {
    *reinterpret_cast<uint32_t*>(dst) = pack_bf16x2(r[0], r[1]);
  } else {
#pragma unroll
    for (int i = 0; i < N; i += 4)
      *reinterpret_cast<uint2*>(dst + i) = make_uint2(pack_bf16x2(r[i], r[i + 1]), pack_bf16x2(r[i + 2], r[i + 3]));
  }
}

constexpr int kTcRing = 8;          // page ring slots (a multiple of the 4 consumer warps)
constexpr int kTcItemQ = 3;         // work items in flight per CTA (queue slots)
constexpr int kTcThreads = 224;     // 4 consumer warps, producer, q-prep, merger
constexpr int kTcPad = 4;           // sO row padding (floats): conflict-free fragment stores
constexpr int kTcMaxSplits = 32;    // split merge weights held in shared memory

// Shared-memory layout of decode_attn_tc_kernel (dynamic part), in bytes.
template <int HD, int G>
struct TcLayout {
  static constexpr int PAGE = kBlock * HD * 2;                 // one K (or V) page
  static constexpr int SLOT = 2 * PAGE;
  static constexpr int RING = kTcRing * SLOT;
  static constexpr int OBUF = 4 * (G * (HD + kTcPad) + 2 * 8) * 4;   // 4 warps: O^T rows, then m[8], l[8]
  static constexpr int QBUF = G * HD * 2;                      // q of the G heads
  static constexpr int BARS = (2 * kTcRing + 3 * kTcItemQ + 4) * 8;
  static constexpr int FIXED = RING + 2 * OBUF + kTcItemQ * QBUF + BARS + 1024;   // + alignment
  static int bytes(int n) { return FIXED + (n + 1) * 4; }
};

// Persistent, warp-specialised pipeline.  Work items are (sequence, split,
// kv head), numbered sequence-major over the non-empty splits; a CTA takes
// items from an atomic counter until they run out:
//   producer  (warp 4): fetches item indices into a kTcItemQ-slot queue and
//             streams each item's K / V pages into the page ring by TMA
//             (block-table entries read 32 at a time by the whole warp);
//   q-prep    (warp 5): for each queued item stages q of its G heads in
//             shared memory (one bulk copy);
//   consumers (warps 0-3): per item, tensor-core S^T / online softmax / O^T
//             over every 4th page, then their (m, l, O) into one of two
//             result buffers;
//   merger    (warp 6): combines the 4 warps, writes o or the split
//             partial, and the last split of a
//             (sequence, kv head) merges all partials in split order.
// So q loads, merges and split merges of one item overlap the page streaming
// of the next.  Local page j of an item always goes to consumer warp j mod 4
// (only the ring slot -- one of that warp's own slots -- depends on the CTA's
// history), so each item is computed identically whichever CTA takes it:
// results are bitwise reproducible.
template <int HD, int G>
__global__ void __launch_bounds__(kTcThreads, 2)
decode_attn_tc_kernel(const __grid_constant__ CUtensorMap kvmap, DecodeAttnParams p) {
  using Lay = TcLayout<HD, G>;
  constexpr int NWC = 4, R = kTcRing, Q = kTcItemQ;
  constexpr int PAGE = Lay::PAGE, SLOT = Lay::SLOT;
  constexpr int NB = HD / 64;                    // 64-column TMA boxes per page
  constexpr int KS = HD / 16;                    // k-steps of S^T / m-tiles of O^T
  constexpr int OS = HD + kTcPad;                // sO row stride (floats)
  constexpr int RW = R / 4;                      // ring slots per consumer warp
  constexpr int CPL = HD / 32;                   // merger: output columns per lane
  static_assert(G >= 1 && G <= 8 && R % NWC == 0, "layout");
  extern __shared__ uint8_t tc_smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
  float* obuf = reinterpret_cast<float*>(ring + Lay::RING);                  // [2][OBUF]
  bf16* qbuf = reinterpret_cast<bf16*>(ring + Lay::RING + 2 * Lay::OBUF);  // [Q][(G+2) HD]
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + Lay::RING + 2 * Lay::OBUF + Q * Lay::QBUF);
  uint64_t* empty = full + R;
  uint64_t* ifull = empty + R;     // item queued (producer)
  uint64_t* qready = ifull + Q;    // its q staged (q-prep)
  uint64_t* iempty = qready + Q;   // its slot free again (merger)
  uint64_t* oready = iempty + Q;   // [2] result buffer written (4 consumer warps)
  uint64_t* ofree = oready + 2;    // [2] result buffer read (merger)
  int* pfx = reinterpret_cast<int*>(ofree + 2);                      // [n + 1] split prefix sums
  __shared__ int s_item[Q];
  __shared__ float s_c[G][kTcMaxSplits];   // merger: split (m, then weights) and l
  __shared__ float s_l[G][kTcMaxSplits];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = p.H;
  const float scale = rsqrtf((float)HD) * kLog2e;
  struct Item {
    int seq, kh, split, n_splits, t_begin, t_end, pg0, npg;
  };
  // item idx = (pfx[r] + split) * Hkv + kh for the r-th sequence of p.order
  // (longest context first: long items are taken first, short ones fill the
  // tail); streamed range [t_begin, t_end)
  __shared__ Item s_desc[Q];   // the queued items, decoded once by the producer
  auto item_of = [&](int idx) {
    Item it;
    const int u = idx / p.Hkv;
    it.kh = idx - u * p.Hkv;
    int lo = 0, hi = p.n - 1;   // last seq with pfx[seq] <= u
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pfx[mid] <= u) lo = mid;
      else hi = mid - 1;
    }
    it.seq = p.order ? p.order[lo] : lo;
    it.split = u - pfx[lo];
    it.n_splits = pfx[lo + 1] - pfx[lo];
    const int ctx = p.ctx[it.seq];
    it.t_begin = it.split * p.split_tokens;
    it.t_end = min(ctx, it.t_begin + p.split_tokens);
    it.pg0 = it.t_begin >> 4;
    it.npg = it.t_end > it.t_begin ? ((it.t_end + 15) >> 4) - it.pg0 : 0;
    return it;
  };
  {   // pfx[i] = sum_{j < i} ceil(ctx[j] / split_tokens): contiguous chunks + a block scan
    __shared__ int s_wsum[kTcThreads / 32];
    const int per = (p.n + kTcThreads - 1) / kTcThreads;
    const int i0 = min(p.n, (int)threadIdx.x * per), i1 = min(p.n, i0 + per);
    int sum = 0;
    auto ctx_at = [&](int i) { return p.ctx[p.order ? p.order[i] : i]; };
    for (int i = i0; i < i1; ++i) sum += (ctx_at(i) + p.split_tokens - 1) / p.split_tokens;
    int incl = sum;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += v;
    }
    if (lane == 31) s_wsum[warp] = incl;
    if (threadIdx.x == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&kvmap)) : "memory");
      // "done reading / writing" barriers take one arrival per thread of the
      // releasing warp(s), so every thread's shared-memory accesses are
      // ordered before the buffer's reuse (racecheck-clean); "data ready"
      // barriers have one writer (or the TMA transaction count)
      for (int i = 0; i < R; ++i) {
        tc_mbar_init(&full[i], 1);
        tc_mbar_init(&empty[i], 32);
      }
      for (int i = 0; i < Q; ++i) {
        tc_mbar_init(&ifull[i], 1);
        tc_mbar_init(&qready[i], 1);
        tc_mbar_init(&iempty[i], 32);
      }
      for (int i = 0; i < 2; ++i) {
        tc_mbar_init(&oready[i], NWC * 32);
        tc_mbar_init(&ofree[i], 32);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int base = 0;
    for (int w = 0; w < warp; ++w) base += s_wsum[w];
    int run = base + incl - sum;
    for (int i = i0; i < i1; ++i) {
      pfx[i] = run;
      run += (ctx_at(i) + p.split_tokens - 1) / p.split_tokens;
    }
    if (threadIdx.x == kTcThreads - 1) pfx[p.n] = run;
  }
  __syncthreads();
  const int n_items = pfx[p.n] * p.Hkv;
#ifdef TDP_TC_PROF
  long long prof[16] = {};
  const long long prof_t0 = clock64();
#endif
  // Every K / V page, the newest token's included, and q were written by
  // earlier kernels; nothing is read before the wait.
  pdl_wait();

  if (warp == NWC) {   // ---------------------------------------------------- producer
    // Page j of an item goes to consumer warp j mod 4 and into one of that
    // warp's own ring slots (w, w + 4, ...): every slot has exactly one
    // consumer, which takes its pages in order, so a parity wait is never two
    // phases ahead even though the warps run items out of step.
    const uint64_t pol = l2_evict_first_policy();
    int c0 = 0, c1 = 0, c2 = 0, c3 = 0;   // pages issued per consumer warp
    // Item indices are fetched two items ahead and the first 32 block-table
    // entries of the next item are loaded while the current one streams, so
    // neither the counter's nor the table's round trip stalls the ring.
    auto fetch = [&]() {
      int v = 0;
      if (lane == 0) v = atomicAdd(p.work, 1);
      return v;
    };
    auto chunk0 = [&](int idx, Item& it) {
      if (idx < 0) return 0;
      it = item_of(idx);
      const int32_t* bt = p.bt + (int64_t)it.seq * p.maxblk + it.pg0;
      return lane < it.npg ? __ldg(bt + lane) : 0;
    };
    int cur = __shfl_sync(0xffffffffu, fetch(), 0);
    cur = cur < n_items ? cur : -1;
    int nxt = -1;
    if (cur >= 0) {
      nxt = __shfl_sync(0xffffffffu, fetch(), 0);
      nxt = nxt < n_items ? nxt : -1;
    }
    Item it_cur{}, it_nxt{};
    int bt_cur = chunk0(cur, it_cur), bt_nxt = chunk0(nxt, it_nxt);
    for (int n = 0;; ++n) {
      const int idx = cur;
      const int q = n % Q;
      if (n >= Q) TC_PW(0, tc_mbar_wait(&iempty[q], ((uint32_t)(n / Q) & 1u) ^ 1u));
      int pend = 0;
      if (lane == 0) {
        s_item[q] = idx;
        if (idx >= 0) s_desc[q] = it_cur;
        tc_mbar_arrive(&ifull[q]);
        if (idx < 0) pdl_trigger();   // no work left for this CTA: the next kernel may start its prologue
        else if (nxt >= 0) pend = atomicAdd(p.work, 1);
      }
      if (idx < 0) break;
      const Item it = it_cur;
      const int32_t* bt = p.bt + (int64_t)it.seq * p.maxblk + it.pg0;
      for (int j0 = 0; j0 < it.npg; j0 += 32) {
        const int btv = j0 == 0 ? bt_cur : (j0 + lane < it.npg ? __ldg(bt + j0 + lane) : 0);
        const int cn = min(32, it.npg - j0);
        for (int j = 0; j < cn; ++j) {
          const int blk = __shfl_sync(0xffffffffu, btv, j);
          const int w = (j0 + j) & 3;
          int& cw = w == 0 ? c0 : w == 1 ? c1 : w == 2 ? c2 : c3;
          const int s = w + NWC * (cw % RW), use = cw / RW;
          ++cw;
          if (use > 0) TC_PW(1, tc_mbar_wait(&empty[s], ((uint32_t)use & 1u) ^ 1u));
          // the page's K and V boxes are issued by 2 lanes at once, one 4-D box
          // each (not 2 x NB 64-column boxes from lane 0): the producer warp's
          // issue rate, not the ring,
          // limited the stream (profiling build TDP_TC_PROF: the producer waited for
          // a free slot only 8-10 % of its time while the consumers waited for
          // pages 56-73 %; profiles/r2/ab/tc_attn_*)
          TC_PW(12, {
            const int row = ((blk * 2) * p.Hkv + it.kh) * kBlock;
            uint8_t* dst = ring + s * SLOT;
            if (lane == 0) tc_mbar_expect(&full[s], SLOT);
            __syncwarp();
            if (lane < 2)   // K, V: one 4-D box each (both 64-column halves)
              tma_load_4d_ef(dst + lane * PAGE, &kvmap, 0, 0, row + lane * p.Hkv * kBlock, p.layer, &full[s], pol);
          });
        }
      }
      // rotate: the next item was fetched (and its table chunk loaded) one item ago
      TC_PW(13, {
        const int after = nxt >= 0 ? __shfl_sync(0xffffffffu, pend, 0) : -1;
        cur = nxt;
        it_cur = it_nxt;
        bt_cur = bt_nxt;
        nxt = after >= 0 && after < n_items ? after : -1;
        bt_nxt = chunk0(nxt, it_nxt);
      });
    }
  } else if (warp == NWC + 1) {   // ------------------------------------------ q-prep
    for (int n = 0;; ++n) {
      const int q = n % Q;
      TC_PW(2, tc_mbar_wait(&ifull[q], (uint32_t)(n / Q) & 1u));
      int idx = 0;
      if (lane == 0) idx = s_item[q];   // read by the lane whose qready arrival orders it
      idx = __shfl_sync(0xffffffffu, idx, 0);
      bf16* sq = qbuf + q * G * HD;
      if (idx < 0) {
        if (lane == 0) tc_mbar_arrive(&qready[q]);
        break;
      }
      if (lane == 0) {
        const Item it = s_desc[q];
        tc_mbar_expect(&qready[q], G * HD * 2);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(sq)),
            "l"(p.q + ((int64_t)it.seq * H + it.kh * G) * HD), "r"(G * HD * 2), "r"(smem_u32(&qready[q]))
            : "memory");
      }
    }
  } else if (warp == NWC + 2) {   // ------------------------------------------ merger
    for (int n = 0;; ++n) {
      const int q = n % Q, b = n & 1;
      TC_PW(3, tc_mbar_wait(&ifull[q], (uint32_t)(n / Q) & 1u));
      const int idx = s_item[q];
      if (idx < 0) break;
      const Item it = s_desc[q];
      TC_PW(4, tc_mbar_wait(&oready[b], (uint32_t)(n >> 1) & 1u));
      const float* so = obuf + b * (Lay::OBUF / 4);
      const float* sm = so + NWC * G * OS;      // [4][8]
      const float* sl = sm + NWC * 8;           // [4][8]
      // lane owns the CPL contiguous columns [lane CPL, lane CPL + CPL): vector
      // shared loads and one packed global store per head (the strided 2-byte
      // stores took 75-78 % of this warp at contexts 128-256; TDP_TC_PROF)
      float A[G][CPL], Mg[G], Lg[G];
#ifdef TDP_TC_PROF
      const long long tm0_ = clock64();
#endif
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < NWC; ++w) M = fmaxf(M, sm[w * 8 + g]);
        float c[NWC], L = 0.f;
#pragma unroll
        for (int w = 0; w < NWC; ++w) {
          c[w] = sm[w * 8 + g] == -INFINITY ? 0.f : exp2f(sm[w * 8 + g] - M);
          L += sl[w * 8 + g] * c[w];
        }
#pragma unroll
        for (int dd = 0; dd < CPL; ++dd) A[g][dd] = 0.f;
#pragma unroll
        for (int w = 0; w < NWC; ++w) {
          float v[CPL];
          ld_vec<CPL>(v, so + (w * G + g) * OS + lane * CPL);
#pragma unroll
          for (int dd = 0; dd < CPL; ++dd) A[g][dd] += v[dd] * c[w];
        }
        Mg[g] = M;
        Lg[g] = L;
      }
      const Item itc = it;
      tc_mbar_arrive(&ofree[b]);    // the consumers may reuse result buffer b
      tc_mbar_arrive(&iempty[q]);   // queue slot q (descriptor, q buffer) free: the results are in registers
#ifdef TDP_TC_PROF
      const long long tm1_ = clock64();
      prof[14] += tm1_ - tm0_;
#endif
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int h = itc.kh * G + g;
        if (itc.n_splits == 1) {
          // one reciprocal per head (as the split merge): no per-element
          // division, whose slow path a zero numerator takes
          const float inv = 1.f / Lg[g];
          float r[CPL];
#pragma unroll
          for (int dd = 0; dd < CPL; ++dd) r[dd] = A[g][dd] * inv;
          st_bf16_vec<CPL>(p.o + ((int64_t)itc.seq * H + h) * HD + lane * CPL, r);
        } else {
          float* part = p.part + (((int64_t)itc.seq * H + h) * p.max_splits + itc.split) * (HD + 2);
#pragma unroll
          for (int dd = 0; dd < CPL; dd += 2) __stcg(reinterpret_cast<float2*>(part + 2 + lane * CPL + dd), make_float2(A[g][dd], A[g][dd + 1]));
          if (lane == 0) __stcg(reinterpret_cast<float2*>(part), make_float2(Mg[g], Lg[g]));
        }
      }
#ifdef TDP_TC_PROF
      prof[15] += clock64() - tm1_;
#endif
      if (itc.n_splits > 1) {
        __syncwarp();
        int last = 0;
        if (lane == 0) {
          __threadfence();
          last = atomicAdd(&p.counters[itc.seq * p.Hkv + itc.kh], 1) == itc.n_splits - 1;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {   // merge every split's partial of the G heads, in split order
          __threadfence();
          const int ns = itc.n_splits;
          const float* part0 = p.part + ((int64_t)itc.seq * H + itc.kh * G) * p.max_splits * (HD + 2);
          // (m, l) of every (head, split) in one round trip, staged in shared memory
          for (int e = lane; e < G * ns; e += 32) {
            const int g = e / ns, s2 = e - g * ns;
            const float2 ml = __ldcg(reinterpret_cast<const float2*>(part0 + ((int64_t)g * p.max_splits + s2) * (HD + 2)));
            s_c[g][s2] = ml.x;
            s_l[g][s2] = ml.y;
          }
          __syncwarp();
          float Lh[G];
#pragma unroll
          for (int g = 0; g < G; ++g) {   // weights c = exp2(m - M), in split order (every lane the same)
            float M = -INFINITY;
            for (int s2 = 0; s2 < ns; ++s2) M = fmaxf(M, s_c[g][s2]);
            float L = 0.f;
            for (int s2 = 0; s2 < ns; ++s2) L += s_l[g][s2] * exp2f(s_c[g][s2] - M);
            Lh[g] = L;
            __syncwarp();
            for (int s2 = lane; s2 < ns; s2 += 32) s_c[g][s2] = exp2f(s_c[g][s2] - M);
            __syncwarp();
          }
          float acc[G][CPL];
#pragma unroll
          for (int g = 0; g < G; ++g)
#pragma unroll
            for (int dd = 0; dd < CPL; ++dd) acc[g][dd] = 0.f;
          for (int s2 = 0; s2 < ns; s2 += 2) {   // split order; 2 splits x G x CPL values in flight
            float v0[G][CPL], v1[G][CPL];
            const bool two = s2 + 1 < ns;
#pragma unroll
            for (int g = 0; g < G; ++g) {
              const float* ps = part0 + ((int64_t)g * p.max_splits + s2) * (HD + 2) + 2 + lane * CPL;
#pragma unroll
              for (int dd = 0; dd < CPL; dd += 2) {
                const float2 a0 = __ldcg(reinterpret_cast<const float2*>(ps + dd));
                const float2 a1 = two ? __ldcg(reinterpret_cast<const float2*>(ps + (HD + 2) + dd)) : make_float2(0.f, 0.f);
                v0[g][dd] = a0.x;
                v0[g][dd + 1] = a0.y;
                v1[g][dd] = a1.x;
                v1[g][dd + 1] = a1.y;
              }
            }
#pragma unroll
            for (int g = 0; g < G; ++g) {
              const float c0 = s_c[g][s2], c1 = two ? s_c[g][s2 + 1] : 0.f;
#pragma unroll
              for (int dd = 0; dd < CPL; ++dd) acc[g][dd] = acc[g][dd] + c0 * v0[g][dd] + c1 * v1[g][dd];
            }
          }
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const float inv = 1.f / Lh[g];
            float r[CPL];
#pragma unroll
            for (int dd = 0; dd < CPL; ++dd) r[dd] = acc[g][dd] * inv;
            st_bf16_vec<CPL>(p.o + ((int64_t)itc.seq * H + itc.kh * G + g) * HD + lane * CPL, r);
          }
          __syncwarp();
          if (lane == 0) p.counters[itc.seq * p.Hkv + itc.kh] = 0;
        }
      }
    }
  } else {             // ---------------------------------------------------- consumers
    const int g = lane >> 2, t4 = lane & 3;
    const int mi = lane >> 3, rr = lane & 7;
    const int k_row = rr + 8 * (mi & 1), k_ch = mi >> 1;    // K: A operand, row-major
    const int v_row = rr + 8 * (mi >> 1), v_ch = mi & 1;    // V^T: A operand via .trans
    int cw = 0;   // pages this warp has taken (its slots: warp, warp + 4, ...)
    for (int n = 0;; ++n) {
      const int q = n % Q, b = n & 1;
      TC_PW(5, tc_mbar_wait(&qready[q], (uint32_t)(n / Q) & 1u));
      const int idx = s_item[q];
      if (idx < 0) break;
      const Item it = s_desc[q];
      const bf16* sq = qbuf + q * G * HD;
      // Q^T as the B operand of S^T = K Q^T: b0 = Q[head g][16j + 2t4 ..], b1 = [.. + 8]
      uint32_t qb[KS][2];
#pragma unroll
      for (int j = 0; j < KS; ++j) {
        qb[j][0] = g < G ? *reinterpret_cast<const uint32_t*>(sq + g * HD + 16 * j + 2 * t4) : 0u;
        qb[j][1] = g < G ? *reinterpret_cast<const uint32_t*>(sq + g * HD + 16 * j + 8 + 2 * t4) : 0u;
      }
      float o[KS][4];
#pragma unroll
      for (int i = 0; i < KS; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
      float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;   // heads 2t4, 2t4+1
      for (int j = warp; j < it.npg; j += NWC, ++cw) {
        const int s = warp + NWC * (cw % RW);
        TC_PW(6, tc_mbar_wait(&full[s], (uint32_t)(cw / RW) & 1u));
        const uint32_t kt = smem_u32(ring + s * SLOT), vt = kt + PAGE;
        float sc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int jj = 0; jj < KS; ++jj) {
          uint32_t a[4];
          ldsm4(a, kt + page_off<NB>(k_row, 2 * jj + k_ch));
          hmma16816(sc, a, qb[jj][0], qb[jj][1]);
        }
        const int tb = (it.pg0 + j) << 4;
        const bool ok0 = tb + g < it.t_end, ok1 = tb + g + 8 < it.t_end;
        const float x0 = ok0 ? sc[0] * scale : -INFINITY, x1 = ok0 ? sc[1] * scale : -INFINITY;
        const float x2 = ok1 ? sc[2] * scale : -INFINITY, x3 = ok1 ? sc[3] * scale : -INFINITY;
        float mx0 = fmaxf(x0, x2), mx1 = fmaxf(x1, x3);
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
        }
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);   // finite: every page holds >= 1 valid token
        const float c0 = exp2f(m0 - mn0), c1 = exp2f(m1 - mn1);
        const float p0 = exp2f(x0 - mn0), p1 = exp2f(x1 - mn1), p2 = exp2f(x2 - mn0), p3 = exp2f(x3 - mn1);
        l0 = l0 * c0 + (p0 + p2);
        l1 = l1 * c1 + (p1 + p3);
        m0 = mn0;
        m1 = mn1;
        const uint32_t b0 = movm_t(pack_bf16x2(p0, p1)), b1 = movm_t(pack_bf16x2(p2, p3));
#pragma unroll
        for (int d = 0; d < KS; ++d) {
          o[d][0] *= c0;
          o[d][1] *= c1;
          o[d][2] *= c0;
          o[d][3] *= c1;
          uint32_t a[4];
          ldsm4_t(a, vt + page_off<NB>(v_row, 2 * d + v_ch));
          hmma16816(o[d], a, b0, b1);
        }
        tc_mbar_arrive(&empty[s]);   // this thread is done with the slot
      }
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, off);
        l1 += __shfl_xor_sync(0xffffffffu, l1, off);
      }
      if (n >= 2) TC_PW(7, tc_mbar_wait(&ofree[b], ((uint32_t)(n >> 1) & 1u) ^ 1u));
      float* so = obuf + b * (Lay::OBUF / 4);
      float* sm = so + NWC * G * OS;
      float* sl = sm + NWC * 8;
      if (g == 0) {
        if (2 * t4 < G) { sm[warp * 8 + 2 * t4] = m0; sl[warp * 8 + 2 * t4] = l0; }
        if (2 * t4 + 1 < G) { sm[warp * 8 + 2 * t4 + 1] = m1; sl[warp * 8 + 2 * t4 + 1] = l1; }
      }
#pragma unroll
      for (int d = 0; d < KS; ++d) {
        const int h0 = 2 * t4, h1 = 2 * t4 + 1, r0 = 16 * d + g;
        if (h0 < G) {
          so[(warp * G + h0) * OS + r0] = o[d][0];
          so[(warp * G + h0) * OS + r0 + 8] = o[d][2];
        }
        if (h1 < G) {
          so[(warp * G + h1) * OS + r0] = o[d][1];
          so[(warp * G + h1) * OS + r0 + 8] = o[d][3];
        }
      }
      tc_mbar_arrive(&oready[b]);
    }
  }
#ifdef TDP_TC_PROF
  if (lane == 0) {
    for (int k = 0; k < 16; ++k)
      if (k < 8 || k >= 12) atomicAdd(&g_tc_prof[k], (unsigned long long)prof[k]);
    // 8 + role: total cycles of the warp (consumers 8, producer 9, q-prep 10, merger 11)
    const int role = warp < NWC ? 8 : 9 + (warp - NWC);
    atomicAdd(&g_tc_prof[role], (unsigned long long)(clock64() - prof_t0));
  }
#endif
  __syncthreads();
  // every producer of the grid has fetched past the end before its CTA counts
  // itself done: the last CTA re-arms the work counters for the next launch
  if (threadIdx.x == 0 && atomicAdd(p.work + 1, 1) == (int)gridDim.x - 1) {
    p.work[0] = 0;
    p.work[1] = 0;
  }
}

#ifdef TDP_TC_PROF
void tc_prof_read(unsigned long long* out, bool reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_tc_prof, sizeof(g_tc_prof));
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(g_tc_prof, z, sizeof(z));
  }
}
#endif

bool make_kv_map(CUtensorMap* map, const bf16* pool, int64_t C, int Hkv, int hd, int n_layers) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  if (hd < 64 || hd % 64) return false;
  const int64_t rows = C * 2 * Hkv * kBlock;
  // (64 columns, hd/64 halves, page rows, layers): one box = a whole 16-token page
  cuuint64_t dims[4] = {64, (cuuint64_t)(hd / 64), (cuuint64_t)rows, (cuuint64_t)std::max(n_layers, 1)};
  cuuint64_t strides[3] = {128, (cuuint64_t)hd * 2, (cuuint64_t)(rows * hd * 2)};
  cuuint32_t box[4] = {64, (cuuint32_t)(hd / 64), (cuuint32_t)kBlock, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<bf16*>(pool), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int HD, int G>
static void launch_tc(const DecodeAttnParams& p, cudaStream_t st) {
  auto kern = decode_attn_tc_kernel<HD, G>;
  const int smem = TcLayout<HD, G>::bytes(p.n);
  static int attr = 0;
  static int occ_smem = -1, occ = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = smem;
  }
  if (smem != occ_smem) {   // persistent grid = the CTAs that are resident at once
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kTcThreads, smem);
    occ_smem = smem;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>(p.n_items, (int64_t)sms * std::max(occ, 1));
  launch_k(kern, dim3(grid), dim3(kTcThreads), smem, st, *p.kvmap, p);
}

static bool use_tc(const DecodeAttnParams& p) {
  const int G = p.H / p.Hkv;
  if (!p.kvmap || p.qkv_ws || G > 8 || (p.hd != 64 && p.hd != 128) || p.impl == 1) return false;
  return G >= 2 || p.impl == 2;
}

bool decode_attn_use_tc(int n, int H, int Hkv, int hd, const int* ctx) {
  if ((hd != 64 && hd != 128) || Hkv < 1 || H / Hkv > 8) return false;
  if (H > Hkv) return true;
#ifdef TDP_NO_MHA_TC
  return false;
#else
  if (n < kMhaTcMinN) return false;
#ifndef TDP_MHA_TC_V1
  if (n < kMhaTcMaxN) return true;
#endif
  int64_t sum = 0;
  for (int i = 0; i < n; ++i) sum += ctx[i];
  return sum >= (int64_t)kMhaTcMinMeanCtx * n;
#endif
}

template <int HD>
static void launch_decode_hd(const DecodeAttnParams& p, cudaStream_t st) {
  const int G = p.H / p.Hkv;
  if constexpr (HD >= 64) {
    if (use_tc(p)) {
      switch (G) {
        case 1: launch_tc<HD, 1>(p, st); return;
        case 2: launch_tc<HD, 2>(p, st); return;
        case 4: launch_tc<HD, 4>(p, st); return;
        case 8: launch_tc<HD, 8>(p, st); return;
        default: break;
      }
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
  int max_ctx = 1;
  for (int i = 0; i < p.n; ++i) max_ctx = std::max(max_ctx, ctx[i]);
  auto ctas_at = [&](int split) {
    int64_t c = 0;
    for (int i = 0; i < p.n; ++i) c += (ctx[i] + split - 1) / split;
    return c * p.Hkv;
  };
  int split = 512;
  if (use_tc(p)) {
    // persistent tensor-core kernel (2 CTAs per SM): the largest split of
    // 1024 .. 32 tokens that still gives >= 148 work items (one per SM; the
    // 2-per-SM grid then balances the rest dynamically), while the partials
    // fit the workspace and the merge weights (<= kTcMaxSplits splits per
    // sequence).  Longer splits amortise the per-item q load and merge
    // (profiles/r2/attn_sweep_gqa8_tc.txt).
    split = 1024;
    while ((max_ctx + split - 1) / split > kTcMaxSplits) split *= 2;
    while (split > kAttnMinSplitGQA && ctas_at(split) < 148) {
      const int ns = split / 2;
      if ((int64_t)p.n * ((max_ctx + ns - 1) / ns) > p.part_cap || (max_ctx + ns - 1) / ns > kTcMaxSplits) break;
      split = ns;
    }
  } else {
    // SIMT kernel: the largest of 512/256/128 context tokens that still
    // yields >= 8 CTAs per SM over the batch's actual context lengths (short
    // CTAs of similar size balance the wave tail; >= 128 tokens amortise a
    // CTA)
    while (split > kAttnMinSplit && ctas_at(split) < 8 * 148) split >>= 1;
    // Small batches: the grid is only Hkv x n x splits CTAs (GQA: few kv
    // heads).  While that is below one CTA per SM, halve the split (down to
    // 32 tokens) as long as a sequence keeps <= 8 splits (one merge round
    // trip) and the workspace holds the partials.  Measured on Llama-2-70B
    // heads (profiles/r1/attn_sweep_gqa8_small.txt): 1.6x at n <= 4 x 256
    // tokens (MHA, Llama-2-7B heads: 1.1-1.3x at n <= 2 x 256); more splits
    // than 8, or splitting a grid that already has >= 1 CTA per SM, was slower.
    if (split == kAttnMinSplit) {
      for (;;) {
        const int ns = split / 2;
        const int64_t nsplits = (max_ctx + ns - 1) / ns;
        if (ctas_at(split) >= 148 || ns < kAttnMinSplitGQA || nsplits > 8) break;
        if ((int64_t)p.n * nsplits > p.part_cap) break;
        split = ns;
      }
    }
  }
  p.split_tokens = split;
  p.max_splits = (max_ctx + split - 1) / split;
  p.n_items = ctas_at(split);
}

// Decode attention is a PDL dependent only for batches of <= kAttnPdlMaxN
// sequences (SIMT kernel).  Its first K / V loads go out before
// griddepcontrol.wait; that is safe because every K / V page it reads
// early was written by an earlier micro-batch, and consecutive micro-batches
// are separated by their metadata H2D copy (a non-kernel stream operation,
// which PDL never overlaps); the newest token is re-read after the wait.
// Larger batches wait for their predecessor in the ordinary way (measured
// faster, profiles/r1/pdl_ab.md).  Enforced here, not left to the caller.
void launch_decode_attn(const DecodeAttnParams& p, cudaStream_t st) {
  if (p.n <= 0) return;
  struct NoPdl {
    bool prev;
    explicit NoPdl(bool on) : prev(!pdl_enabled()) { pdl_suppress(on || prev); }
    ~NoPdl() { pdl_suppress(prev); }
  } no_pdl(p.n > kAttnPdlMaxN || use_tc(p));
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
// (sequence, head, 64-query tile from the sequence's end: longest causal
// ranges first); 4 warps x 16 query rows; 64-key tiles double-buffered with
// cp.async, the Q tile staged in K stage 1 (64 KB smem: 3 CTAs / SM); S = Q K^T
// and O += P V with P kept in registers (accumulator layout == A-fragment
// layout).  Prefill is < 1% of the
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

#ifndef TDP_PREFILL_MINB
#define TDP_PREFILL_MINB 3
#endif
template <int HD>
__global__ void __launch_bounds__(128, HD >= 128 ? TDP_PREFILL_MINB : 4) flash_prefill_kernel(PrefillAttnParams p) {
  constexpr int BQ = 64, BKV = 64, CH = HD / 8;
  constexpr int TILE = BQ * HD * 2;
  extern __shared__ __align__(128) uint8_t fsm[];
  uint8_t* sK = fsm;                 // 2 stages
  uint8_t* sV = fsm + 2 * TILE;      // 2 stages
  uint8_t* sQ = sK + TILE;           // aliases K stage 1: Q goes to registers before tile 1 is loaded
  pdl_trigger_tail(2);
  pdl_wait();
  // grid (sequence, head, query tile counted from the END of the sequence):
  // the tiles with the most causal key tiles of every (sequence, head) are in
  // the first blocks launched, the short ones fill the tail
  const int seq = blockIdx.x, h = blockIdx.y;
  const int L = p.seq_ctx[seq];                  // keys: positions 0 .. L-1
  const int qs = p.seq_qstart ? p.seq_qstart[seq] : 0;
  const int nq = L - qs;                         // queries: positions qs .. L-1
  const int n_qt = (nq + BQ - 1) / BQ;
  if ((int)blockIdx.z >= n_qt) return;
  const int qt = n_qt - 1 - (int)blockIdx.z;
  const int q0 = qt * BQ;                        // (query indices relative to qs)
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
    if (kt == 0) {   // Q and K/V tile 0 landed; Q to registers, then its buffer becomes stage 1
      cp_async_wait<0>();
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        ldsm_x4(qf[kk], smem_u32(sQ + fswz<HD>(warp * 16 + (lane & 15), kk * 2 + (lane >> 4)) * 16));
      __syncthreads();
      if (n_kt > 1) load_kv(1, BKV);
      cp_async_commit();
    } else {
      if (kt + 1 < n_kt) load_kv((kt + 1) & 1, (kt + 1) * BKV);
      cp_async_commit();
      cp_async_wait<1>();
      __syncthreads();
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
  constexpr int smem = 4 * 64 * HD * 2;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(flash_prefill_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid(p.n_seqs, p.H, (p.max_len + 63) / 64);
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
