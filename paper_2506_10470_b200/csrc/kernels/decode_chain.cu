// decode_chain.cu -- persistent decode-layer kernel for small decode
// micro-batches (T <= 128 tokens): one launch runs a whole sequence of a
// layer's weight GEMMs and the reductions between them, so the weight stream
// never stops at a kernel boundary.
//
// What it computes is exactly the per-stage decode forward of §8(a) rows
// a6-a9 (+ a2/a3 of the next layer): PAPER.md:243-245 (a stage = consecutive
// layers), the Llama block  x += Wo·attn;  x += Wd·(silu(Wg·n2(x)) ⊙ Wu·n2(x));
// next layer  q,k,v = RoPE(Wqkv·n1(x))  (oracle/forward.py holds the plain
// definition).  Only the schedule differs from the per-kernel path:
//
//   * one CTA per SM (grid = #SMs, all co-resident), warp-specialised:
//       w0  weight producer  -- cp.async.bulk of the tile-packed 16 KB weight
//           tiles of EVERY GEMM op of the program into a deep smem ring; it
//           never waits for a grid barrier, so the next GEMM's weights stream
//           while the current op's reductions run;
//       w1  TMEM owner + tcgen05.mma issuer (M = 128 weight rows, N = BN tokens);
//       w2-5 epilogue / reduction warps (TMEM lane quarter = warp % 4);
//       w6  activation producer -- TMA of the X tiles, issued only after the
//           grid barrier that publishes X;
//   * a GEMM op splits its U (128-row tile, 64-k block) units stream-K style
//     over G' = min(G, U) CTAs: CTA c owns the contiguous, non-empty unit
//     range [c·U/G', (c+1)·U/G'); each (CTA, tile) intersection is a
//     "segment" whose fp32 partial goes to the workspace slot (tile + c)
//     (unique: c is non-decreasing in tile order);
//   * a weight tile is reduced by its own segment CTAs once all of them have
//     stored their partials (an arrival counter per tile, double-buffered
//     across GEMM ops and re-armed one op ahead): each
//     takes a share of the tokens, sums the tile's segments in CTA order
//     (deterministic, and independent of T: batch-invariant) and applies the
//     op's epilogue right there: residual add (+ the hand-off store), SwiGLU,
//     or RoPE + paged K/V write -- no separate reduction pass;
//   * RMSNorm is split between producer and consumer: the residual reduction
//     writes bf16(x * g) and per-tile sums of squares; the consuming GEMM's
//     reduction scales its sums by 1/rms(x) (W·(x∘g)·inv = W·bf16(x·inv∘g) up
//     to where the bf16 rounding falls);
//   * ops are separated by grid barriers (a monotone 64-bit counter: barrier b
//     of a launch completes at base + (b+1)·G arrivals; the host advances base):
//     three per decoder layer (O | gate/up | down | QKV).
//
// Deadlock freedom: the grid never exceeds one CTA per SM, so every CTA
// becomes resident once the predecessor kernel drains; dependents are
// released (griddepcontrol.launch_dependents) only after the first barrier,
// i.e. once every CTA of this grid is resident.  A barrier that does not
// complete within 10 s traps (a launch error instead of a hung GPU).
#include <cuda.h>

#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace tdp {

namespace {
using namespace tc;

constexpr int kThreads = 224;   // 7 warps
constexpr int kEpiWarp0 = 2;    // epilogue warps 2..5
constexpr int kXWarp = 6;
constexpr int kMaxGemms = 6;    // GEMM ops per program
constexpr int kPfAhead = 24;    // weight tiles (16 KB) prefetched into L2 beyond the smem ring, per CTA
constexpr uint64_t kPfPaceNs = 350;   // one 16 KB prefetch per 350 ns per SM ~ 6.8 TB/s over 148 SMs

TDP_DEV bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(done)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return done != 0;
}
TDP_DEV void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

TDP_DEV uint64_t ld_acquire_u64(const unsigned long long* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
TDP_DEV void red_release_add_u64(unsigned long long* p, uint64_t v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
TDP_DEV uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
TDP_DEV void grid_wait(const unsigned long long* bar, uint64_t target) {
  if (ld_acquire_u64(bar) >= target) return;
  const uint64_t t0 = globaltimer();
  while (ld_acquire_u64(bar) < target) {
    if (globaltimer() - t0 > 10000000000ull) __trap();   // 10 s: never hang the GPU
  }
}

#ifdef TDP_CHAIN_TRACE
// measurement build only (TDP_NVCC_DEFINES=-DTDP_CHAIN_TRACE): globaltimer
// stamps of the last traced launch, [cta][op][k]: k = 0 op start (epilogue),
// 1 op end (epilogue), 2 last weight load issued, 3 last MMA committed,
// 4 X barrier passed (activation producer), 5 kernel entry, 6 segments drained,
// 7 first tile wait passed, 8 tile reductions done
constexpr int kTraceK = 9;
__device__ unsigned long long g_chain_trace[160 * kChainMaxOps * kTraceK];
#define CHAIN_STAMP(i, k) \
  if (P.trace_on) g_chain_trace[(cta * kChainMaxOps + (i)) * kTraceK + (k)] = globaltimer()
#else
#define CHAIN_STAMP(i, k)
#endif

struct Geo {   // a GEMM's unit geometry
  int KB;      // 64-wide k blocks
  int tiles;   // 128-row weight tiles
  int U;       // tiles * KB units
  int Gp;      // CTAs taking part: min(grid, U), so that every one owns >= 1 unit
};
TDP_DEV Geo geo_of(int N, int K, int G) {
  Geo g;
  g.KB = K / BK;
  g.tiles = (N + 127) >> 7;
  g.U = g.tiles * g.KB;
  g.Gp = min(G, g.U);
  return g;
}
// unit range [unit_lo(c), unit_lo(c+1)) of CTA c < Gp (empty for c >= Gp), and
// the CTA owning unit u.  U * Gp < 2^31 for every shape here (U <= 2^16).
TDP_DEV int unit_lo(const Geo& g, int c) { return c >= g.Gp ? g.U : c * g.U / g.Gp; }
TDP_DEV int cta_of(const Geo& g, int u) { return ((u + 1) * g.Gp - 1) / g.U; }

struct ChainSmem {
  float inv[128];        // 1/rms per token (reductions of GEMMs on normalised inputs)
  int pos[128], slot[128];   // QKV reductions: per-token position / KV slot
  float redss[4];        // prep: per-warp sums of squares
  int xcnt;              // activation tiles issued (activation producer -> weight producer)
};

TDP_DEV void red_release_add_s32(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
TDP_DEV void spin_until_ge(const int* p, int target) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  if (v >= target) return;
  const uint64_t t0 = globaltimer();
  do {
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    if (globaltimer() - t0 > 10000000000ull) __trap();   // 10 s: never hang the GPU
  } while (v < target);
}
TDP_DEV int atom_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Reduction of one weight tile's tokens t = share + k * nshare by one of its
// segment CTAs: warp w takes tokens k = w, w+4, ... (two at a time), lane l
// owns the 4 features f = tile*128 + 4l .. 4l+3; the tile's segments (CTAs
// c0..c1) are summed in CTA order with all loads of the two tokens in flight,
// then the op's epilogue:
//   kRedResid   x += sum (+ xpeer); if g: out = bf16(x * g), ssq[tile][t]
//   kRedSwiGLU  h[t][f/2] = bf16(silu(inv_t g_f) * inv_t u_f)  (f even: gate, f+1: up)
//   kRedQKV     epilogue_pair(inv_t * (v_f, v_f+1)): RoPE + q store + paged K/V write
// (the consumer side of the RMSNorm: out = W . bf16(x * g) * inv_t)
TDP_DEV void reduce_tile(const ChainOp& op, const ChainProgram& P, int tile, int c0, int c1, int share, int nshare,
                         int T, int e, ChainSmem& sm) {
  const int n = c1 - c0 + 1;
  const int w = e >> 5, ln = e & 31;
  const int f = tile * 128 + ln * 4;
  const bool fok = f < op.N;   // N % 4 == 0
  const int64_t stride = (int64_t)T * 128;
  const float* base = P.ws + (int64_t)(tile + c0) * stride + ln * 4;
  const bool resid = op.red == kRedResid;
  float4 g4 = make_float4(0.f, 0.f, 0.f, 0.f);
  if (resid && op.g && fok) {
    const uint2 gb = *reinterpret_cast<const uint2*>(op.g + f);
    const float2 ga = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gb.x));
    const float2 gc = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gb.y));
    g4 = make_float4(ga.x, ga.y, gc.x, gc.y);
  }
  EpiParams ep = op.ep;
  ep.pos = sm.pos;
  ep.slot = sm.slot;
  const int ntok = share < T ? (T - share + nshare - 1) / nshare : 0;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int k0 = w; k0 < ntok; k0 += 8) {
    int tt[2];
    tt[0] = share + k0 * nshare;
    tt[1] = k0 + 4 < ntok ? share + (k0 + 4) * nshare : -1;
    float4 acc[2] = {z, z}, xv[2] = {z, z};
#pragma unroll
    for (int qq = 0; qq < 2; ++qq)
      if (resid && fok && tt[qq] >= 0) xv[qq] = __ldcg(reinterpret_cast<const float4*>(op.x + (int64_t)tt[qq] * P.d + f));
    for (int c = 0; c < n; c += 8) {   // <= 8 segments: one L2 round trip
      float4 p[2][8];
#pragma unroll
      for (int qq = 0; qq < 2; ++qq)
#pragma unroll
        for (int r = 0; r < 8; ++r)
          p[qq][r] = (fok && tt[qq] >= 0 && c + r < n)
                         ? __ldcg(reinterpret_cast<const float4*>(base + (c + r) * stride + tt[qq] * 128))
                         : z;
#pragma unroll
      for (int qq = 0; qq < 2; ++qq)
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          acc[qq].x += p[qq][r].x;
          acc[qq].y += p[qq][r].y;
          acc[qq].z += p[qq][r].z;
          acc[qq].w += p[qq][r].w;
        }
    }
#pragma unroll
    for (int qq = 0; qq < 2; ++qq) {
      const int t = tt[qq];
      if (t < 0) break;   // warp-uniform
      if (resid) {
        const float4 v = make_float4(xv[qq].x + acc[qq].x, xv[qq].y + acc[qq].y, xv[qq].z + acc[qq].z,
                                     xv[qq].w + acc[qq].w);
        if (fok) {
          __stcg(reinterpret_cast<float4*>(op.x + (int64_t)t * P.d + f), v);
          if (op.xpeer) *reinterpret_cast<float4*>(op.xpeer + (int64_t)t * P.d + f) = v;
          if (op.g) {
            uint2 pk;
            pk.x = pack_bf16x2(v.x * g4.x, v.y * g4.y);
            pk.y = pack_bf16x2(v.z * g4.z, v.w * g4.w);
            *reinterpret_cast<uint2*>(op.out + (int64_t)t * P.d + f) = pk;
          }
        }
        if (op.g) {
          const float s2 = warp_sum(fok ? v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w : 0.f);
          if (ln == 0) __stcg(P.ssq + tile * kChainSsqStride + t, s2);
        }
      } else if (fok) {
        const float r = sm.inv[t];
        const float4 v = make_float4(acc[qq].x * r, acc[qq].y * r, acc[qq].z * r, acc[qq].w * r);
        if (op.red == kRedSwiGLU) {
          *reinterpret_cast<uint32_t*>(op.out + (int64_t)t * (op.N >> 1) + (f >> 1)) =
              pack_bf16x2(silu(v.x) * v.y, silu(v.z) * v.w);
        } else {
          epilogue_pair(ep, T, op.N, t, f, v.x, v.y);
          epilogue_pair(ep, T, op.N, t, f + 2, v.z, v.w);
        }
      }
    }
  }
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
decode_chain_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmO,
                    const __grid_constant__ CUtensorMap tmH, const __grid_constant__ ChainProgram P) {
  constexpr int X_BYTES = BN * BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + X_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN;   // two accumulators (segment i+1's MMAs overlap segment i's epilogue)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  ChainSmem& sm = *reinterpret_cast<ChainSmem*>(tmem_slot + 4);
  volatile int* xcnt = &sm.xcnt;   // X tiles issued so far (activation producer)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, cta = blockIdx.x;
  const int T = P.T;
  if (threadIdx.x == 0) CHAIN_STAMP(0, 5);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 2);    // weight producer + activation producer each arrive with their bytes
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    *xcnt = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------- weight producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      // this CTA's unit ranges of the program's GEMM ops, in program order
      int nw = 0, wlo[kMaxGemms], whi[kMaxGemms], wop[kMaxGemms];
      const bf16* ww[kMaxGemms];
      for (int i = 0; i < P.n_ops && nw < kMaxGemms; ++i) {
        if (P.op[i].kind != kChGemm) continue;
        const Geo g = geo_of(P.op[i].N, P.op[i].K, G);
        wlo[nw] = unit_lo(g, cta);
        whi[nw] = unit_lo(g, cta + 1);
        ww[nw] = P.op[i].w;
        wop[nw++] = i;
      }
      // L2 prefetch cursor over the same unit sequence: while the ring is full
      // AND its oldest stage still lacks its X tile (the MMAs wait for a
      // barrier-published X: HBM would idle), the next kPfAhead tiles beyond
      // the ring are pulled into L2, so HBM keeps streaming through the
      // program's reductions and barriers
      int pg = 0, pu = nw > 0 ? wlo[0] : 0, pidx = 0;
      auto pf_step = [&]() {
        ++pu;
        ++pidx;
        while (pg < nw && pu >= whi[pg]) {
          if (++pg < nw) pu = wlo[pg];
        }
      };
      while (pg < nw && pu >= whi[pg]) {
        if (++pg < nw) pu = wlo[pg];
      }
      int it = 0;
      uint64_t last_pf = 0;
      for (int j = 0; j < nw; ++j) {
        for (int u = wlo[j]; u < whi[j]; ++u, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) {
            const uint32_t par = (uint32_t)((it / STAGES) & 1) ^ 1u;
            while (!mbar_test(&empty[s], par)) {
              while (pg < nw && pidx < it + STAGES) pf_step();   // the ring loads those itself
              if (pg < nw && pidx < it + STAGES + kPfAhead && *xcnt <= it - STAGES) {
                const uint64_t now = globaltimer();
                if (now - last_pf >= kPfPaceNs) {   // paced at about this SM's share of HBM
                  bulk_prefetch_l2(ww[pg] + ((int64_t)pu << 13), A_BYTES);
                  pf_step();
                  last_pf = now;
                }
              }
            }
          }
          mbar_expect_tx(&full[s], A_BYTES);
          // tile-packed weights: unit u = (tile, kb) is the 16 KB tile at u << 13 elements
          bulk_load(smem + s * STAGE_BYTES, ww[j] + ((int64_t)u << 13), A_BYTES, &full[s], pol);
        }
        CHAIN_STAMP(wop[j], 2);
      }
    }
  } else if (warp == kXWarp) {
    // ------------------------------------------------------ activation producer
    if (lane == 0) {
      pdl_wait();   // the first op's X comes from the previous kernel
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmO)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmH)) : "memory");
      int it = 0;
      for (int i = 0; i < P.n_ops; ++i) {
        const ChainOp& op = P.op[i];
        if (op.kind != kChGemm) continue;
        if (i > 0) {
          grid_wait(P.bar, P.bar_base + (uint64_t)i * G);   // barrier i-1: X is published
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        CHAIN_STAMP(i, 4);
        const CUtensorMap* tm = op.xmap == 0 ? &tmA : op.xmap == 1 ? &tmO : &tmH;
        const Geo g = geo_of(op.N, op.K, G);
        const int hi = unit_lo(g, cta + 1);
        for (int u = unit_lo(g, cta); u < hi; ++u, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty[s], (uint32_t)((it / STAGES) & 1) ^ 1u);
          mbar_expect_tx(&full[s], X_BYTES);
          tma_load_2d(smem + s * STAGE_BYTES + A_BYTES, tm, (u % g.KB) * BK, 0, &full[s]);
          *xcnt = it + 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      // kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M=128, N=BN
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
      int it = 0, sg = 0;
      for (int i = 0; i < P.n_ops; ++i) {
        const ChainOp& op = P.op[i];
        if (op.kind != kChGemm) continue;
        const Geo g = geo_of(op.N, op.K, G);
        const int hi = unit_lo(g, cta + 1);
        for (int u = unit_lo(g, cta); u < hi; ++sg) {
          const int e = min(hi, (u / g.KB + 1) * g.KB);   // segment [u, e) inside one tile
          const int a = sg & 1;
          if (sg >= 2) mbar_wait(&tempty[a], (uint32_t)((sg >> 1) & 1) ^ 1u);
          tc_fence_after();
          const uint32_t acc = tmem + (uint32_t)(a * BN);
          for (int v = u; v < e; ++v, ++it) {
            const int s = it % STAGES;
            mbar_wait(&full[s], (uint32_t)(it / STAGES) & 1u);
            tc_fence_after();
            uint8_t* sa = smem + s * STAGE_BYTES;
            const uint64_t ad = smem_desc_sw128(sa);
            const uint64_t bd = smem_desc_sw128(sa + A_BYTES);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_f16(acc, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc, (v != u || k != 0) ? 1u : 0u);
            umma_commit(&empty[s]);
          }
          umma_commit(&tfull[a]);
          u = e;
        }
        CHAIN_STAMP(i, 3);
      }
    }
  } else {
    // ------------------------------------------- epilogue / reduction warps
    const int e = threadIdx.x - kEpiWarp0 * 32;   // 0..127: TMEM lane = weight row = feature of a tile
    const int q = warp & 3;                       // TMEM lane quarter
    pdl_wait();
    int sg = 0, ng = 0;
    for (int i = 0; i < P.n_ops; ++i) {
      const ChainOp& op = P.op[i];
      if (i > 0) {
        if (e == 0) grid_wait(P.bar, P.bar_base + (uint64_t)i * G);
        named_bar_sync(1, 128);
        if (i == 1) pdl_trigger();   // every CTA of this grid is resident: dependents may launch
      }
      if (e == 0) CHAIN_STAMP(i, 0);
      if (op.kind == kChPrep) {
        // out = bf16(x * g), ssq[t][tile] = sum over the tile's 128 features of x^2
        const int nt = P.d >> 7;
        for (int item = cta; item < T * nt; item += G) {
          const int t = item / nt, tile = item % nt, f = tile * 128 + e;
          const float v = __ldcg(op.x + (int64_t)t * P.d + f);
          op.out[(int64_t)t * P.d + f] = __float2bfloat16_rn(v * __bfloat162float(op.g[f]));
          const float s2 = warp_sum(v * v);
          if ((e & 31) == 0) sm.redss[e >> 5] = s2;
          named_bar_sync(1, 128);
          if (e == 0) __stcg(P.ssq + tile * kChainSsqStride + t, sm.redss[0] + sm.redss[1] + sm.redss[2] + sm.redss[3]);
          named_bar_sync(1, 128);
        }
      } else {
        // GEMM: drain each segment's accumulator into its workspace slot
        const Geo g = geo_of(op.N, op.K, G);
        // tile counters of this GEMM op; the other buffer (used by the previous
        // GEMM op, whose waits all precede the barrier just passed) is re-armed
        // for the next one
        int* cnt = P.cnt + ((P.cnt_parity + ng) & 1) * kChainMaxTiles;
        {
          int* other = P.cnt + ((P.cnt_parity + ng + 1) & 1) * kChainMaxTiles;
          const int per = (kChainMaxTiles + G - 1) / G;
          for (int k = cta * per + e; k < min(kChainMaxTiles, (cta + 1) * per); k += 128) other[k] = 0;
        }
        ++ng;
        if (op.red != kRedResid) {
          // 1/rms per token from the producing residual reduction's per-tile
          // sums of squares (ssq[tile][t]; computed while the GEMM streams)
          const int nt = P.d >> 7;
          for (int t = e; t < T; t += 128) {
            float s2 = 0.f;
#pragma unroll 8
            for (int k = 0; k < nt; ++k) s2 += __ldcg(P.ssq + k * kChainSsqStride + t);
            sm.inv[t] = rsqrtf(s2 / (float)P.d + P.eps);
            if (op.red == kRedQKV) {
              sm.pos[t] = op.ep.pos[t];
              sm.slot[t] = op.ep.slot[t];
            }
          }
        }
        const int hi = unit_lo(g, cta + 1);
        for (int u = unit_lo(g, cta); u < hi; ++sg) {
          const int tile = u / g.KB;
          const int en = min(hi, (tile + 1) * g.KB);
          const int a = sg & 1;
          mbar_wait(&tfull[a], (uint32_t)(sg >> 1) & 1u);
          tc_fence_after();
          float* dst = P.ws + (int64_t)(tile + cta) * T * 128 + q * 32 + lane;
#pragma unroll 1
          for (int c = 0; c < T; c += 32) {
            uint32_t r[32];
            tmem_ld32(tmem + (uint32_t)(a * BN) + ((uint32_t)(q * 32) << 16) + (uint32_t)c, r);
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (c + j < T) __stcg(dst + (int64_t)(c + j) * 128, __uint_as_float(r[j]));
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[a]);
          u = en;
        }
        // tile reductions, shared by each tile's segment CTAs: arrive on every
        // tile this CTA touched (its partials are stored), wait for the tile's
        // other segments, reduce this CTA's share of the tokens, depart (the
        // last to depart re-arms the tile's counters for the next GEMM op)
        const int lo = unit_lo(g, cta);
        if (e == 0) CHAIN_STAMP(i, 6);
        if (lo < hi) {
          const int tf = lo / g.KB, tl = (hi - 1) / g.KB;
          named_bar_sync(1, 128);   // the 4 warps' partial stores precede the arrivals (cumulative release)
          if (e == 0)
            for (int tile = tf; tile <= tl; ++tile) red_release_add_s32(cnt + tile, 1);
          for (int tile = tf; tile <= tl; ++tile) {
            const int c0 = cta_of(g, tile * g.KB), c1 = cta_of(g, (tile + 1) * g.KB - 1);
            const int ns = c1 - c0 + 1;
            if (e == 0 && ns > 1) spin_until_ge(cnt + tile, ns);
            if (e == 0 && tile == tf) CHAIN_STAMP(i, 7);
            named_bar_sync(1, 128);
            reduce_tile(op, P, tile, c0, c1, cta - c0, ns, T, e, sm);
          }
          if (e == 0) CHAIN_STAMP(i, 8);
        }
      }
      if (e == 0) CHAIN_STAMP(i, 1);
      if (i + 1 < P.n_ops) {
        // publish this op's results: barrier i
        asm volatile("fence.proxy.async.global;" ::: "memory");   // consumers read some of them by TMA
        named_bar_sync(1, 128);
        if (e == 0) red_release_add_u64(P.bar, 1);   // release: cumulative over the bar.sync above
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS) : "memory");
  }
}

template <int BN, int STAGES>
constexpr int chain_smem() {
  return STAGES * (A_BYTES + BN * BK * 2) + 1024 + 256 + (int)sizeof(ChainSmem);
}

template <int BN, int STAGES>
void launch_bn(const CUtensorMap* maps, const ChainProgram& p, int G, cudaStream_t st) {
  auto kern = decode_chain_kernel<BN, STAGES>;
  constexpr int sm = chain_smem<BN, STAGES>();
  static_assert(sm <= 227 * 1024, "smem");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    attr = true;
  }
  launch_k(kern, dim3(G), dim3(kThreads), sm, st, maps[0], maps[1], maps[2], p);
}
}  // namespace

int chain_barriers(const ChainProgram& p) { return p.n_ops > 0 ? p.n_ops - 1 : 0; }
int chain_gemms(const ChainProgram& p) {
  int n = 0;
  for (int i = 0; i < p.n_ops; ++i) n += p.op[i].kind == kChGemm;
  return n;
}

#ifdef TDP_CHAIN_TRACE
void chain_trace_read(unsigned long long* out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_chain_trace, sizeof(g_chain_trace));
}
#endif

void launch_decode_chain(const ChainProgram& p, const CUtensorMap* maps, int grid, cudaStream_t st) {
  if (p.T <= 0 || p.n_ops <= 0) return;
  if (p.T <= 32) launch_bn<32, 10>(maps, p, grid, st);
  else if (p.T <= 64) launch_bn<64, 8>(maps, p, grid, st);
  else launch_bn<128, 6>(maps, p, grid, st);
}

}  // namespace tdp
