// gemm_tc.cu -- tcgen05 / TMEM / TMA GEMM for sm_100a (the dense weight GEMMs).
//
//   out[t][f] = sum_k X[t][k] * W[f][k]      X: activations [T, K], W: weights [Nf, K]
//
// Swap-AB: the weight tile is the MMA M operand (128 output features per CTA,
// TMEM lane = feature) and the token tile is the N operand (BN <= 256 tokens,
// TMEM column = token).  Decode batches (T <= 256) therefore need exactly one
// N tile and every weight byte is streamed from HBM once; prefill walks T in
// BN = 256 tiles.  Operands are staged by TMA (128B swizzle, K-major) into a
// STAGES-deep smem ring; one elected thread issues tcgen05.mma (kind::f16,
// bf16 in, fp32 accumulate in TMEM); 4 epilogue warps tcgen05.ld the
// accumulator and apply the fused epilogue (epilogue.cuh), where a feature pair
// (2i, 2i+1) sits in adjacent lanes (RoPE pair / gate-up pair via one shfl).
//
// Warp roles (192 threads): w0 TMA producer, w1 TMEM alloc + MMA issuer,
// w2..w5 epilogue (TMEM lane quarter = warp % 4).
//
// Split-K (decode only): partial fp32 tiles go to a workspace, reduced in
// split order (deterministic) by splitk_reduce_kernel, which applies the
// same fused epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"
#include "gemm_tc.h"
#include "tc_ptx.cuh"

namespace tdp {

namespace {
using namespace tc;

template <int BN, int STAGES>
__global__ void __launch_bounds__(192, BN <= 128 ? 2 : 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, int Nf, int T,
               int kb_per_split, int kb_total, EpiParams ep, float* __restrict__ ws, const bf16* __restrict__ wpk,
               int* __restrict__ counters) {
  constexpr int B_BYTES = BN * BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* accf = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);

  pdl_trigger_tail(BN <= 128 ? 2 : 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid: x = token tile (fastest, so CTAs sharing a weight tile run together
  // and the re-read hits L2), y = 128-row weight tile, z = K split
  const int m0 = blockIdx.y * 128;
  const int n0 = blockIdx.x * BN;
  const int kb0 = blockIdx.z * kb_per_split;
  const int nkb = min(kb_per_split, kb_total - kb0);

  if (warp == 0 && lane == 0) {
    if (!wpk) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accf, 1);
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
    if (lane == 0) {
      // weights do not depend on the previous kernel: stream the first stages
      // before waiting for it (PDL), then the activation tiles
      // packed weights: this CTA's 128 rows are one contiguous run of 16 KB tiles
      const bf16* wrow = wpk ? wpk + ((int64_t)blockIdx.y * kb_total << 13) : nullptr;
      const uint64_t pol = policy_evict_first();
      auto load_w = [&](uint8_t* dst, int kb, uint64_t* bar) {
        if (wpk) bulk_load(dst, wrow + ((int64_t)kb << 13), A_BYTES, bar, pol);
        else tma_load_2d(dst, &tmW, kb * BK, m0, bar);
      };
      const int pre = min(nkb, STAGES);
      for (int i = 0; i < pre; ++i) {
        uint8_t* sa = smem + i * STAGE_BYTES;
        mbar_expect_tx(&full[i], STAGE_BYTES);
        load_w(sa, kb0 + i, &full[i]);
      }
      pdl_wait();
      auto load_x = [&](uint8_t* dst, int kb, uint64_t* bar) { tma_load_2d(dst, &tmX, kb * BK, n0, bar); };
      for (int i = 0; i < pre; ++i) load_x(smem + i * STAGE_BYTES + A_BYTES, kb0 + i, &full[i]);
      for (int i = pre; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        uint8_t* sa = smem + s * STAGE_BYTES;
        mbar_expect_tx(&full[s], STAGE_BYTES);
        load_w(sa, kb0 + i, &full[s]);
        load_x(sa + A_BYTES, kb0 + i, &full[s]);
      }
    }
  } else if (warp == 1) {
    pdl_wait();
    if (lane == 0) {
      // kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M=128, N=BN
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        uint8_t* sa = smem + s * STAGE_BYTES;
        const uint64_t ad = smem_desc_sw128(sa);
        const uint64_t bd = smem_desc_sw128(sa + A_BYTES);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)   // advance 16 elements = 32 B inside the swizzle atom
          umma_f16(tmem, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc, (i | k) != 0);
        umma_commit(&empty[s]);
      }
      umma_commit(accf);
    }
  } else {
    // epilogue: warps 2..5 -> TMEM lane quarter (warp % 4)
    pdl_wait();
    mbar_wait(accf, 0);
    tc_fence_after();
    const int q = warp & 3;
    const int f = m0 + q * 32 + lane;            // this lane's output feature
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t r[32];
      tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c, r);
      if (ws) {
        // split-K partial: ws[split][t][f] (lanes = consecutive features: coalesced)
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int t = n0 + c + j;
          if (t < T && f < Nf) __stcg(ws + ((int64_t)blockIdx.z * T + t) * Nf + f, __uint_as_float(r[j]));
        }
      } else {
        epilogue_chunk(ep, T, Nf, f, n0 + c, r);
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

// ----------------------------------------------------------------------------
// Token-major tcgen05 GEMM for prefill micro-batches (persistent):
//   MMA M = 128 tokens (A = activation tile via TMA, 128B swizzle), N = 256
//   output features (B = two tile-packed 16 KB weight tiles via bulk copies),
//   K = 64 per stage.  TMEM lane = token, column = feature, so the epilogue
//   thread of a token holds 32 consecutive features per tcgen05.ld and writes
//   16-byte vectors (epilogue_row).  One CTA per SM walks the (token tile,
// feature tile) grid (token tile fastest, so concurrently running CTAs share a
// weight tile through L2); the two 256-column TMEM accumulators are double
// buffered so the epilogue of tile i overlaps the MMAs of tile i+1, and the
// smem ring runs continuously across tiles.
template <int STAGES, int BNF>
__global__ void __launch_bounds__(192, 1)
gemm_tnp_kernel(const __grid_constant__ CUtensorMap tmX, const bf16* __restrict__ wpk, int Nf, int T, int kb_total,
                EpiParams ep, int nsplit, int kps, float* __restrict__ ws) {
  static_assert(BNF == 128 || BNF == 256, "feature tile: one or two 128-row packed weight tiles");   // 256 in use
  constexpr int WT = BNF / 128;
  constexpr int X_BYTES = 128 * BK * 2;
  constexpr int W_BYTES = BNF * BK * 2;
  constexpr int STAGE_BYTES = X_BYTES + W_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;      // [2] accumulator ready
  uint64_t* tempty = tfull + 2;          // [2] accumulator drained (4 epilogue warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int MT = (T + 127) / 128;
  const int NT = (Nf + BNF - 1) / BNF;
  // work units: (token tile fastest, feature tile, K split); a split writes
  // its fp32 partial tile to ws [split][T][Nf] for a split-order reduction
  const int n_tiles = MT * NT * nsplit;
  const int wtiles = (Nf + 127) >> 7;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(2 * BNF)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int it = 0;   // global k-block counter (ring position)
      bool waited = false;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int m0 = (tile % MT) * 128, nt = (tile / MT) % NT, ks = tile / (MT * NT);
        const int wt0 = nt * WT;
        const int n_wt = min(WT, wtiles - wt0);
        const uint32_t stage_tx = X_BYTES + n_wt * (W_BYTES / WT);
        for (int kb = ks * kps; kb < min(kb_total, (ks + 1) * kps); ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
          if (it >= STAGES) mbar_wait(&empty[s], ph ^ 1u);
          uint8_t* sa = smem + s * STAGE_BYTES;
          mbar_expect_tx(&full[s], stage_tx);
          for (int h = 0; h < n_wt; ++h)
            bulk_load(sa + X_BYTES + h * (W_BYTES / WT), wpk + (((int64_t)(wt0 + h) * kb_total + kb) << 13),
                      W_BYTES / WT, &full[s], pol);
          if (!waited) {   // activations come from the previous kernel (PDL)
            pdl_wait();
            waited = true;
          }
          tma_load_2d(sa, &tmX, kb * BK, m0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    pdl_wait();
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BNF >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
      int it = 0, i = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++i) {
        const int a = i & 1;
        const uint32_t aph = (uint32_t)(i >> 1) & 1u;
        if (i >= 2) mbar_wait(&tempty[a], aph ^ 1u);
        tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)(a * BNF);
        const int ks = tile / (MT * NT), kb0 = ks * kps;
        for (int kb = kb0; kb < min(kb_total, kb0 + kps); ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (uint32_t)(it / STAGES) & 1u;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          uint8_t* sa = smem + s * STAGE_BYTES;
          const uint64_t ad = smem_desc_sw128(sa);
          const uint64_t bd = smem_desc_sw128(sa + X_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_f16(acc, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[a]);
      }
    }
  } else {
    pdl_wait();
    const int q = warp & 3;
    int i = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++i) {
      const int a = i & 1;
      const int m0 = (tile % MT) * 128, n0 = ((tile / MT) % NT) * BNF, ks = tile / (MT * NT);
      mbar_wait(&tfull[a], (uint32_t)(i >> 1) & 1u);
      tc_fence_after();
      const int t = m0 + q * 32 + lane;
      const bool tok = t < T;
      int pos = 0, slot = 0;
      if (tok && ep.mode == kEpiQKV && !ws) {
        pos = ep.pos[t];
        slot = ep.slot[t];
      }
#pragma unroll 1
      for (int c = 0; c < BNF; c += 32) {
        if (n0 + c >= Nf) break;
        uint32_t r[32];
        tmem_ld32(tmem + (uint32_t)(a * BNF) + ((uint32_t)(q * 32) << 16) + (uint32_t)c, r);
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if (!tok) continue;
        if (ws) {   // split partial (L2-resident until the split-order reduction reads it)
          float* wp = ws + ((int64_t)ks * T + t) * Nf + n0 + c;
          if (n0 + c + 32 <= Nf) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) __stcg(reinterpret_cast<float4*>(wp + j), make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
          } else {
            for (int j = 0; j < 32; ++j)
              if (n0 + c + j < Nf) __stcg(wp + j, v[j]);
          }
        } else {
          epilogue_row(ep, Nf, t, n0 + c, v, pos, slot);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * BNF) : "memory");
  }
}

// split-K reduction: sums the partials in split order (deterministic) and
// applies the fused epilogue; grid-stride over (token, feature pair)
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, int T, int Nf, EpiParams ep) {
  pdl_trigger();
  pdl_wait();
  const int64_t pairs = (int64_t)T * (Nf >> 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < pairs; i += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / (Nf >> 1));
    const int f = (int)(i % (Nf >> 1)) * 2;
    float v0 = 0.f, v1 = 0.f;
    for (int s = 0; s < splits; ++s) {
      const float2 p = __ldcg(reinterpret_cast<const float2*>(ws + ((int64_t)s * T + t) * Nf + f));
      v0 += p.x;
      v1 += p.y;
    }
    epilogue_pair(ep, T, Nf, t, f, v0, v1);
  }
}

template <int BN, int STAGES>
constexpr int smem_bytes() {
  return STAGES * (A_BYTES + BN * BK * 2) + 1024 + 256;   // + alignment + barriers
}

template <int BN, int STAGES>
void launch_bn(const TcOperand& W, const TcOperand& X, int T, const EpiParams& ep, int splits, float* ws,
               int* counters, bool defer, cudaStream_t st) {
  auto kern = gemm_tc_kernel<BN, STAGES>;
  static bool attr = false;
  constexpr int sm = smem_bytes<BN, STAGES>();
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    attr = true;
  }
  const int kb_total = W.K / BK;
  const int kps = (kb_total + splits - 1) / splits;
  const int nsplit = (kb_total + kps - 1) / kps;
  dim3 grid((T + BN - 1) / BN, (W.rows + 127) / 128, nsplit);
  launch_k(kern, grid, dim3(192), sm, st, W.map, X.map, W.rows, T, kps, kb_total, ep, nsplit > 1 ? ws : nullptr,
           W.packed ? W.base : nullptr, counters);
  if (nsplit > 1 && !defer) {
    const int64_t pairs = (int64_t)T * (W.rows / 2);
    const int blocks = (int)std::min<int64_t>((pairs + 255) / 256, 148 * 8);
    launch_k(splitk_reduce_kernel, dim3(blocks), dim3(256), 0, st, ws, nsplit, T, W.rows, ep);
  }
}
}  // namespace

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool make_tc_operand(TcOperand* op, const bf16* base, int rows, int K, int box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  op->base = base;
  op->rows = rows;
  op->K = K;
  op->box_rows = box_rows;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&op->map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<bf16*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

TcOperand packed_weight(const bf16* base, int rows, int K) {
  TcOperand op;
  op.base = base;
  op.rows = rows;
  op.K = K;
  op.box_rows = 128;
  op.packed = true;
  return op;
}

// decode: token tiles of <= 128 (2 CTAs per SM, weight tiles shared through L2);
// prefill: 256-token tiles
int tc_bn_for(int T, bool decode) {
  if (T <= 32) return 32;
  if (T <= 64) return 64;
  if (T <= 128 || decode) return 128;
  return 256;
}

int effective_splits(int K, int splits) {
  const int kb_total = K / BK;
  const int kps = (kb_total + splits - 1) / splits;
  return (kb_total + kps - 1) / kps;
}

int launch_gemm_tc(const TcOperand& W, const TcOperand* Xby_bn, int T, const EpiParams& ep, int splits, float* ws,
                   int* counters, bool decode, cudaStream_t st, bool defer_reduce, int bn) {
  if (T <= 0) return 1;
  if (!decode && W.packed && T > 128) {
    // prefill / 129+-token decode: token-major tiles (vectorised epilogue),
    // persistent.  (128-feature tiles for under-filled grids were measured
    // slower in context: twice the activation re-reads per FLOP,
    // profiles/r2/gemm_sweep_t128.txt)
    constexpr int STAGES = 4;
    constexpr int sm = STAGES * (128 * BK * 2 + 256 * BK * 2) + 1024 + 256;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(gemm_tnp_kernel<STAGES, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      attr = true;
    }
    const int kb_total = W.K / BK;
    const int kps = (kb_total + std::max(splits, 1) - 1) / std::max(splits, 1);
    const int nsplit = (kb_total + kps - 1) / kps;
    const int units = ((T + 127) / 128) * ((W.rows + 255) / 256) * nsplit;
    launch_k(gemm_tnp_kernel<STAGES, 256>, dim3(std::min(units, 148)), dim3(192), sm, st, Xby_bn[2].map, W.base,
             W.rows, T, kb_total, ep, nsplit, kps, nsplit > 1 ? ws : nullptr);
    if (nsplit > 1 && !defer_reduce) {
      const int64_t pairs = (int64_t)T * (W.rows / 2);
      const int blocks = (int)std::min<int64_t>((pairs + 255) / 256, 148 * 8);
      launch_k(splitk_reduce_kernel, dim3(blocks), dim3(256), 0, st, ws, nsplit, T, W.rows, ep);
    }
    return nsplit;
  }
  switch (bn > 0 ? bn : tc_bn_for(T, decode)) {
    // <= 110 KB of smem for BN <= 128 so that two CTAs share an SM
    case 32: launch_bn<32, 5>(W, Xby_bn[0], T, ep, splits, ws, counters, defer_reduce, st); break;
    case 64: launch_bn<64, 4>(W, Xby_bn[1], T, ep, splits, ws, counters, defer_reduce, st); break;
    case 128: launch_bn<128, 3>(W, Xby_bn[2], T, ep, splits, ws, counters, defer_reduce, st); break;
    default: launch_bn<256, 4>(W, Xby_bn[3], T, ep, splits, ws, counters, defer_reduce, st); break;
  }
  return effective_splits(W.K, splits);
}

}  // namespace tdp
