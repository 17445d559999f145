// misc.cu -- weight init (F9 recipe), embedding gather, RMSNorm, argmax.
//
// Memory-bound helpers: vectorised 16-byte loads, one CTA per row, grid sized
// by the row count.  RMSNorm(x) = x / sqrt(mean(x^2) + eps) * g (Llama
// pre-norm) in fp32 from the fp32 residual.
#include <float.h>

#include <cstdlib>
#include <algorithm>
#include <cstring>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace tdp {

static thread_local int g_pdl_suppress = 0;
void pdl_suppress(bool on) { g_pdl_suppress = on ? 1 : 0; }

bool pdl_enabled() { return !g_pdl_suppress; }

static thread_local cudaError_t g_launch_err = cudaSuccess;
void note_launch_error(cudaError_t e) {
  if (e != cudaSuccess && g_launch_err == cudaSuccess) g_launch_err = e;
}
cudaError_t take_launch_error() {
  const cudaError_t e = g_launch_err;
  g_launch_err = cudaSuccess;
  return e;
}

// splitmix64 finaliser (counter-based; both sides implement it independently)
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void init_kernel(bf16* __restrict__ dst, InitSpec s, uint64_t seed) {
  const int64_t total = (int64_t)s.rows * s.cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(e / s.cols);
    const int c = (int)(e % s.cols);
    int tid = s.tid0, row = p;
    if (s.map == kMapQKV) {
      // physical rows: q heads, k heads, v heads; q/k rows interleave the
      // rotate-half pairs (i, i + hd/2) as (2i, 2i+1) so RoPE is an in-thread pair
      const int qrows = s.H * s.hd, krows = s.Hkv * s.hd;
      int base = 0;
      if (p < qrows) { tid = s.tid0; base = 0; }
      else if (p < qrows + krows) { tid = s.tid1; base = qrows; }
      else { tid = s.tid2; base = qrows + krows; }
      const int lp = p - base;
      if (tid == s.tid2) {
        row = lp;
      } else {
        const int h = lp / s.hd, j = lp % s.hd;
        const int i = (j & 1) ? (s.hd / 2 + j / 2) : (j / 2);
        row = h * s.hd + i;
      }
    } else if (s.map == kMapGateUp) {
      tid = (p & 1) ? s.tid1 : s.tid0;
      row = p >> 1;
    }
    const uint64_t idx = (uint64_t)row * (uint64_t)s.cols + (uint64_t)c;
    const uint64_t h = splitmix64(seed ^ ((uint64_t)tid << 40) ^ idx);
    const float u = __fmul_rn((float)(h >> 40), 5.9604644775390625e-08f);   // * 2^-24, exact
    const float v = __fsub_rn(__fmul_rn(2.0f, u), 1.0f);                      // exact
    float w;
    if (s.kind == kInitProj) w = __fmul_rn(s.scale, v);
    else if (s.kind == kInitNorm) w = __fadd_rn(1.0f, __fmul_rn(0.1f, v));
    else w = v;
    dst[s.packed ? pack_offset(p, c, s.cols) : e] = __float2bfloat16_rn(w);
  }
}

void launch_init(bf16* dst, const InitSpec& s, uint64_t seed, cudaStream_t st) {
  const int64_t total = (int64_t)s.rows * s.cols;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 64) blocks = 148 * 64;
  init_kernel<<<blocks, 256, 0, st>>>(dst, s, seed);
  note_launch_error(cudaGetLastError());
}

// ----------------------------------------------------------------- embedding
// x[t] = E[token] (fp32 residual); with g: also out[t] = bf16(RMSNorm(x[t]) * g),
// the first layer's input norm (one launch fewer per micro-batch)
__global__ void __launch_bounds__(128) embed_kernel(const int32_t* __restrict__ arena,
                                                    const int32_t* __restrict__ tok_idx, const bf16* __restrict__ E,
                                                    float* __restrict__ x, int d, const bf16* __restrict__ g,
                                                    bf16* __restrict__ out, float eps) {
  pdl_trigger_tail(8);
  pdl_wait();
  const int t = blockIdx.x;
  const int tok = arena[tok_idx[t]];
  const uint4* src = reinterpret_cast<const uint4*>(E + (int64_t)tok * d);
  float4* dst = reinterpret_cast<float4*>(x + (int64_t)t * d);
  float ss = 0.f;
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) {
    float f[8];
    bf16x8_to_f32(src[i], f);
    dst[2 * i] = make_float4(f[0], f[1], f[2], f[3]);
    dst[2 * i + 1] = make_float4(f[4], f[5], f[6], f[7]);
#pragma unroll
    for (int k = 0; k < 8; ++k) ss += f[k] * f[k];
  }
  if (!g) return;
  __shared__ float red[4];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  const float inv = rsqrtf((red[0] + red[1] + red[2] + red[3]) / (float)d + eps);
  const uint4* gs = reinterpret_cast<const uint4*>(g);
  uint4* o = reinterpret_cast<uint4*>(out + (int64_t)t * d);
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) {
    float f[8], gg[8];
    bf16x8_to_f32(src[i], f);
    bf16x8_to_f32(gs[i], gg);
    uint4 pk;
    pk.x = pack_bf16x2(f[0] * inv * gg[0], f[1] * inv * gg[1]);
    pk.y = pack_bf16x2(f[2] * inv * gg[2], f[3] * inv * gg[3]);
    pk.z = pack_bf16x2(f[4] * inv * gg[4], f[5] * inv * gg[5]);
    pk.w = pack_bf16x2(f[6] * inv * gg[6], f[7] * inv * gg[7]);
    o[i] = pk;
  }
}

void launch_embed(const int32_t* arena, const int32_t* tok_idx, const bf16* E, float* x, int T, int d,
                  cudaStream_t st, const bf16* g, bf16* out, float eps) {
  if (T <= 0) return;
  launch_k(embed_kernel, dim3(T), dim3(128), 0, st, arena, tok_idx, E, x, d, g, out, eps);
}

// ------------------------------------------------------------------- RMSNorm
template <int NT>
__global__ void __launch_bounds__(NT) rmsnorm_kernel(const float* __restrict__ x, const bf16* __restrict__ g,
                                                     bf16* __restrict__ out, const int32_t* __restrict__ rows,
                                                     int d, float eps) {
  pdl_trigger_tail(8);
  pdl_wait();
  const int i = blockIdx.x;
  const int r = rows ? rows[i] : i;
  const float4* xr = reinterpret_cast<const float4*>(x + (int64_t)r * d);
  __shared__ float red[NT / 32];
  float ss = 0.f;
  for (int j = threadIdx.x; j < d / 4; j += NT) {
    float4 v = xr[j];
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < NT / 32 ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / (float)d + eps);
  const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(g);
  uint2* o = reinterpret_cast<uint2*>(out + (int64_t)i * d);
  for (int j = threadIdx.x; j < d / 4; j += NT) {
    float4 v = xr[j];
    float2 ga = __bfloat1622float2(g2[2 * j]);
    float2 gb = __bfloat1622float2(g2[2 * j + 1]);
    uint2 pk;
    pk.x = pack_bf16x2(v.x * inv * ga.x, v.y * inv * ga.y);
    pk.y = pack_bf16x2(v.z * inv * gb.x, v.w * inv * gb.y);
    o[j] = pk;
  }
}

void launch_rmsnorm(const float* x, const bf16* g, bf16* out, const int32_t* rows, int n, int d, float eps,
                    cudaStream_t st) {
  if (n <= 0) return;
  if (n < 148 && d >= 4096)
    launch_k(rmsnorm_kernel<1024>, dim3(n), dim3(1024), 0, st, x, g, out, rows, d, eps);
  else
    launch_k(rmsnorm_kernel<256>, dim3(n), dim3(256), 0, st, x, g, out, rows, d, eps);
}

// ---------------------------------------------- split-K reduce + resid + norm
template <int NT>
__global__ void __launch_bounds__(NT) resid_norm_kernel(const float* __restrict__ ws, int splits, float* __restrict__ x,
                                                        const bf16* __restrict__ g, bf16* __restrict__ out, int T,
                                                        int d, float eps, float* __restrict__ xpeer) {
  pdl_trigger_tail(8);
  pdl_wait();
  const int t = blockIdx.x;
  float4* xr = reinterpret_cast<float4*>(x + (int64_t)t * d);
  float4* xp = xpeer ? reinterpret_cast<float4*>(xpeer + (int64_t)t * d) : nullptr;
  __shared__ float red[NT / 32];
  float ss = 0.f;
  for (int j = threadIdx.x; j < d / 4; j += NT) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < splits; ++s) {
      const float4 p = __ldcg(reinterpret_cast<const float4*>(ws + ((int64_t)s * T + t) * d) + j);
      acc.x += p.x;
      acc.y += p.y;
      acc.z += p.z;
      acc.w += p.w;
    }
    float4 v = xr[j];
    v.x += acc.x;
    v.y += acc.y;
    v.z += acc.z;
    v.w += acc.w;
    xr[j] = v;
    if (xp) xp[j] = v;   // stage hand-off: the same row stored into the next stage's receive slot
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  if (!g) return;
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < NT / 32 ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / (float)d + eps);
  const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(g);
  uint2* o = reinterpret_cast<uint2*>(out + (int64_t)t * d);
  for (int j = threadIdx.x; j < d / 4; j += NT) {
    const float4 v = xr[j];
    const float2 ga = __bfloat1622float2(g2[2 * j]);
    const float2 gb = __bfloat1622float2(g2[2 * j + 1]);
    uint2 pk;
    pk.x = pack_bf16x2(v.x * inv * ga.x, v.y * inv * ga.y);
    pk.y = pack_bf16x2(v.z * inv * gb.x, v.w * inv * gb.y);
    o[j] = pk;
  }
}

// Decode batches of <= kRnClusterMaxT tokens: a row is split over a cluster of
// RC CTAs (RC*128 threads); each reduces its slice of the split-K partials, and
// the row's sum of squares is all-reduced through distributed shared memory, so
// the whole GPU -- not T SMs -- streams the partials.
template <int RC>
__global__ void __launch_bounds__(128) resid_norm_cluster_kernel(const float* __restrict__ ws, int splits,
                                                                  float* __restrict__ x, const bf16* __restrict__ g,
                                                                  bf16* __restrict__ out, int T, int d, float eps,
                                                                  float* __restrict__ xpeer) {
  pdl_trigger_tail(8);
  pdl_wait();
  cg::cluster_group cl = cg::this_cluster();
  const int t = blockIdx.y;
  const int rank = (int)cl.block_rank();
  const int per = d / RC;                      // elements of this CTA's slice
  const int j0 = rank * per / 4;               // float4 index
  float4* xr = reinterpret_cast<float4*>(x + (int64_t)t * d);
  float4* xp = xpeer ? reinterpret_cast<float4*>(xpeer + (int64_t)t * d) : nullptr;
  __shared__ float red[4];
  __shared__ float part_ss[RC];   // every rank's partial sum of squares, written by that rank
  float ss = 0.f;
  for (int j = j0 + threadIdx.x; j < j0 + per / 4; j += 128) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < splits; ++s) {
      const float4 p = __ldcg(reinterpret_cast<const float4*>(ws + ((int64_t)s * T + t) * d) + j);
      acc.x += p.x;
      acc.y += p.y;
      acc.z += p.z;
      acc.w += p.w;
    }
    float4 v = xr[j];
    v.x += acc.x;
    v.y += acc.y;
    v.z += acc.z;
    v.w += acc.w;
    xr[j] = v;
    if (xp) xp[j] = v;
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  // broadcast this rank's partial into slot [rank] of every rank's array, then
  // one cluster barrier: afterwards each rank reads only its own shared memory,
  // so no second barrier has to keep the peers' memory alive
  if (threadIdx.x < RC) *cl.map_shared_rank(&part_ss[rank], threadIdx.x) = red[0] + red[1] + red[2] + red[3];
  cl.sync();
  if (!g) return;
  float tot = 0.f;
#pragma unroll
  for (int r = 0; r < RC; ++r) tot += part_ss[r];   // fixed order: deterministic
  const float inv = rsqrtf(tot / (float)d + eps);
  const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(g);
  uint2* o = reinterpret_cast<uint2*>(out + (int64_t)t * d);
  for (int j = j0 + threadIdx.x; j < j0 + per / 4; j += 128) {
    const float4 v = xr[j];
    const float2 ga = __bfloat1622float2(g2[2 * j]);
    const float2 gb = __bfloat1622float2(g2[2 * j + 1]);
    uint2 pk;
    pk.x = pack_bf16x2(v.x * inv * ga.x, v.y * inv * ga.y);
    pk.y = pack_bf16x2(v.z * inv * gb.x, v.w * inv * gb.y);
    o[j] = pk;
  }
}

#ifndef TDP_RN_CLUSTER
#define TDP_RN_CLUSTER 8
#endif
// CTAs per token row (small batches).  Per 8-layer decode step at b = 1 the
// reductions cost 156 / 107 / 75 / 77 us of marginal time with 2 / 4 / 8 / 16
// (profiles/r2/timeline/README.md)
constexpr int kRnCluster = TDP_RN_CLUSTER;
#ifndef TDP_RN_CLUSTER_MAXT
#define TDP_RN_CLUSTER_MAXT 512
#endif
// token rows up to which the cluster kernel is used (one CTA per row beyond):
// at 128 / 256 tokens it cuts the reductions' marginal time per 8-layer step
// 211 -> 143 / 167 -> 152 us and the step 3,257 -> 3,059 / 5,638 -> 5,199 us
// (profiles/r2/timeline/README.md)
constexpr int kRnClusterMaxT = TDP_RN_CLUSTER_MAXT;

void launch_resid_norm(const float* ws, int splits, float* x, const bf16* g, bf16* out, int T, int d, float eps,
                       cudaStream_t st, float* xpeer) {
  if (T <= 0) return;
  if (T <= kRnClusterMaxT && d % (kRnCluster * 4) == 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kRnCluster, T);
    cfg.blockDim = dim3(128);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kRnCluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    note_launch_error(cudaLaunchKernelEx(&cfg, resid_norm_cluster_kernel<kRnCluster>, ws, splits, x, g, out, T, d, eps, xpeer));
  } else {
    launch_k(resid_norm_kernel<256>, dim3(T), dim3(256), 0, st, ws, splits, x, g, out, T, d, eps, xpeer);
  }
}

// -------------------------------------------------------------------- argmax
__global__ void argmax_kernel(const float* __restrict__ logits, int V, int32_t* __restrict__ arena,
                              const int32_t* __restrict__ outpos) {
  pdl_trigger_tail(8);
  pdl_wait();
  const int i = blockIdx.x;
  const float* l = logits + (int64_t)i * V;
  float best = -FLT_MAX;
  int bi = 0x7fffffff;
  // 4 independent 16-byte loads in flight per thread; each thread visits its
  // indices in increasing order, so '>' keeps the lowest index among ties
  const int V4 = (V & 3) == 0 ? V >> 2 : 0;
  const float4* l4 = reinterpret_cast<const float4*>(l);
  int j = threadIdx.x;
  for (; j + 3 * (int)blockDim.x < V4; j += 4 * blockDim.x) {
    float4 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = l4[j + u * blockDim.x];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int b = (j + u * blockDim.x) * 4;
      if (a[u].x > best) { best = a[u].x; bi = b; }
      if (a[u].y > best) { best = a[u].y; bi = b + 1; }
      if (a[u].z > best) { best = a[u].z; bi = b + 2; }
      if (a[u].w > best) { best = a[u].w; bi = b + 3; }
    }
  }
  for (; j < V4; j += blockDim.x) {
    const float4 a = l4[j];
    const int b = j * 4;
    if (a.x > best) { best = a.x; bi = b; }
    if (a.y > best) { best = a.y; bi = b + 1; }
    if (a.z > best) { best = a.z; bi = b + 2; }
    if (a.w > best) { best = a.w; bi = b + 3; }
  }
  for (int k = V4 * 4 + threadIdx.x; k < V; k += blockDim.x) {
    const float v = l[k];
    if (v > best) { best = v; bi = k; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  __shared__ float sb[32];
  __shared__ int si[32];
  if ((threadIdx.x & 31) == 0) { sb[threadIdx.x >> 5] = best; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
    best = threadIdx.x < nw ? sb[threadIdx.x] : -FLT_MAX;
    bi = threadIdx.x < nw ? si[threadIdx.x] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (threadIdx.x == 0 && outpos[i] >= 0) arena[outpos[i]] = bi;   // -1: no token (PP+HB chunk)
  }
}

void launch_argmax(const float* logits, int n, int V, int32_t* arena, const int32_t* outpos, cudaStream_t st) {
  if (n <= 0) return;
  launch_k(argmax_kernel, dim3(n), dim3(256), 0, st, logits, V, arena, outpos);
}

// ----------------------------------------------- token return (multi-process)
// last stage: (arena position, token) pairs of one micro-batch -> NCCL to stage 0
__global__ void token_pairs_kernel(const int32_t* __restrict__ arena, const int32_t* __restrict__ outpos, int n,
                                   int32_t* __restrict__ pairs) {
  pdl_trigger_tail(8);
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int p = outpos[i];
    pairs[2 * i] = p;
    pairs[2 * i + 1] = p >= 0 ? arena[p] : 0;
  }
}
// stage 0: scatter received pairs into its token arena
__global__ void token_scatter_kernel(const int32_t* __restrict__ pairs, int n, int32_t* __restrict__ arena) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (pairs[2 * i] >= 0) arena[pairs[2 * i]] = pairs[2 * i + 1];
}

void launch_token_pairs(const int32_t* arena, const int32_t* outpos, int n, int32_t* pairs, cudaStream_t st) {
  if (n <= 0) return;
  launch_k(token_pairs_kernel, dim3((n + 255) / 256), dim3(256), 0, st, arena, outpos, n, pairs);
}
void launch_token_scatter(const int32_t* pairs, int n, int32_t* arena, cudaStream_t st) {
  if (n <= 0) return;
  token_scatter_kernel<<<(n + 255) / 256, 256, 0, st>>>(pairs, n, arena);
  note_launch_error(cudaGetLastError());
}


// ------------------------------------------------------- stage hand-off copy
// fp32 row block copy, 16-byte vectors; with a peer (CUDA IPC) destination the
// stores travel over NVLink straight into the next stage's receive slot.
__global__ void copy_f32_kernel(float4* __restrict__ dst, const float4* __restrict__ src, int64_t n4) {
  pdl_trigger_tail(8);
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __ldcg(src + i);
}
void launch_copy_f32(float* dst, const float* src, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  const int64_t n4 = n / 4;   // n = T * d, d % 64 == 0
  const int blocks = (int)std::min<int64_t>((n4 + 255) / 256, 148 * 8);
  launch_k(copy_f32_kernel, dim3(blocks), dim3(256), 0, st, reinterpret_cast<float4*>(dst),
           reinterpret_cast<const float4*>(src), n4);
}

}  // namespace tdp
