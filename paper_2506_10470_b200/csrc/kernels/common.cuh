// common.cuh -- small device helpers shared by the sm_100a kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#define TDP_DEV __device__ __forceinline__

namespace tdp {

constexpr int kBlock = 16;   // KV page size in tokens

TDP_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
TDP_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

TDP_DEV void bf16x8_to_f32(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

TDP_DEV uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

TDP_DEV uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// streaming read that is not kept in L2 (evict-first cache policy `pol`)
TDP_DEV uint64_t l2_evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
TDP_DEV uint4 ld_nc_v4_ef(const void* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  return r;
}

TDP_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

TDP_DEV void cp_async16(void* smem, const void* gmem, bool pred) {
  const int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(sz));
}
TDP_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
TDP_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Programmatic dependent launch (PDL): every hot-path kernel triggers its
// dependents immediately and waits for its predecessors before touching their
// outputs, so a kernel's launch, prologue (barrier init, TMEM alloc, weight
// prefetch) overlaps the previous kernel's tail.
TDP_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
TDP_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
TDP_DEV uint32_t sm_count_upper() {
  uint32_t n;
  asm("mov.u32 %0, %%nsmid;" : "=r"(n));
  return n;
}
// Multi-wave grids: let the dependent grid launch only once this grid's last
// resident wave is running (`per_sm` = resident CTAs per SM).  Dependents
// launched earlier take SM slots (registers, smem) from this grid's remaining
// waves while they sit in griddepcontrol.wait -- measured 5-7 % slower decode
// steps at b >= 64 with an entry trigger (profiles/r1/step_ab.jsonl).  CTAs
// outside the window exit without triggering, which counts as a trigger.
TDP_DEV void pdl_trigger_tail(uint32_t per_sm) {
  const uint32_t nb = gridDim.x * gridDim.y * gridDim.z;
  const uint32_t id = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (id + per_sm * sm_count_upper() >= nb) pdl_trigger();
}

bool pdl_enabled();
// launches from this host thread go without the PDL attribute while on
void pdl_suppress(bool on);
// First kernel-launch failure on this host thread since the last take
// (cudaLaunchKernelEx's return code; the engine checks it per micro-batch).
void note_launch_error(cudaError_t e);
cudaError_t take_launch_error();

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  note_launch_error(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// launch_k with a thread-block cluster of (1, cy, 1)
template <typename... KArgs, typename... Args>
inline void launch_kc(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cy,
                      Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = cy;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  note_launch_error(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

}  // namespace tdp
