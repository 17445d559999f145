// test_entry.cu -- td_test_gemm: kernel-level unit-test entry point (testing only).
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "../../include/tdpipe.h"
#include "kernels/gemm_tc.h"
#include "kernels/kernels.h"

using namespace tdp;

// Device buffers of a decode-chain test program (testing only).
struct ChainBufs {
  float *ws = nullptr, *ssq = nullptr;
  int* cnt = nullptr;
  unsigned long long* bar = nullptr;
  int nsm = 0;
  bool alloc(int device, int max_tiles) {
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    if (cudaMalloc(&ws, (size_t)(max_tiles + nsm) * 128 * 128 * 4) || cudaMalloc(&ssq, 128 * kChainSsqStride * 4) ||
        cudaMalloc(&cnt, 1024 * 4) || cudaMalloc(&bar, 8))
      return false;
    cudaMemset(cnt, 0, 1024 * 4);
    cudaMemset(bar, 0, 8);
    return true;
  }
  void fill(ChainProgram& P, int T, int d) const {
    P.T = T;
    P.d = d;
    P.eps = 1e-5f;
    P.ws = ws;
    P.ssq = ssq;
    P.cnt = cnt;
    P.bar = bar;
    P.bar_base = 0;
  }
  ~ChainBufs() {
    cudaFree(ws);
    cudaFree(ssq);
    cudaFree(cnt);
    cudaFree(bar);
  }
};

static bf16* upload_packed(const uint16_t* W, int N, int K) {
  const int Np = (N + 127) / 128 * 128;
  std::vector<uint16_t> pk((size_t)Np * K, 0);
  for (int r = 0; r < N; ++r)
    for (int c = 0; c < K; ++c) pk[pack_offset(r, c, K)] = W[(size_t)r * K + c];
  bf16* d = nullptr;
  if (cudaMalloc(&d, pk.size() * 2) != cudaSuccess) return nullptr;
  cudaMemcpy(d, pk.data(), pk.size() * 2, cudaMemcpyHostToDevice);
  return d;
}

// The decode chain (decode_chain.cu) on one GEMM op with the residual tile
// reduction into a zeroed residual: out[T, N] = X[T, K] . W[N, K]^T
// (N % 128 == 0, T <= 128).  Testing only.
static td_status test_chain_gemm(int32_t device, const uint16_t* A, const uint16_t* W, int32_t T, int32_t N,
                                 int32_t K, float* out) {
  if (!A || !W || !out || T < 1 || T > 128 || N < 128 || N % 128 || K < 64 || K % 64) return TD_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return TD_ECUDA;
  ChainBufs B;
  bf16 *dA = nullptr, *dP = upload_packed(W, N, K);
  float* x = nullptr;
  td_status st = TD_OK;
  cudaStream_t s;
  cudaStreamCreate(&s);
  if (!dP || !B.alloc(device, N / 128) || cudaMalloc(&dA, (size_t)128 * K * 2) || cudaMalloc(&x, (size_t)T * N * 4)) {
    st = TD_ENOMEM;
  } else {
    cudaMemset(dA, 0, (size_t)128 * K * 2);
    cudaMemcpy(dA, A, (size_t)T * K * 2, cudaMemcpyHostToDevice);
    cudaMemset(x, 0, (size_t)T * N * 4);
    TcOperand xo;
    if (!make_tc_operand(&xo, dA, 128, K, T <= 32 ? 32 : T <= 64 ? 64 : 128)) {
      st = TD_ECUDA;
    } else {
      ChainProgram P{};
      P.op[0].kind = kChGemm;
      P.op[0].red = kRedResid;
      P.op[0].w = dP;
      P.op[0].N = N;
      P.op[0].K = K;
      P.op[0].xmap = 0;
      P.op[0].x = x;
      P.n_ops = 1;
      B.fill(P, T, N);
      const CUtensorMap maps[3] = {xo.map, xo.map, xo.map};
      launch_decode_chain(P, maps, B.nsm, s);
      if (cudaStreamSynchronize(s) != cudaSuccess || cudaGetLastError() != cudaSuccess) st = TD_ECUDA;
      if (take_launch_error() != cudaSuccess) st = TD_ECUDA;
      if (st == TD_OK) cudaMemcpy(out, x, (size_t)T * N * 4, cudaMemcpyDeviceToHost);
    }
  }
  cudaFree(dA);
  cudaFree(dP);
  cudaFree(x);
  cudaStreamDestroy(s);
  return st;
}

extern "C" td_status td_test_gemm(int32_t device, const uint16_t* A, const uint16_t* W, int32_t T, int32_t N,
                                  int32_t K, int32_t impl, int32_t splits, float* out) {
  if (impl == 5) return test_chain_gemm(device, A, W, T, N, K, out);
  if (!A || !W || !out || T < 1 || N < 2 || (N & 1) || K < 64 || K % 64) return TD_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return TD_ECUDA;
  bf16 *dA = nullptr, *dW = nullptr;
  float *dO = nullptr, *ws = nullptr;
  int* cnt = nullptr;
  const int Tcap = ((T + 255) / 256) * 256;
  td_status st = TD_OK;
  cudaStream_t s;
  cudaStreamCreate(&s);
  if (cudaMalloc(&dA, (size_t)Tcap * K * 2) || cudaMalloc(&dW, (size_t)N * K * 2) ||
      cudaMalloc(&dO, (size_t)T * N * 4) ||
      cudaMalloc(&ws, (size_t)std::max(splits, 1) * (Tcap + 256) * ((N + 127) / 128 * 128) * 4) ||
      cudaMalloc(&cnt, 65536 * sizeof(int))) {
    st = TD_ENOMEM;
  } else {
    cudaMemset(dA, 0, (size_t)Tcap * K * 2);
    cudaMemset(cnt, 0, 65536 * sizeof(int));
    cudaMemcpy(dA, A, (size_t)T * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dW, W, (size_t)N * K * 2, cudaMemcpyHostToDevice);
    EpiParams ep{};
    ep.mode = kEpiF32;
    ep.out_f32 = dO;
    ep.ldo = N;
    if (impl != 0 && impl != 2 && impl != 4) {
      st = TD_EINVAL;
    } else {
      // impl 0: tile-packed weights (the engine's layout); impl 2: row-major W via TMA
      TcOperand w, x[4];
      bool ok = true;
      bf16* dP = nullptr;
      if (impl == 0 || impl == 4) {
        const int Np = (N + 127) / 128 * 128;
        std::vector<uint16_t> pk((size_t)Np * K, 0);
        for (int r = 0; r < N; ++r)
          for (int c = 0; c < K; ++c) pk[pack_offset(r, c, K)] = W[(size_t)r * K + c];
        ok = cudaMalloc(&dP, pk.size() * 2) == cudaSuccess;
        if (ok) cudaMemcpy(dP, pk.data(), pk.size() * 2, cudaMemcpyHostToDevice);
        w = packed_weight(dP, N, K);
      } else {
        ok = make_tc_operand(&w, dW, N, K, 128);
      }
      for (int i = 0; i < 4; ++i) ok = ok && make_tc_operand(&x[i], dA, Tcap, K, 32 << i);
      if (!ok) st = TD_ECUDA;
      else if (impl == 4) launch_gemm_tc(w, x, T, ep, splits, ws, cnt, /*decode=*/false, s);   // token-major (+ split-K)
      else launch_gemm_tc(w, x, T, ep, splits, ws, cnt, splits > 1, s);
      cudaStreamSynchronize(s);
      cudaFree(dP);
    }
    if (cudaStreamSynchronize(s) != cudaSuccess || cudaGetLastError() != cudaSuccess) st = TD_ECUDA;
    if (st == TD_OK) cudaMemcpy(out, dO, (size_t)T * N * 4, cudaMemcpyDeviceToHost);
  }
  cudaFree(dA);
  cudaFree(dW);
  cudaFree(dO);
  cudaFree(ws);
  cudaFree(cnt);
  cudaStreamDestroy(s);
  return st;
}

// Benchmark operands: seeded uniform [-1, 1] bf16 (the weight-init hash), not
// zeros -- an all-zero KV pool sends every attention output 0 / l down the
// division slow path and zero operands draw less power than real data.
static void fill_uniform(bf16* dst, int64_t elems, uint64_t seed, cudaStream_t st) {
  const int cols = 64;
  InitSpec sp{};
  sp.map = kMapIdentity;
  sp.kind = kInitEmbed;
  sp.rows = (int)(elems / cols);
  sp.cols = cols;
  sp.tid0 = (int)(seed & 0xffff);
  if (sp.rows > 0) launch_init(dst, sp, seed, st);
}

extern "C" td_status td_bench_gemm(int32_t device, int32_t T, int32_t N, int32_t K, int32_t splits, int32_t decode,
                                   int32_t iters, int32_t copies, float* us_per_call) {
  if (T < 1 || N < 2 || (N & 1) || K < 64 || K % 64 || iters < 1 || copies < 1 || !us_per_call) return TD_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return TD_ECUDA;
  const int Np = (N + 127) / 128 * 128;
  const int Tcap = ((T + 255) / 256) * 256;
  std::vector<bf16*> Ws(copies, nullptr);
  bf16* dA = nullptr;
  float *dO = nullptr, *ws = nullptr;
  int* cnt = nullptr;
  cudaStream_t s;
  cudaStreamCreate(&s);
  td_status st = TD_OK;
  for (auto& w : Ws)
    if (cudaMalloc(&w, (size_t)Np * K * 2) != cudaSuccess) st = TD_ENOMEM;
  if (st || cudaMalloc(&dA, (size_t)Tcap * K * 2) || cudaMalloc(&dO, (size_t)T * N * 4) ||
      cudaMalloc(&ws, (size_t)std::max(splits, 1) * (Tcap + 256) * Np * 4) ||
      cudaMalloc(&cnt, 65536 * 4)) {
    st = TD_ENOMEM;
  } else {
    for (size_t i = 0; i < Ws.size(); ++i) fill_uniform(Ws[i], (int64_t)Np * K, 11 + i, s);
    fill_uniform(dA, (int64_t)Tcap * K, 7, s);
    cudaMemset(cnt, 0, 65536 * 4);
    EpiParams ep{};
    ep.mode = kEpiF32;
    ep.out_f32 = dO;
    ep.ldo = N;
    TcOperand x[4];
    bool ok = true;
    for (int i = 0; i < 4; ++i) ok = ok && make_tc_operand(&x[i], dA, Tcap, K, 32 << i);
    std::vector<TcOperand> w(copies);
    for (int i = 0; i < copies; ++i) w[i] = packed_weight(Ws[i], N, K);
    if (!ok) {
      st = TD_ECUDA;
    } else {
      auto call = [&](int i) {
        // 1: swap-AB (3: with 64-token tiles, 4: 32-token tiles); 2: token-major (+ split-K)
        launch_gemm_tc(w[i % copies], x, T, ep, splits, ws, cnt, decode == 1 || decode >= 3, s, false,
                       decode == 3 ? 64 : decode == 4 ? 32 : 0);
      };
      for (int i = 0; i < 3; ++i) call(i);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, s);
      for (int i = 0; i < iters; ++i) call(i);
      cudaEventRecord(b, s);
      if (cudaEventSynchronize(b) != cudaSuccess || cudaGetLastError() != cudaSuccess) st = TD_ECUDA;
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      *us_per_call = ms * 1000.f / iters;
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
  }
  for (auto& wp : Ws) cudaFree(wp);
  cudaFree(dA);
  cudaFree(dO);
  cudaFree(ws);
  cudaFree(cnt);
  cudaStreamDestroy(s);
  return st;
}

// Decode-attention timing sweep: n sequences with context lengths ctx[] (host),
// pages scattered through the pool the way the block allocator hands them out;
// iterations rotate over `copies` disjoint page sets so the K/V stream from HBM.
extern "C" td_status td_bench_attn(int32_t device, int32_t n, const int32_t* ctx, int32_t H, int32_t Hkv, int32_t hd,
                                   int32_t iters, int32_t split, int32_t impl, float* us_per_call) {
  if (split != 0 && (split < kAttnMinSplitGQA || split % 16)) return TD_EINVAL;
  if (n < 1 || !ctx || H < 1 || Hkv < 1 || H % Hkv || iters < 1 || !us_per_call) return TD_EINVAL;
  if (hd != 16 && hd != 32 && hd != 64 && hd != 128) return TD_EINVAL;
  const int G = H / Hkv;
  if (G != 1 && G != 2 && G != 4 && G != 8) return TD_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return TD_ECUDA;
  int maxblk = 1, max_ctx = 1;
  int64_t nblk = 0;
  for (int i = 0; i < n; ++i) {
    if (ctx[i] < 1) return TD_EINVAL;
    maxblk = std::max(maxblk, (ctx[i] + 15) / 16);
    max_ctx = std::max(max_ctx, ctx[i]);
    nblk += (ctx[i] + 15) / 16;
  }
  const int64_t blk_bytes = 2LL * Hkv * 16 * hd * 2;
  const int copies = (int)std::min<int64_t>(64, std::max<int64_t>(1, (400LL << 20) / (nblk * blk_bytes)));
  const int64_t pool = nblk * copies;
  // block tables: a fixed pseudo-random permutation of the pool
  std::vector<int32_t> perm(pool);
  for (int64_t i = 0; i < pool; ++i) perm[i] = (int32_t)i;
  uint64_t x = 0x9E3779B97F4A7C15ull;
  for (int64_t i = pool - 1; i > 0; --i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    std::swap(perm[i], perm[x % (uint64_t)(i + 1)]);
  }
  std::vector<int32_t> bt((size_t)copies * n * maxblk, 0);
  int64_t k = 0;
  for (int c = 0; c < copies; ++c)
    for (int i = 0; i < n; ++i)
      for (int b = 0; b < (ctx[i] + 15) / 16; ++b) bt[((size_t)c * n + i) * maxblk + b] = perm[k++];
  const int cap = (max_ctx + kAttnMinSplitGQA - 1) / kAttnMinSplitGQA;   // any launch plan fits
  bf16 *kv = nullptr, *q = nullptr, *o = nullptr;
  float* part = nullptr;
  int32_t *dctx = nullptr, *dbt = nullptr, *dord = nullptr;
  int* cnt = nullptr;
  td_status st = TD_OK;
  cudaStream_t s;
  cudaStreamCreate(&s);
  if (cudaMalloc(&kv, pool * blk_bytes) || cudaMalloc(&q, (size_t)n * H * hd * 2) ||
      cudaMalloc(&o, (size_t)n * H * hd * 2) || cudaMalloc(&part, (size_t)n * H * cap * (hd + 2) * 4) ||
      cudaMalloc(&dctx, n * 4) || cudaMalloc(&dbt, bt.size() * 4) || cudaMalloc(&dord, n * 4) ||
      cudaMalloc(&cnt, ((size_t)n * Hkv + 2) * 4)) {
    st = TD_ENOMEM;
  } else {
    fill_uniform(kv, (int64_t)(pool * blk_bytes / 2), 5, s);
    fill_uniform(q, (int64_t)n * H * hd, 6, s);
    cudaMemset(cnt, 0, ((size_t)n * Hkv + 2) * 4);
    cudaMemcpy(dctx, ctx, n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dbt, bt.data(), bt.size() * 4, cudaMemcpyHostToDevice);
    std::vector<int32_t> ord(n);   // longest context first, as the engine's metadata
    for (int i = 0; i < n; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return ctx[a] > ctx[b]; });
    cudaMemcpy(dord, ord.data(), n * 4, cudaMemcpyHostToDevice);
    DecodeAttnParams p{q, kv, dctx, dbt, maxblk, o, part, 0, n, H, Hkv, hd, 0, cnt};
    p.part_cap = (int64_t)n * cap;
    p.work = cnt + (size_t)n * Hkv;
    p.order = dord;
    CUtensorMap kvmap;
    if (hd >= 64 && make_kv_map(&kvmap, kv, pool, Hkv, hd, 1)) p.kvmap = &kvmap;
    p.impl = impl;
    plan_decode_attn(p, ctx);
    if (split) {
      p.split_tokens = split;
      p.max_splits = (max_ctx + split - 1) / split;
      p.n_items = 0;
      for (int i = 0; i < n; ++i) p.n_items += (int64_t)((ctx[i] + split - 1) / split) * Hkv;
    }
    auto run = [&](int i) {
      DecodeAttnParams pi = p;
      pi.bt = dbt + (size_t)(i % copies) * n * maxblk;
      launch_decode_attn(pi, s);
    };
    for (int i = 0; i < 3; ++i) run(i);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    for (int i = 0; i < iters; ++i) run(i);
    cudaEventRecord(b, s);
    if (cudaEventSynchronize(b) != cudaSuccess || cudaGetLastError() != cudaSuccess) st = TD_ECUDA;
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    *us_per_call = ms * 1000.f / iters;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  cudaFree(kv); cudaFree(q); cudaFree(o); cudaFree(part);
  cudaFree(dctx); cudaFree(dbt); cudaFree(dord); cudaFree(cnt);
  cudaStreamDestroy(s);
  return st;
}

// The decode chain on an MLP block (testing only), with its split RMSNorm:
//   a = bf16(x0 * g);  r_t = 1/rms(x0_t);
//   h = bf16(silu(r_t Wgu[2j] . a) * (r_t Wgu[2j+1] . a));  x = x0 + Wd . h
// ops: prep | gate/up GEMM (SwiGLU reduction) | down GEMM (residual reduction).
extern "C" td_status td_test_chain_mlp(int32_t device, const float* x0, const uint16_t* g, const uint16_t* Wgu,
                                       const uint16_t* Wd, int32_t T, int32_t d, int32_t F, float eps, uint16_t* a_out,
                                       uint16_t* h_out, float* x_out) {
  if (!x0 || !g || !Wgu || !Wd || !a_out || !h_out || !x_out || T < 1 || T > 128 || d < 128 || d % 128 || F < 64 ||
      F % 64)
    return TD_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return TD_ECUDA;
  ChainBufs B;
  bf16 *dgu = upload_packed(Wgu, 2 * F, d), *dd = upload_packed(Wd, d, F);
  bf16 *da = nullptr, *dh = nullptr, *dg = nullptr;
  float* x = nullptr;
  td_status st = TD_OK;
  cudaStream_t s;
  cudaStreamCreate(&s);
  if (!dgu || !dd || !B.alloc(device, (2 * F + 127) / 128) || cudaMalloc(&da, (size_t)128 * d * 2) ||
      cudaMalloc(&dh, (size_t)128 * F * 2) || cudaMalloc(&dg, (size_t)d * 2) || cudaMalloc(&x, (size_t)T * d * 4)) {
    st = TD_ENOMEM;
  } else {
    cudaMemset(da, 0, (size_t)128 * d * 2);
    cudaMemset(dh, 0, (size_t)128 * F * 2);
    cudaMemcpy(dg, g, (size_t)d * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(x, x0, (size_t)T * d * 4, cudaMemcpyHostToDevice);
    const int box = T <= 32 ? 32 : T <= 64 ? 64 : 128;
    TcOperand xa, xh;
    if (!make_tc_operand(&xa, da, 128, d, box) || !make_tc_operand(&xh, dh, 128, F, box)) {
      st = TD_ECUDA;
    } else {
      ChainProgram P{};
      int n = 0;
      P.op[n].kind = kChPrep;
      P.op[n].x = x;
      P.op[n].g = dg;
      P.op[n++].out = da;
      P.op[n].kind = kChGemm;
      P.op[n].red = kRedSwiGLU;
      P.op[n].w = dgu;
      P.op[n].N = 2 * F;
      P.op[n].K = d;
      P.op[n].xmap = 0;
      P.op[n++].out = dh;
      P.op[n].kind = kChGemm;
      P.op[n].red = kRedResid;
      P.op[n].w = dd;
      P.op[n].N = d;
      P.op[n].K = F;
      P.op[n].xmap = 2;
      P.op[n++].x = x;
      P.n_ops = n;
      B.fill(P, T, d);
      P.eps = eps;
      const CUtensorMap maps[3] = {xa.map, xa.map, xh.map};
      launch_decode_chain(P, maps, B.nsm, s);
      if (cudaStreamSynchronize(s) != cudaSuccess || cudaGetLastError() != cudaSuccess) st = TD_ECUDA;
      if (take_launch_error() != cudaSuccess) st = TD_ECUDA;
      if (st == TD_OK) {
        cudaMemcpy(a_out, da, (size_t)T * d * 2, cudaMemcpyDeviceToHost);
        cudaMemcpy(h_out, dh, (size_t)T * F * 2, cudaMemcpyDeviceToHost);
        cudaMemcpy(x_out, x, (size_t)T * d * 4, cudaMemcpyDeviceToHost);
      }
    }
  }
  cudaFree(da);
  cudaFree(dh);
  cudaFree(dg);
  cudaFree(dgu);
  cudaFree(dd);
  cudaFree(x);
  cudaStreamDestroy(s);
  return st;
}

#ifdef TDP_CHAIN_TRACE
namespace tdp { void chain_trace_read(unsigned long long* out); }
// measurement builds only: the decode chain's trace buffer (see decode_chain.cu)
extern "C" void td_chain_trace(unsigned long long* out) { tdp::chain_trace_read(out); }
#endif

#ifdef TDP_TC_PROF
namespace tdp { void tc_prof_read(unsigned long long* out, bool reset); }
// measurement builds only: the tensor-core decode attention's per-wait-site cycle sums
extern "C" void td_tc_prof(unsigned long long* out, int32_t reset) { tdp::tc_prof_read(out, reset != 0); }
#endif
