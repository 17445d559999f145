// test_entry.cu -- td_test_gemm: kernel-level unit-test entry point (testing only).
#include <cuda_runtime.h>

#include <vector>

#include "../../include/tdpipe.h"
#include "kernels/gemm_tc.h"
#include "kernels/kernels.h"

using namespace tdp;

extern "C" td_status td_test_gemm(int32_t device, const uint16_t* A, const uint16_t* W, int32_t T, int32_t N,
                                  int32_t K, int32_t impl, int32_t splits, float* out) {
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
    if (impl == 1) {
      launch_gemm(dA, dW, T, N, K, ep, s);
    } else {
      // impl 0: tile-packed weights (the engine's layout); impl 2: row-major W via TMA
      TcOperand w, x[4];
      bool ok = true;
      bf16* dP = nullptr;
      if (impl == 0) {
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
      cudaMalloc(&ws, (size_t)std::max(splits, 1) * (Tcap + 256) * Np * 4) || cudaMalloc(&cnt, 65536 * 4)) {
    st = TD_ENOMEM;
  } else {
    for (auto& w : Ws) cudaMemset(w, 0, (size_t)Np * K * 2);
    cudaMemset(dA, 0, (size_t)Tcap * K * 2);
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
      for (int i = 0; i < 3; ++i) launch_gemm_tc(w[i % copies], x, T, ep, splits, ws, cnt, decode != 0, s);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, s);
      for (int i = 0; i < iters; ++i) launch_gemm_tc(w[i % copies], x, T, ep, splits, ws, cnt, decode != 0, s);
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
