// gemm_tc.h -- host interface of the tcgen05/TMA GEMM (gemm_tc.cu).
#pragma once
#include <cuda.h>

#include "kernels.h"

namespace tdp {

// A K-major bf16 matrix [rows, K] with its TMA descriptor (box = 64 x box_rows,
// 128B swizzle).  Weights use box_rows = 128; activation buffers one operand
// per token-tile width BN in {32, 64, 128, 256}.
struct TcOperand {
  CUtensorMap map;
  const bf16* base = nullptr;
  int rows = 0, K = 0, box_rows = 0;
  bool packed = false;     // weights: tile-packed (kernels.h pack_offset), bulk-copied
};

bool make_tc_operand(TcOperand* op, const bf16* base, int rows, int K, int box_rows);
// A tile-packed weight operand [rows (padded to 128), K]: no tensor map needed.
TcOperand packed_weight(const bf16* base, int rows, int K);
int tc_bn_for(int T, bool decode);
// out = X[T, K] . W[Nf, K]^T with epilogue ep.  Xby_bn[i] = X described with
// box rows 32 << i.  splits > 1: split-K through workspace ws
// [tiles][splits][128][BN] fp32 and zero-initialised per-tile counters.
// Returns the split count actually used.  defer_reduce: leave the partials in
// ws [splits][T][N] for a fused consumer (launch_resid_norm) instead of
// launching the reduction + epilogue.  bn > 0: the swap-AB token tile (32 /
// 64 / 128 / 256) instead of tc_bn_for's (token tiles share each weight tile
// through L2).
int launch_gemm_tc(const TcOperand& W, const TcOperand* Xby_bn, int T, const EpiParams& ep, int splits, float* ws,
                   int* counters, bool decode, cudaStream_t st, bool defer_reduce = false, int bn = 0);

}  // namespace tdp
