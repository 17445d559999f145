// kernels.h -- host-side launchers of the sm_100a kernels (all async on `st`).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace tdp {

// launches from this host thread go without the PDL attribute while on (misc.cu)
void pdl_suppress(bool on);
// first kernel-launch failure on this host thread since the last call (misc.cu)
cudaError_t take_launch_error();

typedef __nv_bfloat16 bf16;

// ---- weight init (F9 counter-based recipe), physical layouts -------------
enum InitMap { kMapIdentity = 0, kMapQKV = 1, kMapGateUp = 2 };
enum InitKind { kInitProj = 0, kInitNorm = 1, kInitEmbed = 2 };
struct InitSpec {
  int map;            // InitMap
  int kind;           // InitKind
  int rows, cols;     // physical [rows, cols]
  int tid0, tid1, tid2;   // tensor ids (QKV: q,k,v; gate/up: g,u)
  int H, Hkv, hd;     // for kMapQKV
  float scale;        // sqrt_f32(3/fan_in) for projections
  int packed;         // 1: store in the UMMA tile-packed layout (pack_offset)
};

// Tile-packed weight layout consumed by the tcgen05 GEMM: 128-row x 64-col
// tiles (16 KB), k-tile fastest, each tile stored exactly as the 128B-swizzled
// K-major smem image (row r, 16-byte chunk c at r*128 + ((c ^ (r & 7)) * 16)),
// rows padded to a multiple of 128 with zeros.  A CTA therefore streams its
// 128 rows as one contiguous run of 16 KB bulk copies.
__host__ __device__ inline int64_t pack_offset(int64_t row, int64_t col, int64_t K) {
  const int64_t mt = row >> 7, r = row & 127, kt = col >> 6, kk = col & 63;
  return ((mt * (K >> 6) + kt) << 13) + r * 64 + ((((kk >> 3) ^ (r & 7))) << 3) + (kk & 7);
}
void launch_init(bf16* dst, const InitSpec& s, uint64_t seed, cudaStream_t st);

// ---- embedding / norms / sampling -----------------------------------------
void launch_embed(const int32_t* arena, const int32_t* tok_idx, const bf16* E, float* x, int T, int d,
                  cudaStream_t st, const bf16* g = nullptr, bf16* out = nullptr, float eps = 0.f);
// (with g: also out[t] = bf16(RMSNorm(x[t]) * g), the first layer's input norm)
// out[i] = bf16(RMSNorm(x[rows ? rows[i] : i]) * g)
void launch_rmsnorm(const float* x, const bf16* g, bf16* out, const int32_t* rows, int n, int d, float eps,
                    cudaStream_t st);
// Fused split-K reduction + residual add + next RMSNorm (decode GEMMs whose
// epilogue is a residual add):  x[t] += sum_s ws[s][t] (split order), then, if
// g != nullptr, out[t] = bf16(RMSNorm(x[t]) * g).
// xpeer (nullable): also store the updated residual rows there (stage hand-off
// into the next stage's receive slot, a CUDA-IPC peer pointer)
void launch_resid_norm(const float* ws, int splits, float* x, const bf16* g, bf16* out, int T, int d, float eps,
                       cudaStream_t st, float* xpeer = nullptr);
// dst[0, n) = src[0, n) (fp32, n % 4 == 0); dst may be a peer (IPC) pointer
void launch_copy_f32(float* dst, const float* src, int64_t n, cudaStream_t st);
// tokens: arena[outpos[i]] = argmax_j logits[i][j] (lowest index on ties)
void launch_argmax(const float* logits, int n, int V, int32_t* arena, const int32_t* outpos, cudaStream_t st);
// multi-process token return: pairs[2i] = outpos[i], pairs[2i+1] = arena[outpos[i]]; and its inverse
void launch_token_pairs(const int32_t* arena, const int32_t* outpos, int n, int32_t* pairs, cudaStream_t st);
void launch_token_scatter(const int32_t* pairs, int n, int32_t* arena, cudaStream_t st);

// ---- GEMM: C[M,N] = A[M,K] . W[N,K]^T, bf16 in, fp32 accumulate ----------
enum GemmEpi { kEpiF32 = 0, kEpiResid = 1, kEpiSwiGLU = 2, kEpiQKV = 3, kEpiBF16 = 4 };
struct EpiParams {
  int mode;
  float* out_f32;        // kEpiF32: [M, ldo]; kEpiResid: x [M, ldo] (+=)
  bf16* out_bf16;        // kEpiSwiGLU: h [M, N/2]; kEpiQKV: q [M, H*hd]; kEpiBF16
  int ldo;
  // QKV epilogue (RoPE + paged KV write)
  bf16* kcache;          // this layer's pool base: [nblk][2][Hkv][16][hd]
  const int32_t* pos;    // [M]
  const int32_t* slot;   // [M] physical token slot = blk*16 + off
  const float* rope_cs;  // [max_pos][hd/2][2] (cos, sin)
  int H, Hkv, hd;
};

// ---- persistent decode-layer chain (decode_chain.cu) -------------------------
// One launch runs a program of ops separated by grid barriers: weight GEMMs
// (partials per stream-K segment into ws) and the reductions consuming them.
enum ChainKind {
  kChGemm = 0,   // X[T, K] . W[N, K]^T (X = TMA map xmap: 0 a, 1 o, 2 h), reduced per tile with `red`
  kChPrep = 1,   // out = bf16(x * g); ssq[t][tile] (the input side of an RMSNorm)
};
enum ChainRed {
  kRedResid = 0,    // x += W.X (+ xpeer store); if g: out = bf16(x * g), ssq[t][tile]
  kRedSwiGLU = 1,   // out[t][j] = bf16(silu(inv_t (W.X)[2j]) * inv_t (W.X)[2j+1])
  kRedQKV = 2,      // ep (RoPE + q store + paged K/V write) of inv_t * W.X
};
constexpr int kChainMaxOps = 12;
constexpr int kChainSsqStride = 128;   // ssq[tile][token] row stride (T <= 128; d / 128 <= 128 tiles)
constexpr int kChainMaxTiles = 512;    // 128-row weight tiles per GEMM op
struct ChainOp {
  int kind, red;
  const bf16* w;     // kChGemm: tile-packed weights [N (padded to 128), K]
  int N, K, xmap;
  float* x;          // kRedResid / kChPrep: fp32 residual [T, d]
  float* xpeer;      // kRedResid: also store the updated rows here (stage hand-off; nullable)
  const bf16* g;     // kRedResid / kChPrep: the next RMSNorm's gain (nullptr: none)
  bf16* out;         // bf16(x * g) [T, d] (kRedResid, kChPrep); h [T, N/2] (kRedSwiGLU)
  EpiParams ep;      // kRedQKV
};
struct ChainProgram {
  ChainOp op[kChainMaxOps];
  int n_ops;
  int T, d;
  float eps;
  float* ws;                  // segment partials [(tiles + grid) * T * 128] fp32 (largest GEMM)
  float* ssq;                 // [d / 128][kChainSsqStride] per-tile sums of squares of x
  int* cnt;                   // [2][kChainMaxTiles] zero-initialised tile arrival counters (re-armed by the kernel)
  int cnt_parity;             // buffer of this launch's first GEMM op (the host alternates, chain_gemms)
  unsigned long long* bar;    // grid-barrier counter (monotone over the engine's lifetime)
  unsigned long long bar_base;   // its value when this launch starts
  int trace_on;               // TDP_CHAIN_TRACE builds: stamp this launch (decode_chain.cu)
};
// grid = number of SMs (one CTA each); T <= 128; maps = X operands a / o / h
// described with box rows 32 (T <= 32), 64 (T <= 64) or 128.  The counter
// advances by grid * chain_barriers(p).
void launch_decode_chain(const ChainProgram& p, const CUtensorMap* maps, int grid, cudaStream_t st);
int chain_barriers(const ChainProgram& p);
int chain_gemms(const ChainProgram& p);   // GEMM ops: the counter parity advances by this much

// ---- attention --------------------------------------------------------------
// Decode: one query token per sequence; q [n, H*hd] (physical RoPE-pair order),
// paged K/V via block tables; o [n, H*hd] bf16.  Split-KV over split_tokens
// chunks, partial (m, l, acc) merged in split order.
struct DecodeAttnParams {
  const bf16* q;
  const bf16* kv;        // layer pool base
  const int32_t* ctx;    // [n] context length incl. the new token
  const int32_t* bt;     // [n, maxblk]
  int maxblk;
  bf16* o;
  float* part;           // [n, H, max_splits, hd + 2] workspace
  int max_splits;
  int n, H, Hkv, hd;
  int split_tokens;      // context tokens per split (multiple of 16)
  int* counters;         // [n * Hkv] zero-initialised split tickets (reset by the merging CTA)
  // Fused QKV split-K reduction: when set, the QKV GEMM left its split partials
  // unreduced in qkv_ws[s][seq][f] (f < nqkv); every CTA sums its q heads from
  // them in split order and applies RoPE at position ctx-1, and the CTA holding
  // the newest token does the same for its k / v and writes them to the paged
  // cache -- the work of the separate split-K epilogue kernel, bit for bit
  const float* qkv_ws = nullptr;
  int qkv_splits = 0, nqkv = 0;
  const float* rope_cs = nullptr;   // [max_pos][hd/2][2] (cos, sin)
  int64_t part_cap = 0;  // part[] capacity in (sequence x split) slots per head (0: no GQA small splits)
  // TMA view of the whole KV pool (make_kv_map) and this layer's index in it:
  // the tensor-core GQA kernel (G > 1, hd 64 / 128) stages K/V pages through
  // it; nullptr -> the SIMT kernel
  const CUtensorMap* kvmap = nullptr;
  int layer = 0;
  int* work = nullptr;   // [2] zero-initialised work-item / done counters (re-armed by the kernel)
  int64_t n_items = 0;   // (sequence, split, kv head) items of the plan (plan_decode_attn)
  const int32_t* order = nullptr;   // [n] sequences longest-first for the tensor-core kernel's items (nullable)
  int impl = 0;          // 0: kernel by shape (tensor cores for GQA hd 64/128); 1: SIMT; 2: tensor cores (td_bench_attn)
};
// 4-D TMA descriptor of a KV pool [n_layers][C blocks][K|V][Hkv][16][hd] bf16
// viewed as (64 columns, hd/64 halves, C*2*Hkv*16 page rows, n_layers), box
// (64, hd/64, 16, 1), 128B swizzle: one box = a whole 16-token K or V page.
bool make_kv_map(CUtensorMap* map, const bf16* pool, int64_t C, int Hkv, int hd, int n_layers);
void launch_decode_attn(const DecodeAttnParams& p, cudaStream_t st);
// Launch plan from the host copy of the context lengths: sets split_tokens
// and max_splits (part[] must hold cdiv(max_seq_len, kAttnMinSplit) splits per
// head).
constexpr int kAttnMinSplit = 128;   // 64 measured slower (profiles/r1/optimisation_log.md)
// Batches too small to occupy the GPU at 128-token splits (mostly GQA) may go
// down to 32-token splits when the workspace holds them: n * max_splits <=
// DecodeAttnParams::part_cap (the engine sizes part[] for kAttnSmallN sequences
// at 32-token splits)
constexpr int kAttnMinSplitGQA = 32;
#ifndef TDP_ATTN_PDL_MAXN
#define TDP_ATTN_PDL_MAXN 0
#endif
constexpr int kAttnPdlMaxN = TDP_ATTN_PDL_MAXN;   // decode attention as a PDL dependent up to this batch size
constexpr int kAttnSmallN = 32;
void plan_decode_attn(DecodeAttnParams& p, const int* ctx_host);
// Which decode-attention kernel a pure decode micro-batch should use (the
// engine decides before the QKV GEMM: the SIMT kernel can absorb the QKV
// split-K reduction, the tensor-core one cannot).  GQA (hd 64 / 128, G <= 8):
// tensor cores.  MHA: tensor cores for kMhaTcMinN <= n < kMhaTcMaxN sequences
// (mixed lengths: its dynamic item queue balances them, 0.78 / 0.87 vs SIMT
// 0.65 / 0.81 of HBM at n = 64 / 128, mean context 250), and above that at a
// mean context >= kMhaTcMinMeanCtx tokens; else SIMT (random-data sweep,
// profiles/r2/attn_sweep_mha_random.jsonl).
constexpr int kMhaTcMinN = 64;
constexpr int kMhaTcMaxN = 256;
constexpr int kMhaTcMinMeanCtx = 512;
bool decode_attn_use_tc(int n, int H, int Hkv, int hd, const int* ctx_host);

// Prefill: varlen causal over each sequence's own (paged) K/V.
struct PrefillAttnParams {
  const bf16* q;         // [T, H*hd]
  const bf16* kv;
  const int32_t* tok_seq;   // [T] sequence index
  const int32_t* tok_pos;   // [T] absolute position
  const int32_t* bt;        // [n, maxblk]
  int maxblk;
  bf16* o;                  // [T, H*hd]
  int T, H, Hkv, hd;
  const int32_t* seq_ctx;   // [n] context length after this step (= q_start + q_len)
  const int32_t* seq_last;  // [n] row of the sequence's last token
  int n_seqs, max_len;      // max_len >= every q_len
  const int32_t* seq_qstart;  // [n] first query position (chunked prefill); nullptr = all 0
};
void launch_prefill_attn(const PrefillAttnParams& p, cudaStream_t st);

}  // namespace tdp
