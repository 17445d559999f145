// engine.cu -- single-process CUDA execution plane.
//
// Executes the micro-batch plan the controller emits, in launch order, on one
// stream of one sm_100a device.  All pipeline stages of a micro-batch run back
// to back; the stage hand-off is the fp32 residual buffer (SURVEY.md §0.1-6:
// keep the residual stream in fp32).  Generated tokens stay on device: the last
// stage writes argmax tokens into the token arena at the request's next
// position and stage 0 gathers them from there, so the host never waits on the
// GPU inside td_run (the controller's decisions depend only on logical events,
// SURVEY.md §0.1-7, so the host runs ahead, bounded by the metadata ring).
//
// HBM layout (per device):
//   weights  per layer: Wqkv [(H+2Hkv)hd, d] (q/k rotate-half pairs interleaved),
//            Wo [d, H hd], Wgu [2F, d] (gate/up rows interleaved), Wd [d, F],
//            g1, g2 [d]; E [V, d]; gf [d]; Wlm [V, d]      (bf16, K-major)
//   KV pool  per layer: [C blocks][K|V][Hkv][16][hd] bf16
//   arena    int32 tokens, request r at offset off[r]: prompt ++ generated
//   work     x fp32 [T, d]; a bf16 [T, d]; q, o bf16 [T, H hd]; h bf16 [T, F];
//            logits fp32 [n, V]; split-KV partials
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "engine.h"
#include "nccl_rt.h"
#include "kernels/gemm_tc.h"
#include "kernels/kernels.h"

namespace tdp {

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      error = std::string(#x) + ": " + cudaGetErrorString(e_);                        \
      return TD_ECUDA;                                                                \
    }                                                                                 \
  } while (0)

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Stream memory operations (driver API, resolved through the runtime so the
// library does not link libcuda): a stream waits until a 32-bit flag reaches a
// sequence number / writes one after all prior work (with a system-wide fence).
typedef CUresult (*PfnStreamValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PfnStreamValue32 g_wait32 = nullptr, g_write32 = nullptr;
static bool load_stream_memops(std::string* err) {
  if (g_wait32 && g_write32) return true;
  void* a = nullptr;
  void* b = nullptr;
  cudaDriverEntryPointQueryResult qa, qb;
  if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &a, 12000, cudaEnableDefault, &qa) != cudaSuccess ||
      qa != cudaDriverEntryPointSuccess || !a ||
      cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &b, 12000, cudaEnableDefault, &qb) != cudaSuccess ||
      qb != cudaDriverEntryPointSuccess || !b) {
    *err = "cuStreamWaitValue32/cuStreamWriteValue32 not available";
    return false;
  }
  g_wait32 = reinterpret_cast<PfnStreamValue32>(a);
  g_write32 = reinterpret_cast<PfnStreamValue32>(b);
  return true;
}

// Peer-store mailbox layout (identical on every rank; include/tdpipe.h
// TD_HANDOFF_PEER): [flags, 4 KB][token ring][residual receive ring].  Flags
// are monotone 32-bit sequence numbers, one per 64-byte line.
constexpr int kFlagRx = 0;       // residual slot seq filled by stage s-1  (written by s-1)
constexpr int kFlagTxAck = 64;   // residual slot seq consumed by stage s+1 (written by s+1)
constexpr int kFlagTok = 128;    // stage 0: token slot seq filled by the last stage
constexpr int kFlagTokAck = 192; // last stage: token slot seq consumed by stage 0

struct LayerW {
  bf16 *wqkv, *wo, *wgu, *wd, *g1, *g2;
  TcOperand tqkv, to, tgu, td;   // TMA descriptors (box 64 x 128)
};

// X operands of the tcgen05 GEMM: one TMA descriptor per token-tile width.
struct XOps {
  TcOperand by_bn[4];
};

// Per-micro-batch metadata (host-built, one H2D copy): int32 arrays.
struct Meta {
  int n = 0, T = 0, maxblk = 0, max_ctx = 0, prefill = 0;
  // PP+HB hybrid micro-batch: members [0, nd) decode one token, members
  // [nd, n) are prefill chunks (q_start >= 0) of at most max_qlen tokens
  int hybrid = 0, nd = 0, max_qlen = 0;
  // offsets (in int32 units) into the packed buffer
  int o_ctx, o_tokidx, o_pos, o_slot, o_seq, o_last, o_outpos, o_bt, o_qs, o_ord;
  int total = 0;
};

struct TimedLaunch {
  cudaEvent_t a, b;
  int cls;
  int sub = -1;     // optional second class (batch-size bucket)
  double bytes, flops;
};

class CudaEngine : public Engine {
 public:
  ~CudaEngine() override { release(); }

  td_status init(const td_model_shape& s, int n_stages, const td_options& o);
  int64_t kv_blocks() const override { return C_; }
  int64_t kv_bytes_per_block() const override { return kv_block_bytes_layer_ * (own_l1_ - own_l0_); }
  int64_t weight_bytes_stage0() const override { return weight_bytes_; }
  td_status upload(const std::vector<HostReq>& reqs) override;
  bool uploaded() const override { return uploaded_; }
  td_status begin_run(const std::vector<HostReq>& reqs, bool record_logits) override;
  int launch(const MicroBatch& mb, const std::vector<Req>& reqs) override;
  td_status end_run(td_run_stats* st) override;
  td_status get_outputs(const std::vector<HostReq>& reqs, const std::vector<int>& n_out,
                        std::vector<std::vector<int32_t>>* out) override;
  td_status get_logits(int64_t rid, std::vector<float>* out, int* n_steps) override;
  td_status stage_forward(int stage, const td_batch& b, const void* in, void* out) override;
  td_status kv_reset() override;
  td_status profile(int b_max, int k_max, int ctx_len, std::vector<int64_t>* tdec,
                    std::vector<int64_t>* tpre) override;
  void set_timing(bool on) override {
    if (on && !timing_) timing_acc_.clear();   // a new timed region starts
    timing_ = on;
  }
  bool get_timing(const std::string& name, KernelTiming* t) override;
  td_status get_weight(int tid, std::vector<uint16_t>* out, int64_t* rows, int64_t* cols) override;
  td_status bench_step(bool prefill, int n, int len, int iters, double* step_ms, double* ideal_ms) override;
  void get_trace(std::vector<TraceSpan>* spans, std::vector<std::pair<int64_t, int64_t>>* kv) override {
    *spans = trace_spans_;
    *kv = trace_kv_;
  }

 private:
  void release();
  td_status ensure_work(int64_t T, int64_t n, int64_t maxblk);
  // build metadata into ring slot `r`; returns the packed layout
  Meta build_meta(int r, bool prefill, int n, const int* q_start, const int* q_len, const int32_t* arena_off,
                  const char* emit,
                  const std::vector<const std::vector<int32_t>*>& blocks, const int32_t* bt_flat, int bt_stride);
  td_status run_stage(int stage, const Meta& M, const int32_t* dmeta, int32_t* arena, float* xpeer = nullptr,
                      bool* sent = nullptr);
  td_status run_stage_chain(int stage, const Meta& M, const int32_t* dmeta, int32_t* arena, float* xpeer,
                            bool* sent);
  void launch_chain(ChainProgram& P, int T, int sub_cls);
  td_status run_microbatch(const Meta& M, const int32_t* dmeta, int32_t* arena);
  td_status make_x_ops();
  int gemm(const XOps& xo, const TcOperand& W, int T, int N, int K, const EpiParams& ep, bool decode,
           bool defer = false);
  int tbegin(int cls);
  void tend(int idx, double bytes, double flops);
  double accumulate_timed();
  void fill_attn_work(size_t t0, int n, const int* q_start, const int* q_len, int T);
  int ring_acquire();

  td_model_shape s_{};
  td_options o_{};
  int S_ = 1, hd_ = 0, H_ = 0, Hkv_ = 0, d_ = 0, F_ = 0, V_ = 0;
  std::vector<int> stage_l0_, stage_l1_;
  // stages executed by this process: [own_s0_, own_s1_) -- all of them in
  // single-process mode, {rank} in multi-process mode; layers [own_l0_, own_l1_)
  int own_s0_ = 0, own_s1_ = 1, own_l0_ = 0, own_l1_ = 0;
  int world_ = 1, rank_ = 0;
#ifndef TDP_NO_NCCL
  const NcclApi* nc_ = nullptr;
  ncclComm_t cf_ = nullptr, cb_ = nullptr;   // forward (residual) / backward (tokens) comms
#endif
  cudaStream_t tst_ = nullptr;               // stage 0: token-return stream
  static constexpr int kTokRing = 16;
  int32_t* tokbuf_ = nullptr;                // [kTokRing][2 * capN]
  cudaEvent_t tok_ev_[kTokRing] = {};
  int64_t tok_k_ = 0;
  bool tok_have_ = false;
  int32_t* pairs_ = nullptr;                 // last stage: [2 * capN]
  td_status nccl_check(int r, const char* what);
  td_status mp_send_recv_x(bool send, int peer, int T);
  // peer-store hand-off (TD_HANDOFF_PEER)
  bool peer_ = false;
  char* mbox_ = nullptr;                 // own mailbox (exported through CUDA IPC)
  std::map<int, char*> peer_mbox_;       // neighbours' mailboxes, opened here
  static constexpr int kRx = 3;          // residual receive slots per boundary
  int64_t rx_T_ = 0, tok_n_ = 0;         // rows per residual slot, pairs per token slot
  int64_t tok_off_ = 0, rx_off_ = 0;
  uint32_t fwd_out_ = 0, fwd_in_ = 0, tok_out_ = 0, tok_in_ = 0;   // monotone over the ctx lifetime
  td_status peer_init(int64_t rx_T, int64_t tok_n);
  td_status peer_release();
  td_status allgather(const void* send, void* recv, size_t bytes);
  td_status flag_wait(cudaStream_t s, const char* base, int off, uint32_t v);
  td_status flag_write(cudaStream_t s, char* base, int off, uint32_t v);
  char* rx_slot(char* base, uint32_t seq) const { return base + rx_off_ + (int64_t)(seq % kRx) * rx_T_ * d_ * 4; }
  char* tok_slot(char* base, uint32_t seq) const { return base + tok_off_ + (int64_t)(seq % kTokRing) * 2 * tok_n_ * 4; }
 public:
  int returned(const MicroBatch& mb) override;
 private:
  int dev_ = 0;
  cudaStream_t st_ = nullptr;
  // weights
  bf16* wbuf_ = nullptr;
  int64_t weight_bytes_ = 0;
  std::vector<LayerW> L_;
  bf16 *E_ = nullptr, *gf_ = nullptr, *Wlm_ = nullptr;
  // kv
  bf16* kv_ = nullptr;
  int64_t C_ = 0, kv_block_bytes_layer_ = 0;
  CUtensorMap kvmap_{};          // TMA view of the KV pool (tensor-core GQA decode attention)
  bool have_kvmap_ = false;
  float* rope_ = nullptr;
  TcOperand tlm_;
  XOps xa_, xo_, xh_;
  float* ws_ = nullptr;
  int64_t ws_cap_ = 0;
  // persistent decode-layer chain (decode_chain.cu): grid = SM count
  int nsm_ = 148;
  bool chain_ok_ = false;
  unsigned long long* chain_bar_ = nullptr;   // grid-barrier counter
  uint64_t chain_base_ = 0;                   // its value after every enqueued chain launch
  float* ssq_ = nullptr;                      // [128][kChainSsqStride] per-tile sums of squares
  int* tile_cnt_ = nullptr;                   // [2][kChainMaxTiles] per-tile arrival counters
  int chain_parity_ = 0;                      // counter buffer of the next chain launch's first GEMM
  int* counters_ = nullptr;
  int* attn_cnt_ = nullptr;   // decode-attention split tickets [capN * Hkv]
  std::vector<int> mb_ctx_;   // context length per sequence of the micro-batch being enqueued
  // work
  int64_t capT_ = 0, capN_ = 0, capBlk_ = 0;
  float *x_ = nullptr, *logits_ = nullptr, *part_ = nullptr;
  bf16 *a_ = nullptr, *q_ = nullptr, *ob_ = nullptr, *h_ = nullptr;
  int max_splits_cap_ = 0;
  int64_t part_cap_ = 0;
  // arena
  int32_t* arena_ = nullptr;
  int64_t arena_cap_ = 0;
  std::vector<int32_t> arena_off_;
  bool uploaded_ = false;
  // metadata ring
  static constexpr int kRing = 8;
  int32_t* hmeta_[kRing] = {};
  int32_t* dmeta_[kRing] = {};
  cudaEvent_t ring_ev_[kRing] = {};
  bool ring_used_[kRing] = {};
  int64_t meta_cap_ = 0;
  int ring_next_ = 0;
  // run bookkeeping
  cudaEvent_t ev_start_ = nullptr, ev_end_ = nullptr;
  bool started_ = false;
  bool record_ = false;
  std::vector<std::vector<float>> rec_;
  float* hlogits_ = nullptr;
  int64_t hlogits_cap_ = 0;
  int64_t launches_ = 0, h2d_bytes_ = 0;
  double ideal_ns_ = 0, alg_bytes_ = 0, alg_flops_ = 0;   // speed-of-light accounting of the run
  // timing
  bool timing_ = false;
  std::vector<TimedLaunch> timed_;
  std::vector<cudaEvent_t> ev_pool_;
  size_t ev_used_ = 0;
  std::map<std::string, KernelTiming> timing_acc_;
  std::vector<std::string> cls_names_{"decode_attn", "prefill_attn", "gemm_qkv_pre", "gemm_o_pre", "gemm_gu_pre",
                                      "gemm_down_pre", "lm_head_pre", "norm", "stage", "mb", "gemm_qkv_dec",
                                      "gemm_o_dec", "gemm_gu_dec", "gemm_down_dec", "lm_head_dec",
                                      "decode_attn@b1-8", "decode_attn@b9-32", "decode_attn@b33-128",
                                      "decode_attn@b129+", "gemm_dec@b1-8", "gemm_dec@b9-32", "gemm_dec@b33-128",
                                      "gemm_dec@b129+", "decode_chain"};
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> stage_ev_;
  // trace of a timed run: (micro-batch, kind, stage, timed_ index of its span),
  // (timed_ index of the micro-batch's first span, KV blocks in use at launch)
  int64_t cur_mid_ = 0;
  char cur_kind_ = 'D';
  std::vector<std::tuple<int64_t, char, int, int>> tr_;
  std::vector<std::pair<int, int64_t>> tr_kv_;
  std::vector<TraceSpan> trace_spans_;
  std::vector<std::pair<int64_t, int64_t>> trace_kv_;
};

enum Cls { cDecAttn = 0, cPreAttn, cQKV, cO, cGU, cDown, cLM, cNorm, cStage, cMB };
constexpr int kDecOff = 8;   // decode-phase GEMM classes = prefill class + kDecOff
constexpr int kAttnBucket = 15, kGemmBucket = 19;
constexpr int cChain = 23;   // the persistent decode-layer chain (T <= 128)   // + bucket(n): batch-size buckets for decode
static inline int bucket_of(int n) { return n <= 8 ? 0 : n <= 32 ? 1 : n <= 128 ? 2 : 3; }

// --------------------------------------------------------------------- init
td_status CudaEngine::init(const td_model_shape& s, int n_stages, const td_options& o) {
  s_ = s;
  o_ = o;
  S_ = n_stages;
  d_ = s.d_model;
  H_ = s.n_heads;
  Hkv_ = s.n_kv_heads;
  hd_ = d_ / H_;
  F_ = s.d_ffn;
  V_ = s.vocab;
  world_ = o.world_size;
  rank_ = o.rank;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (o.device < 0 || o.device >= ndev) { error = "bad device"; return TD_ECUDA; }
  dev_ = o.device;
  CK(cudaSetDevice(dev_));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev_));
  if (prop.major != 10) { error = "needs an sm_100 (B200) device"; return TD_ECUDA; }
  nsm_ = prop.multiProcessorCount;
  CK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  // layer partition: balanced, remainder to earlier stages
  int q = s.n_layers / S_, r = s.n_layers % S_, l = 0;
  for (int i = 0; i < S_; ++i) {
    stage_l0_.push_back(l);
    l += q + (i < r ? 1 : 0);
    stage_l1_.push_back(l);
  }
  own_s0_ = world_ > 1 ? rank_ : 0;
  own_s1_ = world_ > 1 ? rank_ + 1 : S_;
  own_l0_ = stage_l0_[own_s0_];
  own_l1_ = stage_l1_[own_s1_ - 1];
  const bool has_embed = own_s0_ == 0, has_head = own_s1_ == S_;
  peer_ = world_ > 1 && o.handoff == TD_HANDOFF_PEER;
  if (peer_) {
    if (!o.allgather) { error = "TD_HANDOFF_PEER needs allgather"; return TD_EINVAL; }
    if (!load_stream_memops(&error)) return TD_ECUDA;
    CK(cudaStreamCreateWithFlags(&tst_, cudaStreamNonBlocking));
    for (int i = 0; i < kTokRing; ++i) CK(cudaEventCreateWithFlags(&tok_ev_[i], cudaEventDisableTiming));
  } else if (world_ > 1) {
#ifdef TDP_NO_NCCL
    error = "built without nccl.h";
    return TD_ENCCL;
#else
    if (!o.nccl_ids) { error = "world_size > 1 needs nccl_ids"; return TD_EINVAL; }
    std::string e;
    nc_ = nccl_api(&e);
    if (!nc_) { error = e; return TD_ENCCL; }
    ncclUniqueId idf, idb;
    std::memcpy(&idf, o.nccl_ids, sizeof idf);
    std::memcpy(&idb, static_cast<const char*>(o.nccl_ids) + 128, sizeof idb);
    if (td_status r1 = nccl_check(nc_->commInitRank(&cf_, world_, idf, rank_), "ncclCommInitRank(fwd)")) return r1;
    if (td_status r2 = nccl_check(nc_->commInitRank(&cb_, world_, idb, rank_), "ncclCommInitRank(bwd)")) return r2;
    CK(cudaStreamCreateWithFlags(&tst_, cudaStreamNonBlocking));
    for (int i = 0; i < kTokRing; ++i) CK(cudaEventCreateWithFlags(&tok_ev_[i], cudaEventDisableTiming));
#endif
  }
  // ---- weights (this process's layers only; embedding on stage 0, head on the last)
  const int64_t nqkv = (int64_t)(H_ + 2 * Hkv_) * hd_;
  auto pad = [](int64_t r) { return (r + 127) / 128 * 128; };   // packed weights: rows padded to 128
  const int64_t per_layer = pad(nqkv) * d_ + pad(d_) * H_ * hd_ + pad(2LL * F_) * d_ + pad(d_) * F_ + 2LL * d_;
  const int64_t glob = (has_embed ? (int64_t)V_ * d_ : 0) + (has_head ? pad(V_) * d_ + d_ : 0);
  const int64_t nelem = per_layer * (own_l1_ - own_l0_) + glob;
  weight_bytes_ = nelem * 2;
  size_t fr = 0, tot = 0;
  CK(cudaMemGetInfo(&fr, &tot));
  if ((double)weight_bytes_ > 0.9 * fr) { error = "weights do not fit"; return TD_ENOMEM; }
  CK(cudaMalloc(&wbuf_, nelem * 2));
  CK(cudaMemsetAsync(wbuf_, 0, nelem * 2, st_));   // zero the packed-tile row padding
  bf16* p = wbuf_;
  auto take = [&](int64_t n) { bf16* r = p; p += n; return r; };
  const int L = s.n_layers;
  auto tid = [&](int layer, int which) { return 1 + 9 * layer + which; };
  L_.assign(L, LayerW{});
  for (int i = own_l0_; i < own_l1_; ++i) {
    LayerW w;
    w.wqkv = take(pad(nqkv) * d_);
    w.wo = take(pad(d_) * H_ * hd_);
    w.wgu = take(pad(2LL * F_) * d_);
    w.wd = take(pad(d_) * F_);
    w.g1 = take(d_);
    w.g2 = take(d_);
    auto sc = [](int fan_in) { return std::sqrt(3.0f / (float)fan_in); };
    InitSpec a{kMapQKV, kInitProj, (int)nqkv, d_, tid(i, 1), tid(i, 2), tid(i, 3), H_, Hkv_, hd_, sc(d_), 1};
    launch_init(w.wqkv, a, o.weight_seed, st_);
    InitSpec b{kMapIdentity, kInitProj, d_, H_ * hd_, tid(i, 4), 0, 0, 0, 0, 0, sc(H_ * hd_), 1};
    launch_init(w.wo, b, o.weight_seed, st_);
    InitSpec c{kMapGateUp, kInitProj, 2 * F_, d_, tid(i, 6), tid(i, 7), 0, 0, 0, 0, sc(d_), 1};
    launch_init(w.wgu, c, o.weight_seed, st_);
    InitSpec dd{kMapIdentity, kInitProj, d_, F_, tid(i, 8), 0, 0, 0, 0, 0, sc(F_), 1};
    launch_init(w.wd, dd, o.weight_seed, st_);
    InitSpec g1{kMapIdentity, kInitNorm, 1, d_, tid(i, 0), 0, 0, 0, 0, 0, 0.f, 0};
    launch_init(w.g1, g1, o.weight_seed, st_);
    InitSpec g2{kMapIdentity, kInitNorm, 1, d_, tid(i, 5), 0, 0, 0, 0, 0, 0.f, 0};
    launch_init(w.g2, g2, o.weight_seed, st_);
    L_[i] = w;
  }
  if (has_embed) {
    E_ = take((int64_t)V_ * d_);
    InitSpec e{kMapIdentity, kInitEmbed, V_, d_, 0, 0, 0, 0, 0, 0, 0.f, 0};
    launch_init(E_, e, o.weight_seed, st_);
  }
  if (has_head) {
    Wlm_ = take(pad(V_) * d_);
    gf_ = take(d_);
    InitSpec lm{kMapIdentity, kInitProj, V_, d_, 2 + 9 * L, 0, 0, 0, 0, 0, std::sqrt(3.0f / (float)d_), 1};
    launch_init(Wlm_, lm, o.weight_seed, st_);
    InitSpec gf{kMapIdentity, kInitNorm, 1, d_, 1 + 9 * L, 0, 0, 0, 0, 0, 0.f, 0};
    launch_init(gf_, gf, o.weight_seed, st_);
  }
  CK(cudaGetLastError());
  for (int i = own_l0_; i < own_l1_; ++i) {
    LayerW& w = L_[i];
    w.tqkv = packed_weight(w.wqkv, (int)nqkv, d_);
    w.to = packed_weight(w.wo, d_, H_ * hd_);
    w.tgu = packed_weight(w.wgu, 2 * F_, d_);
    w.td = packed_weight(w.wd, d_, F_);
  }
  if (has_head) tlm_ = packed_weight(Wlm_, V_, d_);
  // ---- RoPE table [max_seq_len][hd/2] (cos, sin), from double
  {
    const int P = s.max_seq_len, half = hd_ / 2;
    std::vector<float> cs((size_t)P * half * 2);
    for (int pp = 0; pp < P; ++pp)
      for (int i = 0; i < half; ++i) {
        const double inv = std::pow((double)s.rope_theta, -2.0 * i / hd_);
        const double ang = (double)pp * inv;
        cs[((size_t)pp * half + i) * 2] = (float)std::cos(ang);
        cs[((size_t)pp * half + i) * 2 + 1] = (float)std::sin(ang);
      }
    CK(cudaMalloc(&rope_, cs.size() * 4));
    CK(cudaMemcpyAsync(rope_, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice, st_));
    CK(cudaStreamSynchronize(st_));
  }
  // ---- work buffers for a default capacity, then the KV pool fills HBM
  const int64_t T0 = std::max<int64_t>(o.prefill_token_budget, s.max_seq_len);
  if (td_status e2 = ensure_work(T0, std::min<int64_t>(o.max_batch_seqs, 1024), cdiv(s.max_seq_len, 16))) return e2;
  kv_block_bytes_layer_ = 2LL * Hkv_ * 16 * hd_ * 2;
  const int64_t per_block = kv_block_bytes_layer_ * (own_l1_ - own_l0_);
  if (o.kv_blocks > 0) {
    C_ = o.kv_blocks;
  } else {
    CK(cudaMemGetInfo(&fr, &tot));
    const double avail = (double)fr - o.hbm_reserve_frac * (double)tot - 512.0 * (1 << 20);
    C_ = (int64_t)(avail / (double)per_block);
  }
  if (peer_) {   // one logical block table for all stages: C = min over ranks
    std::vector<int64_t> all(world_);
    if (td_status r3 = allgather(&C_, all.data(), sizeof(int64_t))) return r3;
    C_ = *std::min_element(all.begin(), all.end());
  }
#ifndef TDP_NO_NCCL
  if (world_ > 1 && !peer_) {   // one logical block table for all stages: C = min over ranks
    int64_t* dC = nullptr;
    CK(cudaMalloc(&dC, sizeof(int64_t)));
    CK(cudaMemcpyAsync(dC, &C_, sizeof(int64_t), cudaMemcpyHostToDevice, st_));
    if (td_status r3 = nccl_check(nc_->allReduce(dC, dC, 1, ncclInt64, ncclMin, cf_, st_), "allReduce(C)")) return r3;
    CK(cudaMemcpyAsync(&C_, dC, sizeof(int64_t), cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    cudaFree(dC);
  }
#endif
  if (C_ < 1) { error = "no room for the KV pool"; return TD_ENOMEM; }
  if (cudaMalloc(&kv_, C_ * per_block) != cudaSuccess) { error = "KV pool allocation failed"; return TD_ENOMEM; }
  CK(cudaMemsetAsync(kv_, 0, C_ * per_block, st_));
  if (hd_ >= 64) {   // GQA always, MHA for large long-context decode batches (decode_attn_use_tc)
    have_kvmap_ = make_kv_map(&kvmap_, kv_, C_, Hkv_, hd_, own_l1_ - own_l0_);
    if (!have_kvmap_) { error = "cuTensorMapEncodeTiled failed (KV pool)"; return TD_ECUDA; }
  }
  if (peer_)
    if (td_status e3 = peer_init(std::max<int64_t>({(int64_t)o.prefill_token_budget, (int64_t)s.max_seq_len,
                                                    (int64_t)o.max_batch_seqs + std::max(o.hb_tokens, 0)}),
                                 (int64_t)o.max_batch_seqs + std::max(o.hb_tokens, 0)))
      return e3;
  // the decode chain: shapes whose GEMM dims are whole 64-wide k blocks
  chain_ok_ = o.decode_chain != 0 && d_ % 128 == 0 && d_ / 128 <= kChainSsqStride && F_ % 64 == 0 &&
              cdiv(2LL * F_, 128) <= kChainMaxTiles && cdiv((int64_t)(H_ + 2 * Hkv_) * hd_, 128) <= kChainMaxTiles &&
              (H_ * hd_) % 64 == 0;
  CK(cudaMalloc(&chain_bar_, sizeof(unsigned long long)));
  CK(cudaMemsetAsync(chain_bar_, 0, sizeof(unsigned long long), st_));
  chain_base_ = 0;
  CK(cudaMalloc(&ssq_, 128 * kChainSsqStride * sizeof(float)));
  CK(cudaMalloc(&tile_cnt_, 2 * kChainMaxTiles * sizeof(int)));
  CK(cudaMemsetAsync(tile_cnt_, 0, 2 * kChainMaxTiles * sizeof(int), st_));
  chain_parity_ = 0;
  CK(cudaEventCreate(&ev_start_));
  CK(cudaEventCreate(&ev_end_));
  for (int i = 0; i < kRing; ++i) CK(cudaEventCreateWithFlags(&ring_ev_[i], cudaEventDisableTiming));
  CK(cudaStreamSynchronize(st_));
  return TD_OK;
}

void CudaEngine::release() {
  if (st_) cudaStreamSynchronize(st_);
  if (tst_) cudaStreamSynchronize(tst_);
  if (peer_ && mbox_) peer_release();   // every rank is done storing into its neighbours' mailboxes first
  cudaFree(wbuf_);
  cudaFree(kv_);
  cudaFree(rope_);
  cudaFree(x_);
  cudaFree(logits_);
  cudaFree(part_);
  cudaFree(a_);
  cudaFree(q_);
  cudaFree(ob_);
  cudaFree(h_);
  cudaFree(arena_);
  cudaFree(ws_);
  cudaFree(counters_);
  cudaFree(chain_bar_);
  cudaFree(ssq_);
  cudaFree(tile_cnt_);
  cudaFree(attn_cnt_);
  for (int i = 0; i < kRing; ++i) {
    if (hmeta_[i]) cudaFreeHost(hmeta_[i]);
    cudaFree(dmeta_[i]);
    if (ring_ev_[i]) cudaEventDestroy(ring_ev_[i]);
  }
  if (hlogits_) cudaFreeHost(hlogits_);
  for (auto e : ev_pool_) cudaEventDestroy(e);
  for (auto& pr : stage_ev_) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
  if (ev_start_) cudaEventDestroy(ev_start_);
  if (ev_end_) cudaEventDestroy(ev_end_);
  cudaFree(tokbuf_);
  cudaFree(pairs_);
  for (int i = 0; i < kTokRing; ++i)
    if (tok_ev_[i]) cudaEventDestroy(tok_ev_[i]);
  if (tst_) { cudaStreamSynchronize(tst_); cudaStreamDestroy(tst_); }
#ifndef TDP_NO_NCCL
  if (nc_ && cf_) nc_->commDestroy(cf_);
  if (nc_ && cb_) nc_->commDestroy(cb_);
#endif
  if (st_) cudaStreamDestroy(st_);
  st_ = nullptr;
}

td_status CudaEngine::ensure_work(int64_t T, int64_t n, int64_t maxblk) {
  T = std::max(T, n);
  if (T <= capT_ && n <= capN_ && maxblk <= capBlk_) return TD_OK;
  CK(cudaStreamSynchronize(st_));
  T = std::max(T, capT_);
  n = std::max(n, capN_);
  maxblk = std::max(maxblk, capBlk_);
  cudaFree(x_); cudaFree(a_); cudaFree(q_); cudaFree(ob_); cudaFree(h_); cudaFree(logits_); cudaFree(part_);
  CK(cudaMalloc(&x_, T * d_ * 4));
  CK(cudaMalloc(&a_, T * d_ * 2));
  CK(cudaMalloc(&q_, T * H_ * hd_ * 2));
  CK(cudaMalloc(&ob_, T * H_ * hd_ * 2));
  CK(cudaMalloc(&h_, T * F_ * 2));
  CK(cudaMalloc(&logits_, n * V_ * 4));
  max_splits_cap_ = (int)cdiv(s_.max_seq_len, kAttnMinSplit);
  // (sequence x split) slots per head: every sequence at 128-token splits, or
  // kAttnSmallN sequences at the GQA small-batch 32-token splits
  part_cap_ = std::max<int64_t>(n * max_splits_cap_,
                                std::min<int64_t>(n, kAttnSmallN) * cdiv(s_.max_seq_len, kAttnMinSplitGQA));
  CK(cudaMalloc(&part_, part_cap_ * H_ * (hd_ + 2) * 4));
  cudaFree(attn_cnt_);
  CK(cudaMalloc(&attn_cnt_, (n * Hkv_ + 2) * sizeof(int)));   // + the tensor-core kernel's work counters
  CK(cudaMemsetAsync(attn_cnt_, 0, (n * Hkv_ + 2) * sizeof(int), st_));
  // metadata ring: per seq 5 ints + bt, per token 4 ints, header
  const int64_t need = 16 + 6 * n + 2 + n * maxblk + 4 * T + 64;
  if (need > meta_cap_) {
    for (int i = 0; i < kRing; ++i) {
      if (hmeta_[i]) cudaFreeHost(hmeta_[i]);
      cudaFree(dmeta_[i]);
      CK(cudaMallocHost(&hmeta_[i], need * 4));
      CK(cudaMalloc(&dmeta_[i], need * 4));
    }
    meta_cap_ = need;
  }
  if (tst_) CK(cudaStreamSynchronize(tst_));
  cudaFree(tokbuf_);
  cudaFree(pairs_);
  CK(cudaMalloc(&tokbuf_, (size_t)kTokRing * 2 * n * 4));
  CK(cudaMalloc(&pairs_, (size_t)2 * n * 4));
  capT_ = T;
  capN_ = n;
  capBlk_ = maxblk;
  // split-K workspace (L2-resident partial tiles) + per-tile tickets
  // 64 MB of fp32 (gemm() falls back to fewer splits beyond it), and at least
  // the decode chain's segment partials of its widest GEMM at 128 tokens
  const int64_t max_tiles = cdiv(std::max<int64_t>({2LL * F_, (int64_t)(H_ + 2 * Hkv_) * hd_, (int64_t)d_}), 128);
  const int64_t wneed = std::max<int64_t>(16LL << 20, (max_tiles + nsm_) * 128 * 128);
  if (wneed > ws_cap_) {
    cudaFree(ws_);
    CK(cudaMalloc(&ws_, wneed * 4));
    ws_cap_ = wneed;
  }
  if (!counters_) {
    CK(cudaMalloc(&counters_, (1 << 16) * sizeof(int)));
    CK(cudaMemsetAsync(counters_, 0, (1 << 16) * sizeof(int), st_));
  }
  return make_x_ops();
}

td_status CudaEngine::make_x_ops() {
  for (int i = 0; i < 4; ++i) {
    const int box = 32 << i;
    if (!make_tc_operand(&xa_.by_bn[i], a_, (int)capT_, d_, box) ||
        !make_tc_operand(&xo_.by_bn[i], ob_, (int)capT_, H_ * hd_, box) ||
        !make_tc_operand(&xh_.by_bn[i], h_, (int)capT_, F_, box)) {
      error = "cuTensorMapEncodeTiled failed (activations)";
      return TD_ECUDA;
    }
  }
  return TD_OK;
}

// Dense weight GEMM: tcgen05 kernel on tile-packed weights.  Decode GEMMs
// stream weights; split-K targets ~288 CTAs (about 2 per SM), at most 8 splits
// and >= 4 k-blocks per split (measured sweep: scripts/gemm_sweep.py).
// Returns the split count used; with defer = true and splits > 1 the caller
// consumes the partials (launch_resid_norm).
int CudaEngine::gemm(const XOps& xo, const TcOperand& W, int T, int N, int K, const EpiParams& ep, bool decode,
                     bool defer) {
  int splits = 1;
  if (decode && T > 128) {
    // 129..512-token decode batches are near (or past) the tensor roof: the
    // token-major kernel (128 tokens x 256 features per tile).  The residual
    // GEMMs (O, down: their split partials are summed by the resid_norm launch
    // that follows anyway) split K when their tiles fill the 148 SMs badly
    // (< 96 tiles): the fewest splits giving >= 128 units, >= 16 k-blocks
    // each.  Measured per shape in profiles/r2/gemm_sweep_t128.txt.
    decode = false;
    const int64_t tiles = (int64_t)((T + 127) / 128) * ((N + 255) / 256);
    if (ep.mode == kEpiResid && defer && tiles < 96) {
      while (splits < 4 && tiles * splits < 128 && (K / 64) / (splits + 1) >= 16 &&
             (int64_t)(splits + 1) * T * ((N + 127) / 128 * 128) <= ws_cap_)
        ++splits;
    }
  }
  if (decode) {
    // split-K to ~288 CTAs (about 2 per SM), at most 8 splits, >= 4 k-blocks
    // per split, partials within the workspace (scripts/gemm_sweep.py).
    // (Half-width token tiles at 33..128 tokens measured faster isolated but
    // slower in the job: profiles/r2/ab/README.md.)
    const int bn = tc_bn_for(T, true);
    const int64_t ctas = (int64_t)((N + 127) / 128) * ((T + bn - 1) / bn);
    splits = (int)std::max<int64_t>(1, std::min<int64_t>(8, 288 / ctas));   // (4 / 6 for O, down: slower,
                                                                             //  profiles/r2/timeline/)
    while (splits > 1 && (K / 64) / splits < 4) --splits;
    while (splits > 1 && (int64_t)splits * T * ((N + 127) / 128 * 128) > ws_cap_) --splits;
  }
  const int used = launch_gemm_tc(W, xo.by_bn, T, ep, splits, ws_, counters_, decode, st_, defer);
  launches_ += (used > 1 && !defer) ? 2 : 1;
  return used;
}

// -------------------------------------------------------------------- ring
int CudaEngine::ring_acquire() {
  const int r = ring_next_;
  ring_next_ = (ring_next_ + 1) % kRing;
  if (ring_used_[r]) cudaEventSynchronize(ring_ev_[r]);   // bound the host run-ahead
  ring_used_[r] = true;
  return r;
}

Meta CudaEngine::build_meta(int r, bool prefill, int n, const int* q_start, const int* q_len,
                            const int32_t* arena_off, const char* emit, const std::vector<const std::vector<int32_t>*>& blocks,
                            const int32_t* bt_flat, int bt_stride) {
  Meta M;
  M.n = n;
  M.prefill = prefill ? 1 : 0;
  int T = 0, maxblk = 1, max_ctx = 1;
  for (int i = 0; i < n; ++i) {
    T += q_len[i];
    const int ctx = q_start[i] + q_len[i];
    max_ctx = std::max(max_ctx, ctx);
    maxblk = std::max<int>(maxblk, (int)cdiv(ctx, 16));
  }
  M.T = T;
  M.maxblk = maxblk;
  M.max_ctx = max_ctx;
  int off = 0;
  M.o_ctx = off; off += n;
  M.o_last = off; off += n;
  M.o_outpos = off; off += n;
  M.o_tokidx = off; off += T;
  M.o_pos = off; off += T;
  M.o_slot = off; off += T;
  M.o_seq = off; off += T;
  M.o_bt = off; off += n * maxblk;
  M.o_qs = off; off += n;
  M.o_ord = off; off += n;
  M.total = off;
  int32_t* h = hmeta_[r];
  int t = 0;
  mb_ctx_.resize(n);
  for (int i = 0; i < n; ++i) {
    const int ctx = q_start[i] + q_len[i];
    mb_ctx_[i] = ctx;
    h[M.o_ctx + i] = ctx;
    const int nb = (int)cdiv(ctx, 16);
    int32_t* bt = h + M.o_bt + (int64_t)i * maxblk;
    for (int b = 0; b < maxblk; ++b)
      bt[b] = b < nb ? (blocks.empty() ? bt_flat[(int64_t)i * bt_stride + b] : (*blocks[i])[b]) : 0;
    for (int j = 0; j < q_len[i]; ++j, ++t) {
      const int pos = q_start[i] + j;
      h[M.o_tokidx + t] = arena_off ? arena_off[i] + pos : t;
      h[M.o_pos + t] = pos;
      h[M.o_slot + t] = bt[pos >> 4] * 16 + (pos & 15);
      h[M.o_seq + t] = i;
    }
    h[M.o_last + i] = t - 1;
    // no token for a prefill chunk that does not complete its prompt (PP+HB)
    h[M.o_outpos + i] = emit && !emit[i] ? -1 : arena_off ? arena_off[i] + ctx : 0;
    h[M.o_qs + i] = q_start[i];
  }
  // sequences by context length, longest first (the tensor-core decode
  // attention numbers its work items in this order: longest-processing-first)
  int32_t* ord = h + M.o_ord;
  for (int i = 0; i < n; ++i) ord[i] = i;
  std::stable_sort(ord, ord + n, [&](int32_t a, int32_t b) { return mb_ctx_[a] > mb_ctx_[b]; });
  return M;
}

// ------------------------------------------------------------------ timing
// fold the recorded (event pair, class) spans into timing_acc_; returns the
// summed stage-busy milliseconds.  The stream must be synchronised.
double CudaEngine::accumulate_timed() {
  double busy = 0;
  for (auto& tl : timed_) {
    float t = 0.f;
    cudaEventElapsedTime(&t, tl.a, tl.b);
    for (int c : {tl.cls, tl.sub}) {
      if (c < 0) continue;
      KernelTiming& kt = timing_acc_[cls_names_[c]];
      kt.launches++;
      kt.ms += t;
      kt.bytes += tl.bytes;
      kt.flops += tl.flops;
      if (c == tl.cls) kt.launch_bytes.push_back(tl.bytes);
    }
    if (tl.cls == cStage) busy += t;
  }
  timed_.clear();
  ev_used_ = 0;
  return busy;
}

int CudaEngine::tbegin(int cls) {
  if (!timing_) return -1;
  if (ev_used_ + 2 > ev_pool_.size()) {
    for (int i = 0; i < 256; ++i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev_pool_.push_back(e);
    }
  }
  TimedLaunch tl;
  tl.a = ev_pool_[ev_used_++];
  tl.b = ev_pool_[ev_used_++];
  tl.cls = cls;
  tl.bytes = tl.flops = 0;
  cudaEventRecord(tl.a, st_);
  timed_.push_back(tl);
  return (int)timed_.size() - 1;
}
void CudaEngine::tend(int idx, double bytes, double flops) {
  if (!timing_ || idx < 0) return;
  TimedLaunch& tl = timed_[idx];
  tl.bytes = bytes;
  tl.flops = flops;
  cudaEventRecord(tl.b, st_);
}

// algorithmic work of the attention launches recorded since timed_[t0]:
// decode attention reads every context token's K and V (2*Hkv*hd*2 bytes per
// layer) + q and o; prefill attention does the causal QK^T
// and PV, 4*H*hd FLOPs per (query, key <= query) pair
void CudaEngine::fill_attn_work(size_t t0, int n, const int* q_start, const int* q_len, int T) {
  double kvb = 0;
  for (int i = 0; i < n; ++i) kvb += (double)(q_start[i] + q_len[i]);
  kvb = kvb * 2.0 * Hkv_ * hd_ * 2 + 4.0 * n * H_ * hd_;
  double pf = 0;
  for (int i = 0; i < n; ++i) pf += 0.5 * (double)q_len[i] * (q_len[i] + 1);
  pf *= 4.0 * H_ * hd_;
  const double pb = (double)T * (2.0 * H_ * hd_ * 2 + 2.0 * Hkv_ * hd_ * 2);
  for (size_t k = t0; k < timed_.size(); ++k) {
    if (timed_[k].cls == cDecAttn) timed_[k].bytes = kvb;
    if (timed_[k].cls == cPreAttn) { timed_[k].flops = pf; timed_[k].bytes = pb; }
  }
}

bool CudaEngine::get_timing(const std::string& name, KernelTiming* t) {
  auto it = timing_acc_.find(name);
  if (it == timing_acc_.end()) { *t = KernelTiming(); return true; }
  *t = it->second;
  return true;
}

// ------------------------------------------------------------------ forward
td_status CudaEngine::run_stage(int stage, const Meta& M, const int32_t* dm, int32_t* arena, float* xpeer,
                                bool* sent) {
  if (chain_ok_ && !M.prefill && !M.hybrid && M.T <= 128) return run_stage_chain(stage, M, dm, arena, xpeer, sent);
  if (sent) *sent = false;
  // Decode attention is launched without PDL (a PDL dependent, it made decode
  // steps 2-10 % slower at b >= 8: profiles/r1/pdl_ab.md); every other hot
  // kernel is a PDL dependent of its predecessor.
  const bool attn_nopdl = !M.prefill && M.n > kAttnPdlMaxN;
  const int T = M.T, n = M.n;
  const int nqkv = (H_ + 2 * Hkv_) * hd_;
  const float eps = s_.rms_eps;
  const bool dec = !M.prefill;
  // pure decode on the tensor-core attention kernel (GQA; MHA at large batches
  // of long contexts): the QKV split-K reduction then runs as its own kernel
  const bool attn_tc = dec && !M.hybrid && have_kvmap_ && decode_attn_use_tc(n, H_, Hkv_, hd_, mb_ctx_.data());
  bool normed = false;   // a_ already holds RMSNorm(x; g1) (fused into the embedding / the previous down-proj reduction)
  if (stage == 0) {   // + the first layer's input norm
    launch_embed(arena, dm + M.o_tokidx, E_, x_, T, d_, st_, L_[stage_l0_[stage]].g1, a_, eps);
    launches_++;
    normed = true;
  }
  bool final_normed = false;   // decode at the last stage: the final norm rides on the last down-proj reduction
  for (int l = stage_l0_[stage]; l < stage_l1_[stage]; ++l) {
    const LayerW& w = L_[l];
    bf16* kvl = kv_ + (int64_t)(l - own_l0_) * C_ * (kv_block_bytes_layer_ / 2);
    if (!normed) {
      launch_rmsnorm(x_, w.g1, a_, nullptr, T, d_, eps, st_);
      launches_++;
    }
    normed = false;
    EpiParams ep{};
    ep.mode = kEpiQKV;
    ep.out_bf16 = q_;
    ep.kcache = kvl;
    ep.pos = dm + M.o_pos;
    ep.slot = dm + M.o_slot;
    ep.rope_cs = rope_;
    ep.H = H_;
    ep.Hkv = Hkv_;
    ep.hd = hd_;
    const int iq = tbegin(cQKV + (M.prefill ? 0 : kDecOff));
    if (iq >= 0 && !M.prefill) timed_[iq].sub = kGemmBucket + bucket_of(T);
    // pure decode: the QKV split-K reduction (+ RoPE + K/V write) is left to
    // the attention kernel (DecodeAttnParams::qkv_ws) -- one launch fewer
    // (not for the tensor-core GQA kernel: its single q-prep warp would redo
    // the reduction for every split item of a sequence; the split-K reduce
    // kernel does it once per token and the kernel bulk-copies q)
    const bool defer_qkv = dec && !M.hybrid && !attn_tc;
    const int qsplits = gemm(xa_, w.tqkv, T, nqkv, d_, ep, dec, /*defer=*/defer_qkv);
    tend(iq, (double)nqkv * d_ * 2 + (double)T * d_ * 2 + (double)T * nqkv * 2, 2.0 * T * nqkv * d_);
    if (M.hybrid) {
      // PP+HB: decode members [0, nd) -- one token each, so token row = member
      // index, as the decode kernel expects -- and prefill chunks [nd, n)
      // attending to their paged prefix + causal chunk
      if (M.nd > 0) {
        DecodeAttnParams dp{q_, kvl, dm + M.o_ctx, dm + M.o_bt, M.maxblk, ob_, part_, 0, M.nd, H_, Hkv_, hd_, 0,
                            attn_cnt_};
        dp.part_cap = part_cap_;
        dp.kvmap = have_kvmap_ ? &kvmap_ : nullptr;
        dp.layer = l - own_l0_;
        dp.work = attn_cnt_ + capN_ * Hkv_;
        plan_decode_attn(dp, mb_ctx_.data());
        pdl_suppress(true);
        launch_decode_attn(dp, st_);
        pdl_suppress(false);
        launches_++;
      }
      if (M.nd < n) {
        const int nc = n - M.nd;
        PrefillAttnParams pp{q_, kvl, dm + M.o_seq, dm + M.o_pos, dm + M.o_bt + (int64_t)M.nd * M.maxblk, M.maxblk,
                             ob_, T, H_, Hkv_, hd_, dm + M.o_ctx + M.nd, dm + M.o_last + M.nd, nc, M.max_qlen,
                             dm + M.o_qs + M.nd};
        launch_prefill_attn(pp, st_);
        launches_++;
      }
    } else if (M.prefill) {
      // (q_start > 0: chunked prefill over the paged prefix, td_stage_forward)
      PrefillAttnParams pp{q_, kvl, dm + M.o_seq, dm + M.o_pos, dm + M.o_bt, M.maxblk, ob_, T, H_, Hkv_, hd_,
                           dm + M.o_ctx, dm + M.o_last, n, M.max_ctx, dm + M.o_qs};
      const int ip = tbegin(cPreAttn);
      launch_prefill_attn(pp, st_);
      tend(ip, 0, 0);
      launches_++;
    } else {
      DecodeAttnParams dp{q_, kvl, dm + M.o_ctx, dm + M.o_bt, M.maxblk, ob_, part_, 0, n, H_, Hkv_, hd_, 0,
                          attn_cnt_};
      dp.part_cap = part_cap_;
      dp.kvmap = have_kvmap_ ? &kvmap_ : nullptr;
      dp.layer = l - own_l0_;
      dp.work = attn_cnt_ + capN_ * Hkv_;
      dp.order = dm + M.o_ord;
      dp.impl = attn_tc ? 2 : 1;
      if (defer_qkv && qsplits > 1) {
        dp.qkv_ws = ws_;
        dp.qkv_splits = qsplits;
        dp.nqkv = nqkv;
        dp.rope_cs = rope_;
      }
      plan_decode_attn(dp, mb_ctx_.data());
      const int ida = tbegin(cDecAttn);
      if (ida >= 0) timed_[ida].sub = kAttnBucket + bucket_of(n);
      pdl_suppress(attn_nopdl);
      launch_decode_attn(dp, st_);
      pdl_suppress(false);
      tend(ida, 0, 0);   // bytes filled by the caller-side accumulator (ctx-dependent)
      launches_++;
    }
    EpiParams eo{};
    eo.mode = kEpiResid;
    eo.out_f32 = x_;
    eo.ldo = d_;
    const int io = tbegin(cO + (M.prefill ? 0 : kDecOff));
    if (io >= 0 && !M.prefill) timed_[io].sub = kGemmBucket + bucket_of(T);
    const int so = gemm(xo_, w.to, T, d_, H_ * hd_, eo, dec, /*defer=*/true);
    tend(io, (double)d_ * H_ * hd_ * 2 + (double)T * H_ * hd_ * 2 + 8.0 * T * d_, 2.0 * T * d_ * H_ * hd_);
    if (so > 1) launch_resid_norm(ws_, so, x_, w.g2, a_, T, d_, eps, st_);   // reduce + residual + norm
    else launch_rmsnorm(x_, w.g2, a_, nullptr, T, d_, eps, st_);
    launches_++;
    EpiParams eg{};
    eg.mode = kEpiSwiGLU;
    eg.out_bf16 = h_;
    const int ig = tbegin(cGU + (M.prefill ? 0 : kDecOff));
    if (ig >= 0 && !M.prefill) timed_[ig].sub = kGemmBucket + bucket_of(T);
    gemm(xa_, w.tgu, T, 2 * F_, d_, eg, dec);
    tend(ig, 2.0 * F_ * d_ * 2 + (double)T * d_ * 2 + (double)T * F_ * 2, 2.0 * T * 2 * F_ * d_);
    EpiParams ed{};
    ed.mode = kEpiResid;
    ed.out_f32 = x_;
    ed.ldo = d_;
    const int idn = tbegin(cDown + (M.prefill ? 0 : kDecOff));
    if (idn >= 0 && !M.prefill) timed_[idn].sub = kGemmBucket + bucket_of(T);
    const int sd = gemm(xh_, w.td, T, d_, F_, ed, dec, /*defer=*/true);
    tend(idn, (double)d_ * F_ * 2 + (double)T * F_ * 2 + 8.0 * T * d_, 2.0 * T * d_ * F_);
    if (sd > 1) {   // reduce + residual, fused with the next layer's input norm when it is in this stage
      const bool last_layer = l + 1 == stage_l1_[stage];
      // decode micro-batches (one token per sequence: row i = sequence i) at
      // the last stage also get the final norm here instead of a launch
      const bool fin = last_layer && stage == S_ - 1 && dec && !M.hybrid;
      const bf16* gnext = !last_layer ? L_[l + 1].g1 : fin ? gf_ : nullptr;
      final_normed = fin;
      // the stage's final residual rows are also stored straight into the
      // next stage's receive slot (peer store over NVLink; no separate send)
      float* xp = last_layer ? xpeer : nullptr;
      launch_resid_norm(ws_, sd, x_, gnext, a_, T, d_, eps, st_, xp);
      launches_++;
      normed = gnext != nullptr;
      if (xp && sent) *sent = true;
    }
  }
  if (stage == S_ - 1) {
    if (!final_normed) {
      launch_rmsnorm(x_, gf_, a_, dm + M.o_last, n, d_, eps, st_);
      launches_++;   // final norm
    }
    EpiParams el{};
    el.mode = kEpiF32;
    el.out_f32 = logits_;
    el.ldo = V_;
    const int il = tbegin(cLM + (M.prefill ? 0 : kDecOff));
    gemm(xa_, tlm_, n, V_, d_, el, dec);
    tend(il, (double)V_ * d_ * 2 + (double)n * d_ * 2 + 4.0 * n * V_, 2.0 * n * V_ * d_);
    launches_++;
    if (arena) {
      launch_argmax(logits_, n, V_, arena, dm + M.o_outpos, st_);
      launches_++;
    }
  }
  return TD_OK;
}

// One chain launch (decode_chain.cu); the timed span counts the algorithmic
// bytes / FLOPs of its GEMMs (weights + activations in and out).
void CudaEngine::launch_chain(ChainProgram& P, int T, int sub_cls) {
  P.T = T;
  P.d = d_;
  P.eps = s_.rms_eps;
  P.ws = ws_;
  P.ssq = ssq_;
  P.cnt = tile_cnt_;
  P.cnt_parity = chain_parity_;
  P.bar = chain_bar_;
  P.bar_base = chain_base_;
  P.trace_on = P.n_ops >= 4;   // (trace builds) a full post-attention layer program
  double bytes = 0, flops = 0;
  for (int i = 0; i < P.n_ops; ++i)
    if (P.op[i].kind == kChGemm) {
      const double N = P.op[i].N, K = P.op[i].K;
      bytes += N * K * 2 + (double)T * K * 2 + (double)T * N * 2;
      flops += 2.0 * T * N * K;
    }
  const int bi = T <= 32 ? 0 : T <= 64 ? 1 : 2;
  const CUtensorMap maps[3] = {xa_.by_bn[bi].map, xo_.by_bn[bi].map, xh_.by_bn[bi].map};
  const int it = tbegin(cChain);
  if (it >= 0) timed_[it].sub = sub_cls;
  launch_decode_chain(P, maps, nsm_, st_);
  tend(it, bytes, flops);
  chain_base_ += (uint64_t)nsm_ * chain_barriers(P);
  chain_parity_ = (chain_parity_ + chain_gemms(P)) & 1;
  launches_++;
}

// Decode micro-batch of <= 128 tokens: per layer one attention launch and one
// persistent chain launch covering  O-proj -> residual + RMSNorm -> gate/up ->
// SwiGLU -> down -> residual (+ the stage hand-off store) -> the next layer's
// RMSNorm -> QKV -> RoPE + K/V write.  Same arithmetic as run_stage up to the
// fp32 summation order of the split-K partials and norm sums.
td_status CudaEngine::run_stage_chain(int stage, const Meta& M, const int32_t* dm, int32_t* arena, float* xpeer,
                                      bool* sent) {
  if (sent) *sent = false;
  const int T = M.T, n = M.n;
  const int nqkv = (H_ + 2 * Hkv_) * hd_;
  const int sub = kGemmBucket + bucket_of(T);
  if (stage == 0) {
    launch_embed(arena, dm + M.o_tokidx, E_, x_, T, d_, st_);
    launches_++;
  }
  auto add = [](ChainProgram& P, const ChainOp& op) { P.op[P.n_ops++] = op; };
  auto gemm_op = [](const TcOperand& W, int N, int K, int xmap, int red) {
    ChainOp g{};
    g.kind = kChGemm;
    g.red = red;
    g.w = W.base;
    g.N = N;
    g.K = K;
    g.xmap = xmap;
    return g;
  };
  // residual GEMMs (O, down): x += W.X (+ the hand-off store); a = bf16(x * g)
  // and the sums of squares for the next GEMM's RMSNorm when g != nullptr
  auto resid_gemm = [&](const TcOperand& W, int K, int xmap, float* xp, const bf16* g) {
    ChainOp r = gemm_op(W, d_, K, xmap, kRedResid);
    r.x = x_;
    r.xpeer = xp;
    r.g = g;
    r.out = a_;
    return r;
  };
  auto qkv_op = [&](int l) {
    ChainOp r = gemm_op(L_[l].tqkv, nqkv, d_, 0, kRedQKV);
    EpiParams& ep = r.ep;
    ep.mode = kEpiQKV;
    ep.out_bf16 = q_;
    ep.kcache = kv_ + (int64_t)(l - own_l0_) * C_ * (kv_block_bytes_layer_ / 2);
    ep.pos = dm + M.o_pos;
    ep.slot = dm + M.o_slot;
    ep.rope_cs = rope_;
    ep.H = H_;
    ep.Hkv = Hkv_;
    ep.hd = hd_;
    return r;
  };
  const int l0 = stage_l0_[stage], l1 = stage_l1_[stage];
  {
    ChainProgram P{};
    ChainOp pr{};
    pr.kind = kChPrep;   // a = bf16(x * g1), sums of squares of x
    pr.x = x_;
    pr.g = L_[l0].g1;
    pr.out = a_;
    add(P, pr);
    add(P, qkv_op(l0));
    launch_chain(P, T, sub);
  }
  for (int l = l0; l < l1; ++l) {
    const LayerW& w = L_[l];
    bf16* kvl = kv_ + (int64_t)(l - own_l0_) * C_ * (kv_block_bytes_layer_ / 2);
    DecodeAttnParams dp{q_, kvl, dm + M.o_ctx, dm + M.o_bt, M.maxblk, ob_, part_, 0, n, H_, Hkv_, hd_, 0, attn_cnt_};
    dp.part_cap = part_cap_;
    dp.kvmap = have_kvmap_ ? &kvmap_ : nullptr;
    dp.layer = l - own_l0_;
    dp.work = attn_cnt_ + capN_ * Hkv_;
    dp.order = dm + M.o_ord;
    plan_decode_attn(dp, mb_ctx_.data());
    const int ida = tbegin(cDecAttn);
    if (ida >= 0) timed_[ida].sub = kAttnBucket + bucket_of(n);
    pdl_suppress(n > kAttnPdlMaxN);
    launch_decode_attn(dp, st_);
    pdl_suppress(false);
    tend(ida, 0, 0);
    launches_++;
    const bool last = l + 1 == l1;
    ChainProgram P{};
    add(P, resid_gemm(w.to, H_ * hd_, 1, nullptr, w.g2));
    {
      ChainOp gu = gemm_op(w.tgu, 2 * F_, d_, 0, kRedSwiGLU);
      gu.out = h_;
      add(P, gu);
    }
    // the stage's final residual rows also go straight into the next stage's
    // receive slot (peer store over NVLink; no separate send)
    add(P, resid_gemm(w.td, F_, 2, last ? xpeer : nullptr, last ? nullptr : L_[l + 1].g1));
    if (last && xpeer && sent) *sent = true;
    if (!last) add(P, qkv_op(l + 1));
    launch_chain(P, T, sub);
  }
  if (stage == S_ - 1) {
    launches_++;   // final norm
    launch_rmsnorm(x_, gf_, a_, dm + M.o_last, n, d_, s_.rms_eps, st_);
    EpiParams el{};
    el.mode = kEpiF32;
    el.out_f32 = logits_;
    el.ldo = V_;
    const int il = tbegin(cLM + kDecOff);
    gemm(xa_, tlm_, n, V_, d_, el, true);
    tend(il, (double)V_ * d_ * 2 + (double)n * d_ * 2 + 4.0 * n * V_, 2.0 * n * V_ * d_);
    launches_++;
    if (arena) {
      launch_argmax(logits_, n, V_, arena, dm + M.o_outpos, st_);
      launches_++;
    }
  }
  return TD_OK;
}

td_status CudaEngine::run_microbatch(const Meta& M, const int32_t* dm, int32_t* arena) {
  const int64_t nx = (int64_t)M.T * d_;
  if (peer_ && (M.T > rx_T_ || M.n > tok_n_)) { error = "micro-batch exceeds the hand-off slots"; return TD_ERANGE; }
  for (int s = own_s0_; s < own_s1_; ++s) {
    if (peer_ && s > 0) {
      // residual hand-off from stage s-1: wait for slot `seq`, take it, free it
      const uint32_t seq = ++fwd_in_;
      if (td_status e = flag_wait(st_, mbox_, kFlagRx, seq)) return e;
      launch_copy_f32(x_, reinterpret_cast<const float*>(rx_slot(mbox_, seq)), nx, st_);
      launches_++;
      if (td_status e = flag_write(st_, peer_mbox_.at(rank_ - 1), kFlagTxAck, seq)) return e;
    } else if (world_ > 1 && s > 0) {   // receive the fp32 residual hand-off from stage s-1
      if (td_status e = mp_send_recv_x(false, s - 1, M.T)) return e;
    }
    float* xpeer = nullptr;
    if (peer_ && s < S_ - 1) {   // reserve slot `seq` of stage s+1 (free once it consumed seq - kRx)
      const uint32_t seq = ++fwd_out_;
      if (seq > (uint32_t)kRx)
        if (td_status e = flag_wait(st_, mbox_, kFlagTxAck, seq - kRx)) return e;
      xpeer = reinterpret_cast<float*>(rx_slot(peer_mbox_.at(rank_ + 1), seq));
    }
    const int is = tbegin(cStage);
    if (is >= 0) tr_.emplace_back(cur_mid_, cur_kind_, s, is);
    bool sent = false;
    if (td_status e = run_stage(s, M, dm, arena, xpeer, &sent)) return e;
    tend(is, 0, 0);
    if (peer_ && s < S_ - 1) {
      if (!sent) {   // the stage did not end in a split-K reduce: store the rows now
        launch_copy_f32(xpeer, x_, nx, st_);
        launches_++;
      }
      if (td_status e = flag_write(st_, peer_mbox_.at(rank_ + 1), kFlagRx, fwd_out_)) return e;
    } else if (world_ > 1 && s < S_ - 1) {
      if (td_status e = mp_send_recv_x(true, s + 1, M.T)) return e;
    }
    if (peer_ && s == S_ - 1) {   // sampled tokens -> stage 0's token ring (peer stores)
      const uint32_t k = ++tok_out_;
      if (k > (uint32_t)kTokRing)
        if (td_status e = flag_wait(st_, mbox_, kFlagTokAck, k - kTokRing)) return e;
      launch_token_pairs(arena, dm + M.o_outpos, M.n, reinterpret_cast<int32_t*>(tok_slot(peer_mbox_.at(0), k)),
                         st_);
      launches_++;
      if (td_status e = flag_write(st_, peer_mbox_.at(0), kFlagTok, k)) return e;
    }
#ifndef TDP_NO_NCCL
    if (world_ > 1 && !peer_ && s == S_ - 1) {   // sampled tokens -> stage 0 (token-return comm)
      launch_token_pairs(arena, dm + M.o_outpos, M.n, pairs_, st_);
      if (td_status e = nccl_check(nc_->send(pairs_, (size_t)2 * M.n, ncclInt32, 0, cb_, st_), "ncclSend(tokens)"))
        return e;
    }
#endif
  }
  return TD_OK;
}

td_status CudaEngine::nccl_check(int r, const char* what) {
#ifndef TDP_NO_NCCL
  if (r != ncclSuccess) {
    error = std::string(what) + ": " + (nc_ ? nc_->getErrorString((ncclResult_t)r) : "nccl");
    return TD_ENCCL;
  }
#else
  (void)r;
  (void)what;
#endif
  return TD_OK;
}

td_status CudaEngine::mp_send_recv_x(bool send, int peer, int T) {
#ifndef TDP_NO_NCCL
  const size_t cnt = (size_t)T * d_;
  return send ? nccl_check(nc_->send(x_, cnt, ncclFloat32, peer, cf_, st_), "ncclSend(x)")
              : nccl_check(nc_->recv(x_, cnt, ncclFloat32, peer, cf_, st_), "ncclRecv(x)");
#else
  (void)send;
  (void)peer;
  (void)T;
  return TD_ENCCL;
#endif
}

// Stage 0 of a multi-process pipeline learns the tokens of micro-batch k from
// the last stage when the controller processes k's return (in launch order on
// every rank): receive (position, token) pairs on the token stream, scatter
// into the arena, and let the compute stream wait on it before its next launch.
int CudaEngine::returned(const MicroBatch& mb) {
  if (peer_ && own_s0_ == 0) {
    const int n = (int)mb.members.size();
    const uint32_t k = ++tok_in_;
    const int slot = (int)(tok_k_ % kTokRing);
    if (flag_wait(tst_, mbox_, kFlagTok, k)) return TD_ECUDA;
    launch_token_scatter(reinterpret_cast<const int32_t*>(tok_slot(mbox_, k)), n, arena_, tst_);
    if (flag_write(tst_, peer_mbox_.at(S_ - 1), kFlagTokAck, k)) return TD_ECUDA;
    cudaEventRecord(tok_ev_[slot], tst_);
    tok_have_ = true;
    ++tok_k_;
    return 0;
  }
#ifndef TDP_NO_NCCL
  if (world_ > 1 && own_s0_ == 0) {
    const int n = (int)mb.members.size();
    const int slot = (int)(tok_k_ % kTokRing);
    int32_t* buf = tokbuf_ + (int64_t)slot * 2 * capN_;
    if (nccl_check(nc_->recv(buf, (size_t)2 * n, ncclInt32, S_ - 1, cb_, tst_), "ncclRecv(tokens)")) return TD_ENCCL;
    launch_token_scatter(buf, n, arena_, tst_);
    cudaEventRecord(tok_ev_[slot], tst_);
    tok_have_ = true;
    ++tok_k_;
  }
#else
  (void)mb;
#endif
  return 0;
}

// ------------------------------------------------------------------- runs
td_status CudaEngine::upload(const std::vector<HostReq>& reqs) {
  int64_t total = 0;
  arena_off_.resize(reqs.size());
  for (size_t i = 0; i < reqs.size(); ++i) {
    arena_off_[i] = (int32_t)total;
    total += (int64_t)reqs[i].prompt.size() + reqs[i].max_new + 1;
  }
  if (total > INT32_MAX) { error = "token arena too large"; return TD_ERANGE; }
  if (total > arena_cap_) {
    CK(cudaStreamSynchronize(st_));
    cudaFree(arena_);
    CK(cudaMalloc(&arena_, std::max<int64_t>(total, 1) * 4));
    arena_cap_ = total;
  }
  std::vector<int32_t> h((size_t)std::max<int64_t>(total, 1), 0);
  for (size_t i = 0; i < reqs.size(); ++i)
    std::memcpy(h.data() + arena_off_[i], reqs[i].prompt.data(), reqs[i].prompt.size() * 4);
  CK(cudaMemcpyAsync(arena_, h.data(), total * 4, cudaMemcpyHostToDevice, st_));
  CK(cudaStreamSynchronize(st_));
  h2d_bytes_ = total * 4;
  uploaded_ = true;
  return TD_OK;
}

td_status CudaEngine::begin_run(const std::vector<HostReq>& reqs, bool record_logits) {
  CK(cudaSetDevice(dev_));
  if (!uploaded_ || arena_off_.size() != reqs.size()) {
    if (td_status e = upload(reqs)) return e;
  }
  int64_t maxL = 1;
  for (auto& r : reqs) maxL = std::max<int64_t>(maxL, (int64_t)r.prompt.size() + r.max_new);
  const int64_t T = std::max<int64_t>(o_.prefill_token_budget, maxL);
  if (td_status e = ensure_work(T, std::max<int64_t>((int64_t)reqs.size(), 1), cdiv(maxL + 1, 16))) return e;
  if (peer_) {
    // hand-off slot sizes vs the largest micro-batch this request set can
    // form: a decode micro-batch holds at most every live request, and a live
    // request holds >= 1 KV block, so <= min(requests, C) sequences (+ the
    // PP+HB prefill chunks); a prefill one <= max(budget, longest prompt incl.
    // recompute).  Every rank sees the same requests, so all re-size together.
    const int64_t nseq = std::min<int64_t>((int64_t)reqs.size(), C_) + std::max(o_.hb_tokens, 0);
    const int64_t rxT = std::max<int64_t>({(int64_t)o_.prefill_token_budget, maxL, nseq});
    if (rxT > rx_T_ || nseq > tok_n_) {
      if (td_status e = peer_release()) return e;
      if (td_status e = peer_init(std::max(rxT, rx_T_), std::max(nseq, tok_n_))) return e;
    }
  }
  record_ = record_logits;
  rec_.assign(record_logits ? reqs.size() : 0, {});
  launches_ = 0;
  ideal_ns_ = alg_bytes_ = alg_flops_ = 0;
  timed_.clear();
  ev_used_ = 0;
  started_ = false;
  for (int i = 0; i < kRing; ++i) ring_used_[i] = false;
  tok_k_ = 0;
  tok_have_ = false;
  return TD_OK;
}

int CudaEngine::launch(const MicroBatch& mb, const std::vector<Req>& reqs) {
  const int n = (int)mb.members.size();
  if (!started_) {
    cudaEventRecord(ev_start_, st_);
    started_ = true;
  }
  std::vector<int32_t> aoff(n);
  std::vector<const std::vector<int32_t>*> blocks(n);
  for (int i = 0; i < n; ++i) {
    aoff[i] = arena_off_[mb.members[i]];
    blocks[i] = &reqs[mb.members[i]].blocks;
  }
  {
    int64_t T = 0, mb_blk = 1;
    for (int i = 0; i < n; ++i) {
      T += mb.q_len[i];
      mb_blk = std::max<int64_t>(mb_blk, cdiv(mb.q_start[i] + mb.q_len[i], 16));
    }
    if (T > capT_ || mb_blk > capBlk_ || n > capN_) {
      if (ensure_work(T, n, mb_blk)) return TD_ECUDA;
      for (int i = 0; i < kRing; ++i) ring_used_[i] = false;
    }
  }
  {   // algorithmic work of this micro-batch on this process's layers (td_run_stats.ideal_ns)
    const int nl = own_l1_ - own_l0_;
    const double nqkv = (double)(H_ + 2 * Hkv_) * hd_;
    const double w_layer = 2.0 * (nqkv * d_ + (double)d_ * H_ * hd_ + 2.0 * F_ * d_ + (double)d_ * F_ + 2.0 * d_);
    const bool head = own_s1_ == S_;
    const double kv_tok = 2.0 * Hkv_ * hd_ * 2;   // K + V bytes per token per layer
    double T = 0, ctx_sum = 0, att = 0;
    for (int i = 0; i < n; ++i) {
      const double qs = mb.q_start[i], ql = mb.q_len[i];
      T += ql;
      ctx_sum += qs + ql;
      att += ql * (qs + (ql + 1) / 2);   // causal (query, key) pairs
    }
    const double bytes = nl * (w_layer + ctx_sum * kv_tok + T * kv_tok) + (head ? 2.0 * V_ * d_ + 2.0 * d_ : 0.0);
    const double flops = nl * (T * w_layer + 4.0 * H_ * hd_ * att) + (head ? 2.0 * n * V_ * d_ : 0.0);
    alg_bytes_ += bytes;
    alg_flops_ += flops;
    if (o_.hbm_peak_gbs > 0 && o_.tc_peak_tflops > 0)
      ideal_ns_ += std::max(bytes / o_.hbm_peak_gbs, flops / (o_.tc_peak_tflops * 1e3));
  }
  const int r = ring_acquire();
  // PP+HB hybrid micro-batch: decode members (q_start >= L) lead, then chunks;
  // a chunk emits a token only if it completes its prompt
  std::vector<char> emit(n, 1);
  int nd = 0;
  if (mb.kind == 'H') {
    for (int i = 0; i < n; ++i) {
      const Req& rq = reqs[mb.members[i]];
      emit[i] = mb.q_start[i] + mb.q_len[i] >= rq.L;
      if (mb.q_start[i] >= rq.L && i == nd) ++nd;
    }
  }
  Meta M = build_meta(r, mb.kind == 'P', n, mb.q_start.data(), mb.q_len.data(), aoff.data(), emit.data(), blocks,
                      nullptr, 0);
  cur_mid_ = mb.mid;
  cur_kind_ = mb.kind;
  if (timing_) {   // KV-usage timeline (PAPER.md:580-585 fig:memory_usage): blocks held at this launch
    int64_t used = 0;
    for (const auto& rq : reqs) used += (int64_t)rq.blocks.size();
    tr_kv_.emplace_back((int)timed_.size(), used);
  }
  if (mb.kind == 'H') {
    M.hybrid = 1;
    M.nd = nd;
    for (int i = nd; i < n; ++i) M.max_qlen = std::max(M.max_qlen, mb.q_len[i]);
  }
  if (cudaMemcpyAsync(dmeta_[r], hmeta_[r], (size_t)M.total * 4, cudaMemcpyHostToDevice, st_) != cudaSuccess) {
    error = "metadata H2D failed";
    return TD_ECUDA;
  }
  if (world_ > 1 && own_s0_ == 0 && tok_have_)   // tokens of every returned micro-batch are in the arena
    cudaStreamWaitEvent(st_, tok_ev_[(tok_k_ - 1) % kTokRing], 0);
  h2d_bytes_ += (int64_t)M.total * 4;
  const size_t t0 = timed_.size();
  if (td_status e = run_microbatch(M, dmeta_[r], arena_)) return e;
  if (timing_) fill_attn_work(t0, n, mb.q_start.data(), mb.q_len.data(), M.T);
  cudaEventRecord(ring_ev_[r], st_);
  cudaError_t e = take_launch_error();
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) { error = std::string("launch: ") + cudaGetErrorString(e); return TD_ECUDA; }
  if (record_) {
    if (hlogits_cap_ < (int64_t)n * V_) {
      if (hlogits_) cudaFreeHost(hlogits_);
      cudaMallocHost(&hlogits_, (size_t)n * V_ * 4);
      hlogits_cap_ = (int64_t)n * V_;
    }
    cudaMemcpyAsync(hlogits_, logits_, (size_t)n * V_ * 4, cudaMemcpyDeviceToHost, st_);
    if (cudaStreamSynchronize(st_) != cudaSuccess) { error = "sync failed"; return TD_ECUDA; }
    for (int i = 0; i < n; ++i) {
      if (!emit[i]) continue;
      auto& v = rec_[mb.members[i]];
      v.insert(v.end(), hlogits_ + (size_t)i * V_, hlogits_ + (size_t)(i + 1) * V_);
    }
  }
  return 0;
}

td_status CudaEngine::end_run(td_run_stats* st) {
  if (tst_) {   // stage 0: the last token scatter belongs to the job
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventRecord(e, tst_));
    CK(cudaStreamWaitEvent(st_, e, 0));
    cudaEventDestroy(e);
  }
  CK(cudaEventRecord(ev_end_, st_));
  CK(cudaStreamSynchronize(st_));
  float ms = 0.f;
  if (started_) CK(cudaEventElapsedTime(&ms, ev_start_, ev_end_));
  st->makespan_ns = (int64_t)((double)ms * 1e6);
  if (timing_ && started_) {   // the run's trace, in ns from its first launch
    auto at = [&](cudaEvent_t e) {
      float t = 0.f;
      cudaEventElapsedTime(&t, ev_start_, e);
      return (int64_t)((double)t * 1e6);
    };
    trace_spans_.clear();
    trace_kv_.clear();
    for (const auto& x : tr_) {
      const TimedLaunch& tl = timed_[std::get<3>(x)];
      trace_spans_.push_back({std::get<0>(x), std::get<1>(x), std::get<2>(x), at(tl.a), at(tl.b)});
    }
    for (const auto& kv : tr_kv_)
      if (kv.first < (int)timed_.size()) trace_kv_.emplace_back(at(timed_[kv.first].a), kv.second);
  }
  tr_.clear();
  tr_kv_.clear();
  const double busy = accumulate_timed();
  if (timing_ && ms > 0) {
    st->bubble_frac = 1.0 - busy / ((double)S_ * ms);
    st->busy_ns[0] = (int64_t)(busy * 1e6 / S_);
  }
  st->gpu_launches = launches_;
  st->h2d_bytes = h2d_bytes_;
  st->ideal_ns = ideal_ns_;
  st->alg_bytes = alg_bytes_;
  st->alg_flops = alg_flops_;
  return TD_OK;
}

td_status CudaEngine::get_outputs(const std::vector<HostReq>& reqs, const std::vector<int>& n_out,
                                  std::vector<std::vector<int32_t>>* out) {
  int64_t total = 0;
  for (size_t i = 0; i < reqs.size(); ++i) total += (int64_t)reqs[i].prompt.size() + reqs[i].max_new + 1;
  std::vector<int32_t> h((size_t)std::max<int64_t>(total, 1));
  CK(cudaMemcpyAsync(h.data(), arena_, total * 4, cudaMemcpyDeviceToHost, st_));
  CK(cudaStreamSynchronize(st_));
  out->assign(reqs.size(), {});
  for (size_t i = 0; i < reqs.size(); ++i) {
    const int32_t* base = h.data() + arena_off_[i] + reqs[i].prompt.size();
    (*out)[i].assign(base, base + n_out[i]);
  }
  return TD_OK;
}

td_status CudaEngine::get_logits(int64_t rid, std::vector<float>* out, int* n_steps) {
  if (!record_ || rid < 0 || rid >= (int64_t)rec_.size()) { error = "logits not recorded"; return TD_ESTATE; }
  *out = rec_[rid];
  *n_steps = (int)(out->size() / V_);
  return TD_OK;
}

td_status CudaEngine::kv_reset() {
  CK(cudaMemsetAsync(kv_, 0, C_ * kv_block_bytes_layer_ * (own_l1_ - own_l0_), st_));
  CK(cudaStreamSynchronize(st_));
  return TD_OK;
}

// ------------------------------------------------------- weight read-back
// td_get_weight: copy the physical tensor D2H and undo the device layout on the
// host -- tile packing (pack_offset), the rotate-half pair interleave of the q
// and k rows ((i, i+hd/2) stored as rows (2i, 2i+1)) and the gate/up row
// interleave (gate j = row 2j, up j = row 2j+1).
td_status CudaEngine::get_weight(int tid, std::vector<uint16_t>* out, int64_t* rows, int64_t* cols) {
  CK(cudaSetDevice(dev_));
  const int L = s_.n_layers;
  const int64_t nqkv = (int64_t)(H_ + 2 * Hkv_) * hd_;
  const bf16* src = nullptr;
  int64_t phys_elems = 0, K = 0;
  bool packed = false;
  std::function<int64_t(int64_t)> prow = [](int64_t r) { return r; };   // logical row -> physical row
  auto pad = [](int64_t r) { return (r + 127) / 128 * 128; };
  auto rope_row = [this](int64_t base, int64_t r) {
    const int64_t h = r / hd_, i = r % hd_;
    const int64_t j = i < hd_ / 2 ? 2 * i : 2 * (i - hd_ / 2) + 1;
    return base + h * hd_ + j;
  };
  if (tid == 0) {
    if (!E_) { error = "embedding not held by this process"; return TD_EINVAL; }
    src = E_; *rows = V_; *cols = d_; phys_elems = (int64_t)V_ * d_;
  } else if (tid == 1 + 9 * L) {
    if (!gf_) { error = "final norm not held by this process"; return TD_EINVAL; }
    src = gf_; *rows = 1; *cols = d_; phys_elems = d_;
  } else if (tid == 2 + 9 * L) {
    if (!Wlm_) { error = "LM head not held by this process"; return TD_EINVAL; }
    src = Wlm_; *rows = V_; *cols = d_; K = d_; packed = true; phys_elems = pad(V_) * d_;
  } else if (tid >= 1 && tid < 1 + 9 * L) {
    const int l = (tid - 1) / 9, which = (tid - 1) % 9;
    if (l < own_l0_ || l >= own_l1_) { error = "layer not held by this process"; return TD_EINVAL; }
    const LayerW& w = L_[l];
    switch (which) {
      case 0: src = w.g1; *rows = 1; *cols = d_; phys_elems = d_; break;
      case 5: src = w.g2; *rows = 1; *cols = d_; phys_elems = d_; break;
      case 1: case 2: case 3: {
        src = w.wqkv; K = d_; packed = true; phys_elems = pad(nqkv) * d_;
        *cols = d_;
        *rows = which == 1 ? (int64_t)H_ * hd_ : (int64_t)Hkv_ * hd_;
        if (which == 1) prow = [=](int64_t r) { return rope_row(0, r); };
        else if (which == 2) prow = [=](int64_t r) { return rope_row((int64_t)H_ * hd_, r); };
        else prow = [=](int64_t r) { return (int64_t)(H_ + Hkv_) * hd_ + r; };
        break;
      }
      case 4: src = w.wo; K = (int64_t)H_ * hd_; packed = true; phys_elems = pad(d_) * K; *rows = d_; *cols = K; break;
      case 6: case 7:
        src = w.wgu; K = d_; packed = true; phys_elems = pad(2LL * F_) * d_; *rows = F_; *cols = d_;
        prow = [=](int64_t r) { return 2 * r + (which == 7 ? 1 : 0); };
        break;
      case 8: src = w.wd; K = F_; packed = true; phys_elems = pad(d_) * F_; *rows = d_; *cols = F_; break;
    }
  } else {
    error = "tensor id out of range";
    return TD_EINVAL;
  }
  std::vector<uint16_t> phys((size_t)phys_elems);
  CK(cudaStreamSynchronize(st_));
  CK(cudaMemcpy(phys.data(), src, (size_t)phys_elems * 2, cudaMemcpyDeviceToHost));
  out->assign((size_t)(*rows * *cols), 0);
  for (int64_t r = 0; r < *rows; ++r) {
    const int64_t p = prow(r);
    for (int64_t c = 0; c < *cols; ++c)
      (*out)[(size_t)(r * *cols + c)] = phys[(size_t)(packed ? pack_offset(p, c, K) : p * *cols + c)];
  }
  return TD_OK;
}

// ----------------------------------------------------------- stage forward
td_status CudaEngine::stage_forward(int stage, const td_batch& b, const void* in, void* out) {
  CK(cudaSetDevice(dev_));
  if (stage < own_s0_ || stage >= own_s1_) { error = "stage not owned by this process"; return TD_EINVAL; }
  const int n = b.n_seqs;
  if (n < 1) { error = "empty batch"; return TD_EINVAL; }
  int T = 0, maxctx = 1;
  for (int i = 0; i < n; ++i) {
    if (b.q_len[i] < 1 || b.q_start[i] < 0) { error = "bad q_len/q_start"; return TD_EINVAL; }
    if (b.kind == TD_BATCH_DECODE && b.q_len[i] != 1) { error = "decode q_len must be 1"; return TD_EINVAL; }
    if (b.kind == TD_BATCH_PREFILL && b.q_start[i] < 0) { error = "q_start < 0"; return TD_EINVAL; }
    T += b.q_len[i];
    maxctx = std::max(maxctx, b.q_start[i] + b.q_len[i]);
    if (maxctx > s_.max_seq_len) { error = "context > max_seq_len"; return TD_ERANGE; }
    if (cdiv(b.q_start[i] + b.q_len[i], 16) > b.max_blocks) { error = "block table too short"; return TD_EINVAL; }
    for (int k = 0; k < cdiv(b.q_start[i] + b.q_len[i], 16); ++k) {
      const int32_t blk = b.block_table[(int64_t)i * b.max_blocks + k];
      if (blk < 0 || blk >= C_) { error = "block id out of range"; return TD_ERANGE; }
    }
  }
  if (td_status e = ensure_work(T, n, cdiv(maxctx, 16))) return e;
  CK(cudaStreamSynchronize(st_));
  for (int i = 0; i < kRing; ++i) ring_used_[i] = false;
  const int r = 0;
  Meta M = build_meta(r, b.kind == TD_BATCH_PREFILL, n, b.q_start, b.q_len, nullptr, nullptr, {}, b.block_table,
                      b.max_blocks);
  CK(cudaMemcpyAsync(dmeta_[r], hmeta_[r], (size_t)M.total * 4, cudaMemcpyHostToDevice, st_));
  int32_t* tok = nullptr;
  if (stage == 0) {
    CK(cudaMalloc(&tok, (size_t)T * 4));
    CK(cudaMemcpyAsync(tok, in, (size_t)T * 4, cudaMemcpyHostToDevice, st_));
  } else {
    CK(cudaMemcpyAsync(x_, in, (size_t)T * d_ * 4, cudaMemcpyHostToDevice, st_));
  }
  td_status e = run_stage(stage, M, dmeta_[r], tok);
  if (e == TD_OK) {
    const cudaError_t le = take_launch_error();
    if (le != cudaSuccess) { error = std::string("launch: ") + cudaGetErrorString(le); e = TD_ECUDA; }
  }
  if (e == TD_OK) {
    if (stage == S_ - 1) CK(cudaMemcpyAsync(out, logits_, (size_t)n * V_ * 4, cudaMemcpyDeviceToHost, st_));
    else CK(cudaMemcpyAsync(out, x_, (size_t)T * d_ * 4, cudaMemcpyDeviceToHost, st_));
  }
  CK(cudaStreamSynchronize(st_));
  CK(cudaGetLastError());
  if (tok) cudaFree(tok);
  return e;
}

// ----------------------------------------------------------------- profile
// Eq.1 needs "the execution time ... for each batch size":
// per-stage decode-step ns at a representative context, prefill ns per token
// count; sampled grid, integer linear interpolation, per-stage max.
td_status CudaEngine::profile(int b_max, int k_max, int ctx_len, std::vector<int64_t>* tdec,
                              std::vector<int64_t>* tpre) {
  CK(cudaSetDevice(dev_));
  ctx_len = std::min(ctx_len, s_.max_seq_len - 1);
  const int nb = (int)cdiv(ctx_len, 16);
  if (td_status e = ensure_work(std::max(k_max, b_max), b_max, nb + 1)) return e;
  int32_t* tok = nullptr;
  CK(cudaMalloc(&tok, (size_t)std::max(k_max, b_max) * 4));
  CK(cudaMemsetAsync(tok, 0, (size_t)std::max(k_max, b_max) * 4, st_));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto time_batch = [&](bool prefill, int n, const std::vector<int>& qs, const std::vector<int>& ql,
                        int64_t* out_ns) -> td_status {
    std::vector<int32_t> bt((size_t)n * (nb + 1));
    for (int i = 0; i < n; ++i)
      for (int k = 0; k <= nb; ++k) bt[(size_t)i * (nb + 1) + k] = (int32_t)(((int64_t)i * (nb + 1) + k) % C_);
    for (int i = 0; i < kRing; ++i) ring_used_[i] = false;
    Meta M = build_meta(0, prefill, n, qs.data(), ql.data(), nullptr, nullptr, {}, bt.data(), nb + 1);
    CK(cudaMemcpyAsync(dmeta_[0], hmeta_[0], (size_t)M.total * 4, cudaMemcpyHostToDevice, st_));
    int64_t worst = 0;
    for (int s = own_s0_; s < own_s1_; ++s) {
      std::vector<float> ts;
      for (int rep = 0; rep < 6; ++rep) {
        CK(cudaEventRecord(e0, st_));
        if (td_status e = run_stage(s, M, dmeta_[0], tok)) return e;
        CK(cudaEventRecord(e1, st_));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (rep >= 2) ts.push_back(ms);
      }
      std::sort(ts.begin(), ts.end());
      worst = std::max<int64_t>(worst, (int64_t)(ts[ts.size() / 2] * 1e6));
    }
    *out_ns = worst;
    return TD_OK;
  };
  const bool saved = timing_;
  timing_ = false;
  std::vector<int> bgrid;
  for (int b = 1; b <= b_max; b = b < 16 ? b * 2 : b + (b < 256 ? 16 : 64)) bgrid.push_back(b);
  if (bgrid.back() != b_max) bgrid.push_back(b_max);
  std::vector<int64_t> bval;
  for (int b : bgrid) {
    std::vector<int> qs(b, ctx_len - 1), ql(b, 1);
    int64_t ns = 0;
    if (td_status e = time_batch(false, b, qs, ql, &ns)) return e;
    bval.push_back(ns);
  }
  std::vector<int> kgrid;
  for (int k = 16; k < k_max; k *= 2) kgrid.push_back(k);
  kgrid.push_back(k_max);
  std::vector<int64_t> kval;
  for (int k : kgrid) {
    std::vector<int> qs, ql;
    for (int left = k; left > 0; left -= ctx_len) { qs.push_back(0); ql.push_back(std::min(left, ctx_len)); }
    int64_t ns = 0;
    if (td_status e = time_batch(true, (int)qs.size(), qs, ql, &ns)) return e;
    kval.push_back(ns);
  }
  timing_ = saved;
  if (peer_) {   // every rank must hold the same frozen table: per-stage max over ranks
    std::vector<int64_t> mine(bval);
    mine.insert(mine.end(), kval.begin(), kval.end());
    std::vector<int64_t> all(mine.size() * world_);
    if (td_status r = allgather(mine.data(), all.data(), mine.size() * sizeof(int64_t))) return r;
    for (int rr = 0; rr < world_; ++rr)
      for (size_t i = 0; i < mine.size(); ++i) mine[i] = std::max(mine[i], all[rr * mine.size() + i]);
    std::copy(mine.begin(), mine.begin() + bval.size(), bval.begin());
    std::copy(mine.begin() + bval.size(), mine.end(), kval.begin());
  }
#ifndef TDP_NO_NCCL
  if (world_ > 1 && !peer_) {   // every rank must hold the same frozen table: per-stage max over ranks
    std::vector<int64_t> all(bval);
    all.insert(all.end(), kval.begin(), kval.end());
    int64_t* dv = nullptr;
    CK(cudaMalloc(&dv, all.size() * sizeof(int64_t)));
    CK(cudaMemcpyAsync(dv, all.data(), all.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st_));
    if (td_status r = nccl_check(nc_->allReduce(dv, dv, all.size(), ncclInt64, ncclMax, cf_, st_), "allReduce(profile)"))
      return r;
    CK(cudaMemcpyAsync(all.data(), dv, all.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    cudaFree(dv);
    std::copy(all.begin(), all.begin() + bval.size(), bval.begin());
    std::copy(all.begin() + bval.size(), all.end(), kval.begin());
  }
#endif
  auto interp = [](const std::vector<int>& g, const std::vector<int64_t>& v, int maxv, std::vector<int64_t>* out) {
    out->assign(maxv + 1, 0);
    for (int x = 1; x <= maxv; ++x) {
      size_t j = 0;
      while (j + 1 < g.size() && g[j + 1] < x) ++j;
      if (x <= g[0]) { (*out)[x] = v[0]; continue; }
      if (j + 1 >= g.size()) { (*out)[x] = v.back(); continue; }
      const int64_t x0 = g[j], x1 = g[j + 1];
      (*out)[x] = v[j] + (v[j + 1] - v[j]) * (x - x0) / (x1 - x0);
    }
  };
  interp(bgrid, bval, b_max, tdec);
  interp(kgrid, kval, k_max, tpre);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(tok);
  CK(cudaMemsetAsync(kv_, 0, C_ * kv_block_bytes_layer_ * (own_l1_ - own_l0_), st_));
  CK(cudaStreamSynchronize(st_));
  return TD_OK;
}

// -------------------------------------------------------------- bench step
// One synthetic micro-batch through this process's stages, `iters` times:
// decode = n sequences at context `len` (each decodes its token at position
// len-1), prefill = n prompts of `len` tokens.  Pages are distinct and
// scattered like the profile's.  Per-kernel CUDA-event timing accumulates into
// timing_acc_ (cleared first); *step_ms = mean device time of one pass over
// the stages, *ideal_ms = its speed of light max(bytes / HBM, FLOPs / TC)
// under the td_options peaks (the td_run_stats accounting).
td_status CudaEngine::bench_step(bool prefill, int n, int len, int iters, double* step_ms, double* ideal_ms) {
  CK(cudaSetDevice(dev_));
  if (n < 1 || len < 1 || iters < 1 || len > s_.max_seq_len) { error = "bad bench_step shape"; return TD_EINVAL; }
  const int nb = (int)cdiv(len, 16);
  if ((int64_t)n * nb > C_) { error = "KV pool too small for the bench step"; return TD_ERANGE; }
  const int T = prefill ? n * len : n;
  if (td_status e = ensure_work(T, n, nb)) return e;
  int32_t* tok = nullptr;
  CK(cudaMalloc(&tok, (size_t)T * 4));
  CK(cudaMemsetAsync(tok, 0, (size_t)T * 4, st_));
  std::vector<int32_t> bt((size_t)n * nb);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < nb; ++k) bt[(size_t)i * nb + k] = (int32_t)(((int64_t)k * n + i) % C_);   // interleaved pages
  std::vector<int> qs(n, prefill ? 0 : len - 1), ql(n, prefill ? len : 1);
  for (int i = 0; i < kRing; ++i) ring_used_[i] = false;
  Meta M = build_meta(0, prefill, n, qs.data(), ql.data(), nullptr, nullptr, {}, bt.data(), nb);
  CK(cudaMemcpyAsync(dmeta_[0], hmeta_[0], (size_t)M.total * 4, cudaMemcpyHostToDevice, st_));
  const bool saved = timing_;
  timing_ = false;
  for (int w = 0; w < 2; ++w)
    for (int s = own_s0_; s < own_s1_; ++s)
      if (td_status e = run_stage(s, M, dmeta_[0], tok)) { cudaFree(tok); return e; }
  timing_acc_.clear();
  timed_.clear();
  ev_used_ = 0;
  timing_ = true;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, st_));
  for (int it = 0; it < iters; ++it) {
    const size_t t0 = timed_.size();
    for (int s = own_s0_; s < own_s1_; ++s)
      if (td_status e = run_stage(s, M, dmeta_[0], tok)) { cudaFree(tok); timing_ = saved; return e; }
    fill_attn_work(t0, n, qs.data(), ql.data(), T);
  }
  CK(cudaEventRecord(e1, st_));
  CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  accumulate_timed();
  timing_ = saved;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(tok);
  *step_ms = ms / iters;
  {   // speed of light of one pass (as launch())
    const int nl = own_l1_ - own_l0_;
    const double nqkv = (double)(H_ + 2 * Hkv_) * hd_;
    const double w_layer = 2.0 * (nqkv * d_ + (double)d_ * H_ * hd_ + 2.0 * F_ * d_ + (double)d_ * F_ + 2.0 * d_);
    const bool head = own_s1_ == S_;
    const double kv_tok = 2.0 * Hkv_ * hd_ * 2;
    const double ctx_sum = (double)n * len, att = prefill ? n * (0.5 * len * (len + 1.0)) : (double)n * len;
    const double bytes = nl * (w_layer + ctx_sum * kv_tok + T * kv_tok) + (head ? 2.0 * V_ * d_ + 2.0 * d_ : 0.0);
    const double flops = nl * (T * w_layer + 4.0 * H_ * hd_ * att) + (head ? 2.0 * n * V_ * d_ : 0.0);
    *ideal_ms = (o_.hbm_peak_gbs > 0 && o_.tc_peak_tflops > 0)
                    ? std::max(bytes / o_.hbm_peak_gbs, flops / (o_.tc_peak_tflops * 1e3)) / 1e6
                    : 0.0;
  }
  CK(cudaMemsetAsync(kv_, 0, C_ * kv_block_bytes_layer_ * (own_l1_ - own_l0_), st_));
  CK(cudaStreamSynchronize(st_));
  return TD_OK;
}

// ------------------------------------------------------ peer-store hand-off
td_status CudaEngine::allgather(const void* send, void* recv, size_t bytes) {
  if (!o_.allgather || o_.allgather(o_.allgather_user, send, recv, bytes) != 0) {
    error = "allgather callback failed";
    return TD_EINVAL;
  }
  return TD_OK;
}

td_status CudaEngine::flag_wait(cudaStream_t s, const char* base, int off, uint32_t v) {
  const CUresult r = g_wait32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(base + off), v,
                              CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) { error = "cuStreamWaitValue32 failed (" + std::to_string((int)r) + ")"; return TD_ECUDA; }
  return TD_OK;
}

td_status CudaEngine::flag_write(cudaStream_t s, char* base, int off, uint32_t v) {
  // default flags: the value becomes visible only after every prior store of
  // the stream (including peer stores over NVLink) -- a release
  const CUresult r = g_write32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(base + off), v,
                               CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) { error = "cuStreamWriteValue32 failed (" + std::to_string((int)r) + ")"; return TD_ECUDA; }
  return TD_OK;
}

// Every rank allocates one mailbox with the same layout, exports it through
// CUDA IPC, and opens the mailboxes of the ranks it stores into: s+1 (residual
// + its flag), s-1 (slot-free acks), and for stages 0 / S-1 each other (token
// ring, token acks).  Slot capacities are fixed here from the options, so no
// mailbox is ever reallocated (a micro-batch over them fails with TD_ERANGE).
td_status CudaEngine::peer_init(int64_t rx_T, int64_t tok_n) {
  rx_T_ = rx_T;
  tok_n_ = tok_n;
  fwd_out_ = fwd_in_ = tok_out_ = tok_in_ = 0;   // a fresh mailbox: every flag is 0
  tok_off_ = 4096;
  rx_off_ = tok_off_ + cdiv((int64_t)kTokRing * 2 * tok_n_ * 4, 4096) * 4096;
  const int64_t bytes = rank_ == 0 ? rx_off_ : rx_off_ + (int64_t)kRx * rx_T_ * d_ * 4;
  CK(cudaMalloc(&mbox_, bytes));
  CK(cudaMemset(mbox_, 0, 4096));
  CK(cudaDeviceSynchronize());
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, mbox_));
  std::vector<cudaIpcMemHandle_t> all(world_);
  if (td_status e = allgather(&h, all.data(), sizeof h)) return e;
  std::vector<int> need;
  if (rank_ > 0) need.push_back(rank_ - 1);
  if (rank_ < S_ - 1) need.push_back(rank_ + 1);
  if (rank_ == 0) need.push_back(S_ - 1);
  if (rank_ == S_ - 1) need.push_back(0);
  for (int r : need) {
    if (r == rank_ || peer_mbox_.count(r)) continue;
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, all[r], cudaIpcMemLazyEnablePeerAccess));
    peer_mbox_[r] = static_cast<char*>(p);
  }
  int one = 1;   // every mailbox is open (and its flags zeroed) before anyone stores into it
  std::vector<int> ok(world_);
  return allgather(&one, ok.data(), sizeof one);
}

// Every rank frees its mailbox after all ranks are done storing into it
// (td_destroy, or a re-size in begin_run).
td_status CudaEngine::peer_release() {
  if (!mbox_) return TD_OK;
  CK(cudaStreamSynchronize(st_));
  if (tst_) CK(cudaStreamSynchronize(tst_));
  int one = 1;
  std::vector<int> all(world_);
  if (td_status e = allgather(&one, all.data(), sizeof one)) return e;
  for (auto& kv : peer_mbox_) cudaIpcCloseMemHandle(kv.second);
  peer_mbox_.clear();
  cudaFree(mbox_);
  mbox_ = nullptr;
  return TD_OK;
}

// ------------------------------------------------------------------ factory
td_status Engine::create(const td_model_shape& s, int n_stages, const td_options& o, Engine** out,
                         std::string* err) {
  auto* e = new CudaEngine();
  td_status st = e->init(s, n_stages, o);
  if (st != TD_OK) {
    *err = e->error;
    delete e;
    return st;
  }
  *out = e;
  return TD_OK;
}

}  // namespace tdp
