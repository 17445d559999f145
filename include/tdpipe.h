/*
 * tdpipe.h -- C ABI of the B200-native TD-Pipe hot path.
 *
 * TD-Pipe (arxiv 2506.10470): temporally-disaggregated pipeline-parallel LLM
 * inference.  The library owns a Llama-style model sharded by layer over
 * pipeline stages (§2.2.3 "PP splits a model layer-wise"),
 * a paged KV cache per stage, and the hierarchy controller (PAPER.md:295-314
 * §3.2) that alternates long prefill phases and long decode phases using
 * Alg.1, inter-batch work stealing and
 * the spatial-temporal intensity switch (Eq.1/Eq.2).
 *
 * Conventions
 *  - Every call returns td_status (0 = TD_OK, < 0 = error); no C++ exception
 *    crosses the ABI.  On error, td_last_error(ctx) holds a message; a failed
 *    td_create leaves its message in td_last_error(NULL) (per thread).
 *  - All pointers in signatures are HOST pointers unless stated otherwise;
 *    the library copies what it needs (caller keeps ownership).
 *  - A td_ctx must not be used by two caller threads at once.
 *  - Token ids are int32; activations crossing the ABI are fp32 row-major.
 *  - Device memory, streams, kernels and NCCL communicators are owned by the
 *    ctx and released by td_destroy.
 */
#ifndef TDPIPE_H_
#define TDPIPE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t td_status;
#define TD_OK 0
#define TD_EINVAL (-1)   /* bad argument / shape (e.g. n_stages > n_layers) */
#define TD_ENOMEM (-2)   /* weights or KV pool do not fit in HBM          */
#define TD_ECUDA (-3)    /* CUDA runtime / driver error, or no sm_100 device             */
#define TD_ENCCL (-4)    /* NCCL error (multi-process pipeline)                          */
#define TD_ERANGE (-5)   /* request too long for max_seq_len / KV pool; buffer too small */
#define TD_ESTATE (-6)   /* call not valid in the current state                          */

/* Scheduling policies.  TDPIPE = the paper's method (§3.3-§3.5); PPSB_* are the
 * naive phase-interleaved PP + separate-batching baselines:
 * PRIO issues a prefill whenever one is admissible, ALT alternates.  PPHB =
 * PP + hybrid batching with chunked prefill:
 * every micro-batch carries its engine's decode tokens plus prefill chunks up
 * to hb_tokens (reading R23). */
#define TD_POLICY_TDPIPE 0
#define TD_POLICY_PPSB_PRIO 1
#define TD_POLICY_PPSB_ALT 2
#define TD_POLICY_PPHB 3

/* Executors.  CUDA = the real sm_100a path.  NULL = controller only (no GPU
 * touched; micro-batches complete logically) -- used to test the scheduler. */
#define TD_EXEC_CUDA 0
#define TD_EXEC_NULL 1

/* Stage hand-off in the multi-process pipeline (one process per GPU).
 * PEER = the library's own peer-store path ("a single
 * point-to-point communication"): every rank exports one device "mailbox"
 * allocation through CUDA IPC; stage s stores its fp32 residual [T, d] straight
 * into stage s+1's receive ring over NVLink, the last stage stores (arena
 * position, token) pairs into stage 0's token ring, and readiness / slot reuse
 * is signalled with 32-bit sequence flags written and waited on by the GPU
 * streams themselves (stream memory operations; no host round trip, no SM
 * spinning).  Needs `allgather` (host all-gather used for the IPC handles, the
 * KV-capacity min and the profile-table max).  NCCL = ncclSend/ncclRecv on two
 * library-owned communicators (needs nccl_ids); kept as the baseline. */
#define TD_HANDOFF_PEER 0
#define TD_HANDOFF_NCCL 1

/* Host all-gather across the ranks of a multi-process pipeline: every rank
 * passes `bytes` bytes in `send`; on return `recv` holds world_size * bytes,
 * rank r's contribution at offset r * bytes.  Returns 0 on success.  Provided
 * by the caller (e.g. torch.distributed over gloo); called only from td_create,
 * td_profile, td_run (when the request set needs larger hand-off slots than
 * the mailboxes hold -- every rank decides identically) and td_destroy, on the
 * calling thread, in the same order on every rank. */
typedef int32_t (*td_allgather_fn)(void* user, const void* send, void* recv, size_t bytes);

/* Model shape (Llama-style pre-norm decoder; Table 2). */
typedef struct td_model_shape {
  int32_t n_layers;
  int32_t d_model;
  int32_t n_heads;
  int32_t n_kv_heads;   /* GQA: must divide n_heads */
  int32_t d_ffn;
  int32_t vocab;
  float rope_theta;     /* 1e4: rotate-half RoPE */
  float rms_eps;        /* 1e-5 */
  int32_t max_seq_len;  /* prompt + generated tokens per request */
} td_model_shape;

typedef struct td_options {
  int32_t executor;             /* TD_EXEC_CUDA | TD_EXEC_NULL                         */
  int32_t device;               /* CUDA device of this process (every stage it runs)   */
  int32_t block_size;           /* KV block (page) size in tokens, B (default 16)      */
  int64_t kv_blocks;            /* C; 0 = fill HBM (min over stages)                   */
  double hbm_reserve_frac;      /* HBM kept free when kv_blocks = 0 (default 0.06)     */
  int32_t prefill_token_budget; /* tokens per prefill micro-batch (2048)  */
  int32_t max_batch_seqs;       /* max sequences per micro-batch (default 1024)        */
  int32_t fp_stride;            /* futurePoints stride (32)              */
  int32_t fp_horizon;           /* futurePoints horizon (1024)           */
  int32_t policy;               /* TD_POLICY_*                                         */
  int32_t steal;                /* inter-batch work stealing on/off     */
  int32_t alg1_check_before_launch; /* 0 = verbatim Alg.1 (launch precedes check)     */
  int32_t eq2_bubble_scale;     /* sigma in Eq.2's bubble: 1 = verbatim, S-1 = depth   */
  uint64_t weight_seed;         /* F9 counter-based weight recipe seed                 */
  const char* profile_csv;      /* frozen profile table "D,b,ns"/"P,k,ns"; NULL = none */
  int32_t log_decisions;        /* keep the decision log (td_get_log)                  */
  int32_t record_logits;        /* keep fp32 logits of every generated token           */
  /* multi-process pipeline (one process per GPU, SPMD runtime PAPER.md:310-314) */
  int32_t world_size;           /* 1 = single process                                  */
  int32_t rank;                 /* this process's stage                                */
  const void* nccl_ids;         /* 2 x 128-byte ncclUniqueId (fwd, bwd) from td_nccl_ids */
  /* ablations of the paper's §4.4 (0 = the paper's method) */
  int32_t p2d_kv_permille;      /* P->D once allocated KV >= x/1000 of C */
  int32_t d2p_finish_permille;  /* D->P once x/1000 of the decode cohort finished */
  int32_t hb_tokens;            /* PPHB: tokens per hybrid micro-batch (default 512)   */
  /* multi-process stage hand-off */
  int32_t handoff;              /* TD_HANDOFF_PEER (default) | TD_HANDOFF_NCCL          */
  td_allgather_fn allgather;    /* PEER: host all-gather (see td_allgather_fn)          */
  void* allgather_user;         /* opaque first argument of allgather                  */
  /* roofline accounting (td_run_stats.ideal_ns): peaks of this device; 0 = off */
  double hbm_peak_gbs;          /* HBM bandwidth, GB/s (measured copy bandwidth)        */
  double tc_peak_tflops;        /* dense bf16 tensor-core TFLOP/s                       */
  /* execution plan of decode micro-batches of <= 128 tokens (same results up to
     fp32 summation order) */
  int32_t decode_chain;         /* 0 (default): one kernel per GEMM / reduction (PDL);
                                   1: one persistent kernel per layer for the weight
                                   GEMMs + reductions, attention separate (measured
                                   1-10 % slower: profiles/r2/chain/)               */
} td_options;

typedef struct td_run_stats {
  int64_t n_requests;
  int64_t prompt_tokens;        /* prompt tokens processed (incl. recompute)           */
  int64_t generated_tokens;
  int64_t makespan_ns;          /* first prefill launch -> last return  */
  double gen_tokens_per_s;
  double total_tokens_per_s;    /* (prompt + generated) / makespan      */
  double bubble_frac;           /* 1 - sum_s busy_s / (S * makespan)                   */
  int64_t n_microbatches;
  int64_t n_prefill_mb;
  int64_t n_decode_mb;
  int64_t n_p2d;
  int64_t n_d2p;
  int64_t n_stolen;
  int64_t n_evicted;
  int64_t gpu_launches;         /* kernels this process launched during td_run         */
  int64_t h2d_bytes;
  int64_t d2h_bytes;
  int64_t busy_ns[8];           /* per-stage busy time (first 8 stages)                */
  /* Speed-of-light accounting of this process's micro-batches:
   * per micro-batch, algorithmic HBM bytes (every weight of its layers once,
   * every context token's K and V per layer, the new K/V written) and FLOPs
   * (2 x tokens x weights + causal attention); ideal_ns = sum over micro-batches
   * of max(bytes / hbm_peak, flops / tc_peak) (0 if the peaks are not set).
   * ideal_ns / makespan_ns is the whole job's roofline fraction. */
  double ideal_ns;
  double alg_bytes;
  double alg_flops;
} td_run_stats;

/* A single micro-batch for td_stage_forward (testing entry point). */
#define TD_BATCH_PREFILL 0
#define TD_BATCH_DECODE 1
typedef struct td_batch {
  int32_t kind;                 /* TD_BATCH_PREFILL | TD_BATCH_DECODE                  */
  int32_t n_seqs;
  const int32_t* seq_slot;      /* [n] request slot (0 .. max_requests-1), KV owner    */
  const int32_t* q_start;       /* [n] absolute position of the first new token        */
  const int32_t* q_len;         /* [n] new tokens (prefill: L, or a chunk continuing at
                                   q_start > 0 over the paged prefix; decode: 1)        */
  const int32_t* block_table;   /* [n * max_blocks] physical KV block ids              */
  int32_t max_blocks;
} td_batch;

/* Fill `o` with defaults (executor CUDA, device 0, B=16, budget 2048, ...). */
void td_default_options(td_options* o);

/* Create a context: validate the shape (n_stages <= n_layers, SPEC.md:118;
 * n_kv_heads | n_heads; head_dim in {16,32,64,128}), partition layers
 * (balanced, remainder to earlier stages), allocate and
 * hash-initialise the weights on device, size the paged KV pool.
 * Errors: TD_EINVAL, TD_ENOMEM, TD_ECUDA, TD_ENCCL. */
td_status td_create(const td_model_shape* shape, int32_t n_stages, const td_options* opts,
                    struct td_ctx** out);
void td_destroy(struct td_ctx* ctx);
/* Message of the last error on `ctx`; ctx == NULL: the message of the last
 * failed td_create on the calling thread ("" if none).  The pointer stays
 * valid until the next call on the same ctx (or thread, for NULL). */
const char* td_last_error(const struct td_ctx* ctx);

/* Submit one request (offline request set).  The prompt is
 * copied.  predicted_len < 1 is clamped to 1; max_new_tokens
 * (>= 1) is the stop length (EOS is disabled for random weights).
 * Returns the request id (submission order = FIFO order) or a negative
 * td_status: TD_ERANGE if n_prompt + max_new_tokens > max_seq_len or the
 * request alone exceeds the KV pool. */
int64_t td_submit(struct td_ctx* ctx, const int32_t* prompt, int32_t n_prompt,
                  int32_t predicted_len, int32_t max_new_tokens);

/* Stage the submitted prompts in device memory (H2D) so that td_run starts
 * with inputs resident in HBM.  Optional: td_run calls it if needed. */
td_status td_upload(struct td_ctx* ctx);

/* Run every submitted request to completion (blocks).  Generated tokens stay
 * on device until td_get_output.  st may be NULL. */
td_status td_run(struct td_ctx* ctx, td_run_stats* st);

/* Generated tokens of request `id` into caller buffer `buf` (capacity `cap`);
 * *n = number of tokens.  TD_ERANGE if cap < *n (n still set). */
td_status td_get_output(struct td_ctx* ctx, int64_t id, int32_t* buf, int32_t cap, int32_t* n);

/* All outputs at once (one D2H copy): out[id * stride + j] for j < n_out[id],
 * id < number of submitted requests.  `out` holds n_rows * stride int32 and
 * `n_out` n_rows int32, both caller-owned.  TD_ERANGE (nothing written) if
 * n_rows < the number of submitted requests or stride < the longest output. */
td_status td_get_outputs(struct td_ctx* ctx, int32_t* out, int32_t n_rows, int32_t stride, int32_t* n_out);

/* fp32 logits [n_steps, vocab] of request `id` (requires record_logits). */
td_status td_get_logits(struct td_ctx* ctx, int64_t id, float* buf, int64_t cap, int32_t* n_steps);

/* Forget all submitted requests (outputs, logs) and clear KV; weights kept. */
td_status td_reset(struct td_ctx* ctx);

/* Run ONE pipeline stage on one micro-batch (testing):
 * in  = stage 0: int32 tokens [T]; else fp32 residual [T, d_model]
 * out = last stage: fp32 logits [n_seqs, vocab] of each sequence's last token;
 *       else fp32 residual [T, d_model]
 * T = sum(q_len).  Reads/writes the stage's KV pool through block_table, so a
 * DECODE call follows a PREFILL into the same blocks.  Host pointers. */
td_status td_stage_forward(struct td_ctx* ctx, int32_t stage, const td_batch* b,
                           const void* in, void* out);

/* Zero every stage's KV pool. */
td_status td_kv_reset(struct td_ctx* ctx);

/* Measure per-stage decode-step ns for b = 1..b_max at context ctx_len and
 * prefill ns for k = 1..k_max tokens (sampled grid, linearly interpolated),
 * write the dense CSV read through td_options.profile_csv (§3.5 "we profile
 * the execution time") and load it into this ctx. */
td_status td_profile(struct td_ctx* ctx, const char* out_csv, int32_t b_max, int32_t k_max,
                     int32_t ctx_len);

/* Load a profile CSV into this ctx (replaces the current table). */
td_status td_load_profile(struct td_ctx* ctx, const char* csv);

/* Decision log of the last td_run, '\n'-separated.
 * Copies min(cap, need) bytes; *need = full length (without NUL). */
td_status td_get_log(struct td_ctx* ctx, char* buf, size_t cap, size_t* need);

/* Timed replay of the whole schedule on an S-stage pipeline model (no GPU
 * work): every micro-batch occupies each stage for the frozen profile time
 * (Tpre[tokens] or Tdec[batch], per-stage), stages are FIFO servers, a return
 * reaches the controller host_return_ns after the last stage.  Produces the
 * same decision log as td_run and fills makespan / tokens/s / bubble /
 * busy_ns -- used to project multi-GPU TD-Pipe vs PP+SB from measured
 * per-stage B200 times.  Needs a loaded profile table. */
td_status td_simulate(struct td_ctx* ctx, td_run_stats* st, int64_t host_return_ns);

/* Write the last td_simulate run -- or the last td_run executed with timing
 * on (td_set_timing(ctx, 1): spans are CUDA events on the library stream, ns
 * from the run's first launch) -- as a Chrome trace (chrome://tracing /
 * Perfetto JSON): one complete event per (micro-batch, stage) on thread =
 * stage, plus a "kv_used_blocks" counter track sampled at every launch (the
 * KV-usage timeline of PAPER.md:580-585 fig:memory_usage). */
td_status td_write_trace(struct td_ctx* ctx, const char* path);

/* Model / pool facts: kv_blocks, layers of `stage`, weight bytes per stage. */
td_status td_info(struct td_ctx* ctx, int64_t* kv_blocks, int32_t* n_stages,
                  int64_t* weight_bytes_stage0, int64_t* kv_bytes_per_block);

/* Per-kernel timing over the last td_run (CUDA events on the launching
 * stream, measured when td_options.executor = CUDA and timing is enabled with
 * td_set_timing(ctx, 1)).  name = kernel class ("decode_attn", "gemm_qkv", ...). */
td_status td_set_timing(struct td_ctx* ctx, int32_t on);
td_status td_get_timing(struct td_ctx* ctx, const char* name, int64_t* launches,
                        double* total_ms, double* bytes, double* flops);

/* Stage step benchmark (testing / measurement): one synthetic micro-batch
 * through every stage this process holds, `iters` times after 2 warm-up
 * passes -- kind DECODE: n_seqs sequences at context `len` (each decodes the
 * token at position len-1, pages scattered over the pool); kind PREFILL:
 * n_seqs prompts of `len` tokens.  *step_us = mean device microseconds of one
 * pass (CUDA events on the library stream), *ideal_us (nullable) = its speed
 * of light max(bytes / hbm_peak_gbs, FLOPs / tc_peak_tflops) with the
 * td_run_stats accounting (0 if the peaks are unset).  Per-kernel timing of
 * the timed passes is left in the td_get_timing accumulators.  Clears the KV
 * pool.  TD_ERANGE if n_seqs * ceil(len/16) > kv_blocks. */
td_status td_bench_step(struct td_ctx* ctx, int32_t kind, int32_t n_seqs, int32_t len, int32_t iters,
                        double* step_us, double* ideal_us);

/* Algorithmic bytes of every launch of kernel class `name` accumulated by
 * per-kernel timing (td_set_timing), in launch order -- lets a DRAM-traffic
 * capture of a subset of a run's launches (ncu) be compared with exactly the
 * same launches' algorithmic bytes.  *n = number of launches; copies
 * min(cap, n) values into `out` (nullable: size query).  TD_ERANGE if cap < n
 * and out != NULL. */
td_status td_get_launch_bytes(struct td_ctx* ctx, const char* name, double* out, int64_t cap, int64_t* n);

/* Kernel unit test (testing only): out[T, N] fp32 = A[T, K] . W[N, K]^T with
 * A, W given as bf16 bit patterns (host), on the tcgen05 kernels: impl 0
 * packs W into the tile-packed layout the engine uses, impl 2 reads row-major
 * W through a TMA descriptor; splits > 1 exercises the split-K reduction
 * (T > 128 with impl 0 and splits == 1: the persistent token-major prefill
 * kernel); impl 4 = the token-major kernel with `splits` K splits (T > 128;
 * the engine's path for 129+-token decode micro-batches); impl 5 = the
 * persistent decode chain (decode_chain.cu) on one GEMM op whose weight tiles
 * are reduced into a zeroed residual (T <= 128, N % 128 == 0).  Runs on `device`,
 * allocates and frees its own buffers, synchronous.  TD_EINVAL for any other
 * impl. */
td_status td_test_gemm(int32_t device, const uint16_t* A, const uint16_t* W, int32_t T, int32_t N, int32_t K,
                       int32_t impl, int32_t splits, float* out);

/* The persistent decode chain (decode_chain.cu) on one MLP block (testing
 * only): a = bf16(RMSNorm(x0) * g), h = bf16(silu(Wgu[2j] . a) * (Wgu[2j+1] . a)),
 * x = x0 + Wd . h -- the chain ops residual + norm, GEMM, SwiGLU, GEMM,
 * residual with grid barriers between them.  x0 [T, d] fp32;
 * g [d], Wgu [2F, d] (gate / up rows interleaved), Wd [d, F] bf16 bit
 * patterns; outputs a [T, d] and h [T, F] (bf16 bits) and x [T, d] fp32,
 * host buffers owned by the caller.  T in [1, 128], d and F multiples of 64;
 * TD_EINVAL otherwise.  Allocates and frees its own device buffers, synchronous. */
td_status td_test_chain_mlp(int32_t device, const float* x0, const uint16_t* g, const uint16_t* Wgu,
                            const uint16_t* Wd, int32_t T, int32_t d, int32_t F, float eps, uint16_t* a_out,
                            uint16_t* h_out, float* x_out);

/* GEMM timing sweep (testing only): average device microseconds per call of
 * the tcgen05 GEMM on [T, K] x [N, K]^T (tile-packed weights, fp32 output),
 * cycling over `copies` weight buffers so that the weights stream from HBM;
 * splits = split-K count (1 = none); decode = 1 selects the swap-AB decode
 * kernel (weight rows x token tiles; 3 / 4: with 64- / 32-token tiles),
 * decode = 2 the token-major kernel with `splits` K splits (reduction +
 * epilogue launch included). */
td_status td_bench_gemm(int32_t device, int32_t T, int32_t N, int32_t K, int32_t splits, int32_t decode,
                        int32_t iters, int32_t copies, float* us_per_call);

/* Decode-attention timing sweep (testing only): average device microseconds
 * per decode-attention launch for n sequences of context lengths ctx[n] (host),
 * H query / Hkv kv heads of size hd, pages scattered through a pool rotated
 * over enough copies (<= 400 MiB) that K/V stream from HBM, launched with
 * the engine's plan (split = 0) or with `split`-token splits (a multiple of
 * 16, >= 32); impl 0 = the engine's kernel choice, 1 = the SIMT kernel,
 * 2 = the tensor-core kernel (hd 64 / 128).  K/V, q are zeros (timing only). */
td_status td_bench_attn(int32_t device, int32_t n, const int32_t* ctx, int32_t H, int32_t Hkv, int32_t hd,
                        int32_t iters, int32_t split, int32_t impl, float* us_per_call);

/* Weight read-back (testing only): the bf16 bit patterns of F9 tensor
 * `tensor_id` (SURVEY.md §8(c) F9 enumeration: 0 = embedding [V, d]; layer l:
 * 1+9l+{0 g1 [d], 1 Wq [H hd, d], 2 Wk [Hkv hd, d], 3 Wv [Hkv hd, d],
 * 4 Wo [d, H hd], 5 g2 [d], 6 Wg [F, d], 7 Wu [F, d], 8 Wd [d, F]};
 * 1+9L = final norm [d]; 2+9L = LM head [V, d]) in its LOGICAL row-major
 * [rows, cols] layout, undoing the device's tile packing and the RoPE-pair /
 * gate-up row interleaving.  Copies min(cap, rows*cols) elements into `out`
 * (caller-owned); *rows / *cols are always set.  TD_EINVAL if the tensor is
 * not held by this process (another rank's stage), TD_ERANGE if cap is too
 * small.  Lets a test check the device weights bit for bit against the
 * oracle's independent implementation of the recipe. */
td_status td_get_weight(struct td_ctx* ctx, int32_t tensor_id, uint16_t* out, int64_t cap, int64_t* rows,
                        int64_t* cols);

/* Generate the two ncclUniqueIds (256 bytes) rank 0 shares with all ranks. */
td_status td_nccl_ids(void* out256);

#ifdef __cplusplus
}
#endif
#endif /* TDPIPE_H_ */
