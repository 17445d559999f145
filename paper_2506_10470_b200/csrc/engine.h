// engine.h -- CUDA execution plane (distributed runtime).
//
// One Engine per process.  In single-process mode it executes every pipeline
// stage of every micro-batch on one device, in launch order on one stream
// (the stage hand-off is the fp32 residual buffer itself).  In multi-process
// mode (world_size > 1) the process executes only stage `rank` and exchanges
// the fp32 residual with its neighbours and the sampled tokens with stage 0
// over NCCL (engine_nccl.cu).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/tdpipe.h"
#include "controller.h"

namespace tdp {

struct HostReq {
  std::vector<int32_t> prompt;
  int32_t predicted = 1;
  int32_t max_new = 1;
};

struct KernelTiming {
  int64_t launches = 0;
  double ms = 0.0;
  double bytes = 0.0;
  double flops = 0.0;
  std::vector<double> launch_bytes;   // algorithmic bytes of every launch, in launch order
};

// One (micro-batch, stage) span of a timed td_run, ns from the run's first
// launch (CUDA events on the library stream), for td_write_trace.
struct TraceSpan {
  int64_t mid;
  char kind;
  int stage;
  int64_t a_ns, b_ns;
};

class Engine : public ExecHooks {
 public:
  virtual ~Engine() {}
  static td_status create(const td_model_shape& s, int n_stages, const td_options& o, Engine** out,
                          std::string* err);
  virtual int64_t kv_blocks() const = 0;
  virtual int64_t kv_bytes_per_block() const = 0;
  virtual int64_t weight_bytes_stage0() const = 0;
  virtual td_status upload(const std::vector<HostReq>& reqs) = 0;      // prompts -> device arena
  virtual bool uploaded() const = 0;
  virtual td_status begin_run(const std::vector<HostReq>& reqs, bool record_logits) = 0;
  virtual td_status end_run(td_run_stats* st) = 0;                       // waits for the GPU
  virtual td_status get_outputs(const std::vector<HostReq>& reqs, const std::vector<int>& n_out,
                                std::vector<std::vector<int32_t>>* out) = 0;
  virtual td_status get_logits(int64_t rid, std::vector<float>* out, int* n_steps) = 0;
  virtual td_status stage_forward(int stage, const td_batch& b, const void* in, void* out) = 0;
  virtual td_status kv_reset() = 0;
  virtual td_status profile(int b_max, int k_max, int ctx_len, std::vector<int64_t>* tdec,
                            std::vector<int64_t>* tpre) = 0;
  // logical [rows, cols] bf16 bits of F9 tensor `tid` (td_get_weight)
  virtual td_status get_weight(int tid, std::vector<uint16_t>* out, int64_t* rows, int64_t* cols) = 0;
  // td_bench_step: one synthetic micro-batch of this process's stages, timed
  // per kernel class (accumulators readable through get_timing)
  virtual td_status bench_step(bool prefill, int n, int len, int iters, double* step_ms, double* ideal_ms) = 0;
  // spans and (time ns, KV blocks in use) samples of the last timed td_run
  virtual void get_trace(std::vector<TraceSpan>* spans, std::vector<std::pair<int64_t, int64_t>>* kv) = 0;
  virtual void set_timing(bool on) = 0;
  virtual bool get_timing(const std::string& name, KernelTiming* t) = 0;
  std::string error;
};

}  // namespace tdp
