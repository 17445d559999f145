// controller.h -- TD-Pipe hierarchy controller (control plane), host C++.
//
// The centralized engine of PAPER.md:297-308 (§3.2.1): batch scheduling "based
// on memory capacity, request status, and profiling results".  Decisions are a
// function of the logical event sequence only (micro-batch returns arrive in
// launch order because every stage is FIFO), so every rank of a multi-process
// pipeline runs an identical replica and no control messages cross the wire.
//
// Steps implemented (readings R1-R20):
//   S2/S3  Alg.1 UpdateUsage / CheckSwitch, block form
//   S4     SchedulePrefill loop, eager
//   S5     decode batches = #GPUs, equal sizes
//   S6     return processing; S7 work stealing
//   S8     recompute eviction
//   S9/S10 Eq.1 / Eq.2 and the switch rule
//   S11    naive PP+SB baselines; PP+HB hybrid batching + chunked prefill [R23];
//          S12 decision log
#pragma once
#include <cstdint>
#include <deque>
#include <queue>
#include <set>
#include <string>
#include <vector>

namespace tdp {

enum Policy { kTDPipe = 0, kPPSBPrio = 1, kPPSBAlt = 2, kPPHB = 3 };

struct SchedOptions {
  int W = 1;                 // pipeline stages = decode batches
  int B = 16;                // KV block size
  int64_t C = 1 << 30;       // KV capacity in blocks (min over stages)
  int budget = 2048;         // prefill token budget
  int max_seqs = 1 << 30;
  int fp_stride = 32;
  int fp_horizon = 1024;
  int policy = kTDPipe;
  int steal = 1;
  int check_before_launch = 0;
  int eq2_bubble_scale = 1;
  int p2d_kv_permille = 0;      // ablation A22: KV-occupancy-ratio P->D switch
  int d2p_finish_permille = 0;  // ablation A23: request-finish-ratio D->P switch
  int hb_tokens = 512;          // PP+HB: tokens per hybrid micro-batch [R23]
};

struct Req {
  int rid = 0;
  int n_prompt = 0;
  int L = 0;      // current prompt length (incl. recomputed tokens)
  int P = 1;      // predicted output length
  int N = 1;      // stop length from this admission
  int g = 0;      // generated since (re)admission
  int d = 0;      // decode steps returned since (re)admission
  int64_t adm = -1;
  int n_out = 0;  // generated in total
  std::vector<int32_t> blocks;
  bool in_flight = false;
  bool done = false;
  int slot = -1;
  int64_t evict_key = -1;
  int pf = 0;     // PP+HB: prompt tokens prefilled so far
};

struct MicroBatch {
  int64_t mid = 0;
  char kind = 'P';   // 'P', 'D' or 'H' (PP+HB: decode members first, then prefill chunks)
  int slot = -1;
  int epoch = 0;
  std::vector<int> members, q_start, q_len;
};

// Execution plane hook: the controller calls launch() for every micro-batch in
// global launch order and returned() when it processes that micro-batch's
// return (logically, in the same order).
struct ExecHooks {
  virtual ~ExecHooks() {}
  virtual int launch(const MicroBatch& mb, const std::vector<Req>& reqs) = 0;
  virtual int returned(const MicroBatch& mb) { (void)mb; return 0; }
};

struct SchedStats {
  int64_t p2d = 0, d2p = 0, stolen = 0, evicted = 0, refilled = 0;
  int64_t n_mb = 0, n_prefill = 0, n_decode = 0, prompt_tokens = 0;
};

class Controller {
 public:
  Controller(const SchedOptions& o, const std::vector<Req>& reqs, const std::vector<int64_t>& tdec,
             const std::vector<int64_t>& tpre, bool keep_log);
  // Runs the whole offline job; returns 0 or the first non-zero hook status.
  int run(ExecHooks* ex);
  const std::string& log() const { return log_; }
  const std::vector<Req>& reqs() const { return reqs_; }
  const SchedStats& stats() const { return stats_; }
  std::string error;

 private:
  struct Slot {
    int idx;
    std::vector<int> members;
    bool launched = false, inflight = false, retired = false;
  };

  // utils
  void emit(const std::string& s);
  void emit_ids(const char* head, const std::vector<int64_t>& nums);
  bool pending_empty() const { return pending_evicted_.empty() && pending_fresh_.empty(); }
  std::vector<int> pending_list() const;
  int64_t tdec(int64_t b) const;
  int64_t tpre(int64_t k) const;
  // Alg.1
  void update_usage(std::vector<int64_t>& U, const Req& r) const;
  std::vector<int64_t> rebuild_usage() const;
  bool check_switch(const std::vector<int64_t>& U) const;
  int64_t max_usage(const std::vector<int64_t>& U) const;
  std::vector<int> form_prefill_batch(const std::vector<int>& pending, int64_t limit) const;
  void add_usage_fresh(std::vector<int64_t>& U, const std::vector<int>& batch) const;
  void pop_pending(const std::vector<int>& batch);
  int prefill_phase();
  std::vector<int64_t> dry_run_prefill() const;
  int launch_prefill(const std::vector<int>& batch, int slot);
  // decode
  void form_decode();
  int try_launch_formed();
  void evict(int rid);
  int64_t decode_need(const std::vector<int>& members) const;
  void ensure_blocks(Slot& sl);
  int launch_decode(Slot& sl);
  void retire(Slot& sl);
  void steal_refill(Slot& sl);
  bool decide_switch(Slot& sl);
  void finish(Req& r);
  int on_return(const MicroBatch& mb);
  int run_tdpipe();
  int run_baseline();
  int run_hybrid();
  // allocator (lowest free id first)
  int64_t free_blocks() const { return opt_.C - watermark_ + (int64_t)free_heap_.size(); }
  int32_t alloc_one();
  void release(const std::vector<int32_t>& b);

  SchedOptions opt_;
  std::vector<Req> reqs_;
  std::vector<int64_t> tdec_, tpre_;
  bool keep_log_;
  std::string log_;
  std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> free_heap_;
  int64_t watermark_ = 0;
  std::vector<int> pending_evicted_;
  std::deque<int> pending_fresh_;
  std::set<int> live_;
  std::deque<MicroBatch> inflight_;
  std::vector<Slot> slots_;
  std::deque<int> pool_;
  int epoch_ = 0;
  int64_t adm_counter_ = 0;
  int64_t mb_counter_ = 0;
  std::vector<int> fps_;
  int64_t ctx_rep_ = 1, b_mem_ = 1, Bp_ = 1;
  int64_t cohort_n_ = 0, cohort_done_ = 0;
  ExecHooks* ex_ = nullptr;
  SchedStats stats_;
};

}  // namespace tdp
