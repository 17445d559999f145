// api.cpp -- the C ABI (include/tdpipe.h).  Argument validation, request
// bookkeeping and the glue between the controller (control plane) and the
// CUDA engine (execution plane).  No torch types cross this boundary.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/tdpipe.h"
#include "controller.h"
#include "engine.h"

using namespace tdp;

struct td_ctx {
  td_model_shape shape{};
  int n_stages = 1;
  td_options opt{};
  std::string profile_path;
  std::string err;
  std::vector<HostReq> reqs;
  std::vector<int64_t> tdec, tpre;
  std::string log;
  std::vector<int> n_out;
  bool have_run = false;
  int64_t kv_blocks = 0;
  std::unique_ptr<Engine> engine;
  std::vector<std::vector<int32_t>> outputs;   // cached after first td_get_output
  bool outputs_cached = false;
  // last td_simulate: (mid, kind, stage, start_ns, end_ns) and (t_ns, used blocks)
  struct Span { int64_t mid; char kind; int stage; int64_t a, b; };
  std::vector<Span> spans;
  std::vector<std::pair<int64_t, int64_t>> kv_samples;
};

static thread_local std::string g_create_err;   // td_last_error(NULL)

static td_status create_fail(td_status st, const std::string& m) {
  g_create_err = m;
  return st;
}

static td_status fail(td_ctx* c, td_status st, const std::string& m) {
  if (c) c->err = m;
  return st;
}

extern "C" void td_default_options(td_options* o) {
  std::memset(o, 0, sizeof *o);
  o->executor = TD_EXEC_CUDA;
  o->device = 0;
  o->block_size = 16;
  o->kv_blocks = 0;
  o->hbm_reserve_frac = 0.06;
  o->prefill_token_budget = 2048;
  o->max_batch_seqs = 1024;
  o->fp_stride = 32;
  o->fp_horizon = 1024;
  o->policy = TD_POLICY_TDPIPE;
  o->steal = 1;
  o->alg1_check_before_launch = 0;
  o->eq2_bubble_scale = 1;
  o->weight_seed = 0x5EED7DULL;
  o->profile_csv = nullptr;
  o->log_decisions = 1;
  o->record_logits = 0;
  o->world_size = 1;
  o->rank = 0;
  o->nccl_ids = nullptr;
  o->p2d_kv_permille = 0;
  o->d2p_finish_permille = 0;
  o->hb_tokens = 512;
  o->handoff = TD_HANDOFF_PEER;
  o->allgather = nullptr;
  o->allgather_user = nullptr;
  o->hbm_peak_gbs = 0.0;
  o->tc_peak_tflops = 0.0;
  o->decode_chain = 0;
}

static bool read_profile(const std::string& path, std::vector<int64_t>* tdec, std::vector<int64_t>* tpre,
                         std::string* err) {
  std::ifstream f(path);
  if (!f) { *err = "cannot open profile csv " + path; return false; }
  std::vector<std::pair<int64_t, int64_t>> d, p;
  std::string line;
  while (std::getline(f, line)) {
    if (line.empty() || line[0] == '#') continue;
    char kind = 0;
    long long i = 0, ns = 0;
    if (sscanf(line.c_str(), "%c,%lld,%lld", &kind, &i, &ns) != 3 || i < 1) { *err = "bad csv line: " + line; return false; }
    (kind == 'D' ? d : p).push_back({i, ns});
  }
  if (d.empty() || p.empty()) { *err = "profile csv needs D and P rows"; return false; }
  int64_t bm = 0, km = 0;
  for (auto& x : d) bm = std::max(bm, x.first);
  for (auto& x : p) km = std::max(km, x.first);
  tdec->assign(bm + 1, 0);
  tpre->assign(km + 1, 0);
  for (auto& x : d) (*tdec)[x.first] = x.second;
  for (auto& x : p) (*tpre)[x.first] = x.second;
  return true;
}

extern "C" td_status td_create(const td_model_shape* s, int32_t n_stages, const td_options* opts, td_ctx** out) {
  if (!s || !out) return TD_EINVAL;
  *out = nullptr;
  auto c = std::make_unique<td_ctx>();
  c->shape = *s;
  c->n_stages = n_stages;
  if (opts) c->opt = *opts; else td_default_options(&c->opt);
  if (c->opt.profile_csv) c->profile_path = c->opt.profile_csv;
  c->opt.profile_csv = nullptr;
  const auto& m = c->shape;
  g_create_err.clear();
  if (n_stages < 1 || n_stages > m.n_layers) return create_fail(TD_EINVAL, "n_stages must be in [1, n_layers]");
  if (m.n_heads <= 0 || m.n_kv_heads <= 0 || m.n_heads % m.n_kv_heads)
    return create_fail(TD_EINVAL, "n_kv_heads must divide n_heads");
  if (m.d_model <= 0 || m.d_model % m.n_heads) return create_fail(TD_EINVAL, "n_heads must divide d_model");
  const int hd = m.d_model / m.n_heads;
  if (hd != 16 && hd != 32 && hd != 64 && hd != 128) return create_fail(TD_EINVAL, "head_dim must be 16/32/64/128");
  if (m.d_model % 64 || m.d_ffn % 64 || m.d_ffn <= 0 || m.vocab <= 0 || m.max_seq_len <= 0)
    return create_fail(TD_EINVAL, "d_model and d_ffn must be multiples of 64; vocab, max_seq_len > 0");
  if (c->opt.block_size < 1) return create_fail(TD_EINVAL, "block_size < 1");
  if (c->opt.executor != TD_EXEC_NULL && c->opt.block_size != 16)
    return create_fail(TD_EINVAL, "the CUDA executor uses 16-token KV pages (block_size 16)");
  if (c->opt.prefill_token_budget < 1 || c->opt.max_batch_seqs < 1 || c->opt.fp_stride < 1)
    return create_fail(TD_EINVAL, "prefill_token_budget, max_batch_seqs and fp_stride must be >= 1");
  if (c->opt.world_size < 1 || c->opt.rank < 0 || c->opt.rank >= c->opt.world_size)
    return create_fail(TD_EINVAL, "rank must be in [0, world_size)");
  if (c->opt.world_size > 1 && c->opt.world_size != n_stages)
    return create_fail(TD_EINVAL, "world_size > 1 needs world_size == n_stages (one stage per process)");
  if (c->opt.handoff != TD_HANDOFF_PEER && c->opt.handoff != TD_HANDOFF_NCCL)
    return create_fail(TD_EINVAL, "unknown handoff");
  if (c->opt.executor != TD_EXEC_NULL && c->opt.world_size > 1 && c->opt.handoff == TD_HANDOFF_PEER &&
      !c->opt.allgather)
    return create_fail(TD_EINVAL, "TD_HANDOFF_PEER needs the allgather callback");
  if (!c->profile_path.empty()) {
    std::string e;
    if (!read_profile(c->profile_path, &c->tdec, &c->tpre, &e)) return create_fail(TD_EINVAL, e);
  }
  if (c->opt.executor == TD_EXEC_NULL) {
    c->kv_blocks = c->opt.kv_blocks > 0 ? c->opt.kv_blocks : (int64_t)1 << 30;
  } else {
    Engine* e = nullptr;
    std::string err;
    td_status st = Engine::create(c->shape, n_stages, c->opt, &e, &err);
    if (st != TD_OK) return create_fail(st, err);
    c->engine.reset(e);
    c->kv_blocks = e->kv_blocks();
  }
  *out = c.release();
  return TD_OK;
}

extern "C" void td_destroy(td_ctx* c) { delete c; }

extern "C" const char* td_last_error(const td_ctx* c) { return c ? c->err.c_str() : g_create_err.c_str(); }

extern "C" int64_t td_submit(td_ctx* c, const int32_t* prompt, int32_t n_prompt, int32_t predicted_len,
                             int32_t max_new_tokens) {
  if (!c || !prompt || n_prompt < 1 || max_new_tokens < 1) return fail(c, TD_EINVAL, "bad request");
  if ((int64_t)n_prompt + max_new_tokens > c->shape.max_seq_len)
    return fail(c, TD_ERANGE, "n_prompt + max_new_tokens > max_seq_len");
  const int64_t B = c->opt.block_size;
  if ((n_prompt + max_new_tokens + B - 1) / B > c->kv_blocks) return fail(c, TD_ERANGE, "request exceeds the KV pool");
  for (int i = 0; i < n_prompt; ++i)
    if (prompt[i] < 0 || prompt[i] >= c->shape.vocab) return fail(c, TD_EINVAL, "token id out of range");
  HostReq r;
  r.prompt.assign(prompt, prompt + n_prompt);
  r.predicted = std::max(predicted_len, 1);
  r.max_new = max_new_tokens;
  c->reqs.push_back(std::move(r));
  c->have_run = false;
  return (int64_t)c->reqs.size() - 1;
}

extern "C" td_status td_upload(td_ctx* c) {
  if (!c) return TD_EINVAL;
  if (!c->engine) return TD_OK;
  td_status st = c->engine->upload(c->reqs);
  if (st) c->err = c->engine->error;
  return st;
}

extern "C" td_status td_run(td_ctx* c, td_run_stats* st) {
  if (!c) return TD_EINVAL;
  SchedOptions so;
  so.W = c->n_stages;
  so.B = c->opt.block_size;
  so.C = c->kv_blocks;
  so.budget = c->opt.prefill_token_budget;
  so.max_seqs = c->opt.max_batch_seqs;
  so.fp_stride = c->opt.fp_stride;
  so.fp_horizon = c->opt.fp_horizon;
  so.policy = c->opt.policy;
  so.steal = c->opt.steal;
  so.check_before_launch = c->opt.alg1_check_before_launch;
  so.eq2_bubble_scale = c->opt.eq2_bubble_scale;
  so.p2d_kv_permille = c->opt.p2d_kv_permille;
  so.d2p_finish_permille = c->opt.d2p_finish_permille;
  so.hb_tokens = c->opt.hb_tokens;
  if (so.policy == TD_POLICY_TDPIPE && c->tdec.size() < 2 && c->reqs.size() > 0) {
    // without a profile table Eq.1/Eq.2 cannot be evaluated: use a flat one
    // (never switches before the queue drains is NOT implied; document it)
    return fail(c, TD_ESTATE, "TDPIPE policy needs a profile table (profile_csv or td_profile)");
  }
  std::vector<Req> reqs(c->reqs.size());
  for (size_t i = 0; i < c->reqs.size(); ++i) {
    Req& r = reqs[i];
    r.rid = (int)i;
    r.n_prompt = (int)c->reqs[i].prompt.size();
    r.L = r.n_prompt;
    r.P = c->reqs[i].predicted;
    r.N = c->reqs[i].max_new;
  }
  Controller ctl(so, reqs, c->tdec, c->tpre, c->opt.log_decisions != 0);
  td_status rc = TD_OK;
  auto t0 = std::chrono::steady_clock::now();
  if (c->engine) {
    rc = c->engine->begin_run(c->reqs, c->opt.record_logits != 0);
    if (rc) return fail(c, rc, c->engine->error);
  }
  int crc = ctl.run(c->engine.get());
  if (crc) {
    if (c->engine) { td_run_stats tmp{}; c->engine->end_run(&tmp); }
    return fail(c, crc < 0 ? crc : TD_ECUDA, ctl.error.empty() && c->engine ? c->engine->error : ctl.error);
  }
  td_run_stats s{};
  if (c->engine) {
    rc = c->engine->end_run(&s);
    if (rc) return fail(c, rc, c->engine->error);
  } else {
    s.makespan_ns = (int64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                        std::chrono::steady_clock::now() - t0).count();
  }
  c->log = ctl.log();
  if (c->engine) {   // a timed run leaves its CUDA-event spans + KV timeline for td_write_trace
    std::vector<TraceSpan> sp;
    std::vector<std::pair<int64_t, int64_t>> kv;
    c->engine->get_trace(&sp, &kv);
    if (!sp.empty()) {
      c->spans.clear();
      for (const auto& x : sp) c->spans.push_back({x.mid, x.kind, x.stage, x.a_ns, x.b_ns});
      c->kv_samples = kv;
    }
  }
  c->n_out.assign(c->reqs.size(), 0);
  int64_t gen = 0;
  for (size_t i = 0; i < c->reqs.size(); ++i) { c->n_out[i] = ctl.reqs()[i].n_out; gen += c->n_out[i]; }
  c->have_run = true;
  c->outputs_cached = false;
  const auto& ss = ctl.stats();
  s.n_requests = (int64_t)c->reqs.size();
  s.prompt_tokens = ss.prompt_tokens;
  s.generated_tokens = gen;
  s.n_microbatches = ss.n_mb;
  s.n_prefill_mb = ss.n_prefill;
  s.n_decode_mb = ss.n_decode;
  s.n_p2d = ss.p2d;
  s.n_d2p = ss.d2p;
  s.n_stolen = ss.stolen;
  s.n_evicted = ss.evicted;
  if (s.makespan_ns > 0) {
    s.gen_tokens_per_s = gen * 1e9 / (double)s.makespan_ns;
    s.total_tokens_per_s = (gen + ss.prompt_tokens) * 1e9 / (double)s.makespan_ns;
  }
  if (st) *st = s;
  return TD_OK;
}

// Timed pipeline model for td_simulate: stages are FIFO servers with the
// frozen per-stage profile times; launch time = the controller event time.
struct SimHooks : ExecHooks {
  int S;
  const std::vector<int64_t>& tdec;
  const std::vector<int64_t>& tpre;
  int64_t host_ns;
  std::vector<int64_t> free_at, busy;
  std::vector<int64_t> ret;   // by micro-batch id
  int64_t now = 0, makespan = 0;
  std::vector<td_ctx::Span>* spans = nullptr;
  std::vector<std::pair<int64_t, int64_t>>* kv = nullptr;
  SimHooks(int s, const std::vector<int64_t>& d, const std::vector<int64_t>& p, int64_t h)
      : S(s), tdec(d), tpre(p), host_ns(h), free_at(s, 0), busy(s, 0) {}
  static int64_t at(const std::vector<int64_t>& t, int64_t i) {
    return t[std::min<int64_t>(std::max<int64_t>(i, 1), (int64_t)t.size() - 1)];
  }
  int launch(const MicroBatch& mb, const std::vector<Req>& reqs) override {
    int64_t tok = 0;
    for (int q : mb.q_len) tok += q;
    int64_t t;
    if (mb.kind == 'H') {
      // hybrid micro-batch [R23]: the GEMMs see all its tokens like a prefill
      // of that many tokens (and stream the weights at least once, D(1)); the
      // decode members add their attention, taken as the decode table's growth
      // over a batch of one.  The chunks' re-read of their prefix KV is not
      // charged (favours PP+HB)
      int64_t nd = 0;
      for (size_t i = 0; i < mb.members.size(); ++i) nd += mb.q_start[i] >= reqs[mb.members[i]].L ? 1 : 0;
      t = std::max(at(tpre, tok), at(tdec, 1)) + (nd > 0 ? std::max<int64_t>(0, at(tdec, nd) - at(tdec, 1)) : 0);
    } else {
      t = mb.kind == 'P' ? at(tpre, tok) : at(tdec, (int64_t)mb.members.size());
    }
    int64_t arrive = now;
    for (int s = 0; s < S; ++s) {
      const int64_t start = std::max(arrive, free_at[s]);
      free_at[s] = start + t;
      busy[s] += t;
      arrive = start + t;
      if (spans) spans->push_back({mb.mid, mb.kind, s, start, start + t});
    }
    if (kv) {
      int64_t used = 0;
      for (const auto& r : reqs) used += (int64_t)r.blocks.size();
      kv->push_back({now, used});
    }
    if ((int64_t)ret.size() <= mb.mid) ret.resize(mb.mid + 1, 0);
    ret[mb.mid] = arrive + host_ns;
    return 0;
  }
  int returned(const MicroBatch& mb) override {
    now = std::max(now, ret[mb.mid]);
    makespan = std::max(makespan, now);
    return 0;
  }
};

extern "C" td_status td_simulate(td_ctx* c, td_run_stats* st, int64_t host_return_ns) {
  if (!c || !st) return TD_EINVAL;
  if (c->tdec.size() < 2 || c->tpre.size() < 2) return fail(c, TD_ESTATE, "td_simulate needs a profile table");
  SchedOptions so;
  so.W = c->n_stages;
  so.B = c->opt.block_size;
  so.C = c->kv_blocks;
  so.budget = c->opt.prefill_token_budget;
  so.max_seqs = c->opt.max_batch_seqs;
  so.fp_stride = c->opt.fp_stride;
  so.fp_horizon = c->opt.fp_horizon;
  so.policy = c->opt.policy;
  so.steal = c->opt.steal;
  so.check_before_launch = c->opt.alg1_check_before_launch;
  so.eq2_bubble_scale = c->opt.eq2_bubble_scale;
  so.p2d_kv_permille = c->opt.p2d_kv_permille;
  so.d2p_finish_permille = c->opt.d2p_finish_permille;
  so.hb_tokens = c->opt.hb_tokens;
  std::vector<Req> reqs(c->reqs.size());
  for (size_t i = 0; i < c->reqs.size(); ++i) {
    reqs[i].rid = (int)i;
    reqs[i].n_prompt = (int)c->reqs[i].prompt.size();
    reqs[i].L = reqs[i].n_prompt;
    reqs[i].P = c->reqs[i].predicted;
    reqs[i].N = c->reqs[i].max_new;
  }
  Controller ctl(so, reqs, c->tdec, c->tpre, c->opt.log_decisions != 0);
  SimHooks sim(c->n_stages, c->tdec, c->tpre, host_return_ns);
  c->spans.clear();
  c->kv_samples.clear();
  sim.spans = &c->spans;
  sim.kv = &c->kv_samples;
  if (int rc = ctl.run(&sim)) return fail(c, rc < 0 ? rc : TD_ESTATE, ctl.error);
  td_run_stats s{};
  const auto& ss = ctl.stats();
  int64_t gen = 0;
  for (const auto& r : ctl.reqs()) gen += r.n_out;
  s.n_requests = (int64_t)reqs.size();
  s.prompt_tokens = ss.prompt_tokens;
  s.generated_tokens = gen;
  s.makespan_ns = sim.makespan;
  s.n_microbatches = ss.n_mb;
  s.n_prefill_mb = ss.n_prefill;
  s.n_decode_mb = ss.n_decode;
  s.n_p2d = ss.p2d;
  s.n_d2p = ss.d2p;
  s.n_stolen = ss.stolen;
  s.n_evicted = ss.evicted;
  double busy = 0;
  for (int i = 0; i < c->n_stages; ++i) {
    busy += (double)sim.busy[i];
    if (i < 8) s.busy_ns[i] = sim.busy[i];
  }
  if (sim.makespan > 0) {
    s.gen_tokens_per_s = gen * 1e9 / (double)sim.makespan;
    s.total_tokens_per_s = (gen + ss.prompt_tokens) * 1e9 / (double)sim.makespan;
    s.bubble_frac = 1.0 - busy / ((double)c->n_stages * (double)sim.makespan);
  }
  c->log = ctl.log();
  *st = s;
  return TD_OK;
}

extern "C" td_status td_write_trace(td_ctx* c, const char* path) {
  if (!c || !path) return TD_EINVAL;
  std::ofstream f(path);
  if (!f) return fail(c, TD_EINVAL, "cannot open trace path");
  f << "{\"traceEvents\":[";
  bool first = true;
  char buf[256];
  for (const auto& sp : c->spans) {
    snprintf(buf, sizeof buf, "%s{\"name\":\"%c %lld\",\"ph\":\"X\",\"ts\":%.3f,\"dur\":%.3f,\"pid\":0,\"tid\":%d}",
             first ? "" : ",", sp.kind, (long long)sp.mid, sp.a / 1e3, (sp.b - sp.a) / 1e3, sp.stage);
    f << buf;
    first = false;
  }
  for (const auto& kv : c->kv_samples) {
    snprintf(buf, sizeof buf, "%s{\"name\":\"kv_used_blocks\",\"ph\":\"C\",\"ts\":%.3f,\"pid\":0,\"args\":{\"blocks\":%lld}}",
             first ? "" : ",", kv.first / 1e3, (long long)kv.second);
    f << buf;
    first = false;
  }
  f << "]}\n";
  return TD_OK;
}

static td_status cache_outputs(td_ctx* c) {
  if (c->outputs_cached) return TD_OK;
  if (!c->have_run) return fail(c, TD_ESTATE, "td_run has not completed");
  if (!c->engine) {
    c->outputs.assign(c->reqs.size(), {});
    for (size_t i = 0; i < c->reqs.size(); ++i) c->outputs[i].assign(c->n_out[i], 0);
  } else {
    td_status st = c->engine->get_outputs(c->reqs, c->n_out, &c->outputs);
    if (st) return fail(c, st, c->engine->error);
  }
  c->outputs_cached = true;
  return TD_OK;
}

extern "C" td_status td_get_output(td_ctx* c, int64_t id, int32_t* buf, int32_t cap, int32_t* n) {
  if (!c || id < 0 || id >= (int64_t)c->reqs.size()) return TD_EINVAL;
  if (td_status st = cache_outputs(c)) return st;
  const auto& o = c->outputs[id];
  if (n) *n = (int32_t)o.size();
  if (cap < (int32_t)o.size()) return TD_ERANGE;
  if (buf && !o.empty()) std::memcpy(buf, o.data(), o.size() * sizeof(int32_t));
  return TD_OK;
}

extern "C" td_status td_get_outputs(td_ctx* c, int32_t* out, int32_t n_rows, int32_t stride, int32_t* n_out) {
  if (!c || !out || !n_out || stride < 0) return TD_EINVAL;
  if (td_status st = cache_outputs(c)) return st;
  if ((size_t)std::max(n_rows, 0) < c->outputs.size())
    return fail(c, TD_ERANGE, "n_rows < number of submitted requests");
  for (const auto& o : c->outputs)
    if ((int32_t)o.size() > stride) return fail(c, TD_ERANGE, "stride < longest output");
  for (size_t i = 0; i < c->outputs.size(); ++i) {
    const auto& o = c->outputs[i];
    n_out[i] = (int32_t)o.size();
    if (!o.empty()) std::memcpy(out + i * (size_t)stride, o.data(), o.size() * sizeof(int32_t));
  }
  return TD_OK;
}

extern "C" td_status td_get_logits(td_ctx* c, int64_t id, float* buf, int64_t cap, int32_t* n_steps) {
  if (!c || id < 0 || id >= (int64_t)c->reqs.size()) return TD_EINVAL;
  if (!c->engine) return fail(c, TD_ESTATE, "no logits with the null executor");
  std::vector<float> v;
  int n = 0;
  td_status st = c->engine->get_logits(id, &v, &n);
  if (st) return fail(c, st, c->engine->error);
  if (n_steps) *n_steps = n;
  if (cap < (int64_t)v.size()) return TD_ERANGE;
  if (buf && !v.empty()) std::memcpy(buf, v.data(), v.size() * sizeof(float));
  return TD_OK;
}

extern "C" td_status td_reset(td_ctx* c) {
  if (!c) return TD_EINVAL;
  c->reqs.clear();
  c->log.clear();
  c->n_out.clear();
  c->outputs.clear();
  c->have_run = false;
  c->outputs_cached = false;
  return TD_OK;
}

extern "C" td_status td_stage_forward(td_ctx* c, int32_t stage, const td_batch* b, const void* in, void* out) {
  if (!c || !b || !in || !out) return TD_EINVAL;
  if (!c->engine) return fail(c, TD_ESTATE, "null executor");
  if (stage < 0 || stage >= c->n_stages) return fail(c, TD_EINVAL, "bad stage");
  td_status st = c->engine->stage_forward(stage, *b, in, out);
  if (st) c->err = c->engine->error;
  return st;
}

extern "C" td_status td_kv_reset(td_ctx* c) {
  if (!c) return TD_EINVAL;
  if (!c->engine) return TD_OK;
  return c->engine->kv_reset();
}

static td_status write_profile(td_ctx* c, const char* path) {
  std::ofstream f(path);
  if (!f) return fail(c, TD_EINVAL, "cannot write profile csv");
  for (size_t b = 1; b < c->tdec.size(); ++b) f << "D," << b << "," << c->tdec[b] << "\n";
  for (size_t k = 1; k < c->tpre.size(); ++k) f << "P," << k << "," << c->tpre[k] << "\n";
  return TD_OK;
}

extern "C" td_status td_profile(td_ctx* c, const char* out_csv, int32_t b_max, int32_t k_max, int32_t ctx_len) {
  if (!c || b_max < 1 || k_max < 1 || ctx_len < 1) return TD_EINVAL;
  if (!c->engine) return fail(c, TD_ESTATE, "null executor");
  std::vector<int64_t> tdec, tpre;
  td_status st = c->engine->profile(b_max, k_max, ctx_len, &tdec, &tpre);
  if (st) return fail(c, st, c->engine->error);
  c->tdec = tdec;
  c->tpre = tpre;
  if (out_csv) return write_profile(c, out_csv);
  return TD_OK;
}

extern "C" td_status td_load_profile(td_ctx* c, const char* csv) {
  if (!c || !csv) return TD_EINVAL;
  std::string e;
  if (!read_profile(csv, &c->tdec, &c->tpre, &e)) return fail(c, TD_EINVAL, e);
  return TD_OK;
}

extern "C" td_status td_get_log(td_ctx* c, char* buf, size_t cap, size_t* need) {
  if (!c) return TD_EINVAL;
  if (need) *need = c->log.size();
  if (buf && cap) std::memcpy(buf, c->log.data(), std::min(cap, c->log.size()));
  return TD_OK;
}

extern "C" td_status td_info(td_ctx* c, int64_t* kv_blocks, int32_t* n_stages, int64_t* weight_bytes_stage0,
                             int64_t* kv_bytes_per_block) {
  if (!c) return TD_EINVAL;
  if (kv_blocks) *kv_blocks = c->kv_blocks;
  if (n_stages) *n_stages = c->n_stages;
  if (weight_bytes_stage0) *weight_bytes_stage0 = c->engine ? c->engine->weight_bytes_stage0() : 0;
  if (kv_bytes_per_block) *kv_bytes_per_block = c->engine ? c->engine->kv_bytes_per_block() : 0;
  return TD_OK;
}

extern "C" td_status td_bench_step(td_ctx* c, int32_t kind, int32_t n_seqs, int32_t len, int32_t iters,
                                   double* step_us, double* ideal_us) {
  if (!c || !step_us || (kind != TD_BATCH_PREFILL && kind != TD_BATCH_DECODE)) return TD_EINVAL;
  if (!c->engine) return fail(c, TD_ESTATE, "null executor");
  double ms = 0, ideal = 0;
  if (td_status st = c->engine->bench_step(kind == TD_BATCH_PREFILL, n_seqs, len, iters, &ms, &ideal))
    return fail(c, st, c->engine->error);
  *step_us = ms * 1e3;
  if (ideal_us) *ideal_us = ideal * 1e3;
  return TD_OK;
}

extern "C" td_status td_set_timing(td_ctx* c, int32_t on) {
  if (!c) return TD_EINVAL;
  if (c->engine) c->engine->set_timing(on != 0);
  return TD_OK;
}

extern "C" td_status td_get_timing(td_ctx* c, const char* name, int64_t* launches, double* total_ms,
                                   double* bytes, double* flops) {
  if (!c || !name) return TD_EINVAL;
  KernelTiming t;
  if (!c->engine || !c->engine->get_timing(name, &t)) return TD_EINVAL;
  if (launches) *launches = t.launches;
  if (total_ms) *total_ms = t.ms;
  if (bytes) *bytes = t.bytes;
  if (flops) *flops = t.flops;
  return TD_OK;
}

extern "C" td_status td_get_weight(td_ctx* c, int32_t tensor_id, uint16_t* out, int64_t cap, int64_t* rows,
                                   int64_t* cols) {
  if (!c || !rows || !cols) return TD_EINVAL;
  if (!c->engine) return fail(c, TD_ESTATE, "null executor");
  std::vector<uint16_t> w;
  int64_t r = 0, k = 0;
  if (td_status st = c->engine->get_weight(tensor_id, &w, &r, &k)) return fail(c, st, c->engine->error);
  *rows = r;
  *cols = k;
  if (!out) return TD_OK;
  if (cap < r * k) return fail(c, TD_ERANGE, "cap < rows * cols");
  std::memcpy(out, w.data(), (size_t)(r * k) * sizeof(uint16_t));
  return TD_OK;
}

extern "C" td_status td_get_launch_bytes(td_ctx* c, const char* name, double* out, int64_t cap, int64_t* n) {
  if (!c || !name || !n) return TD_EINVAL;
  KernelTiming t;
  if (!c->engine || !c->engine->get_timing(name, &t)) return TD_EINVAL;
  *n = (int64_t)t.launch_bytes.size();
  if (!out) return TD_OK;
  if (cap < *n) return fail(c, TD_ERANGE, "cap < launches");
  std::memcpy(out, t.launch_bytes.data(), t.launch_bytes.size() * sizeof(double));
  return TD_OK;
}

// NCCL is loaded lazily (dlopen) so that single-process and CPU-only use never
// needs it; td_nccl_ids returns two ncclUniqueIds (forward and token-return comms).
typedef int (*nccl_get_unique_id_fn)(void*);
void* tdp_nccl_handle(std::string* err);

extern "C" td_status td_nccl_ids(void* out256) {
  if (!out256) return TD_EINVAL;
  std::string err;
  void* h = tdp_nccl_handle(&err);
  if (!h) { fprintf(stderr, "td_nccl_ids: %s\n", err.c_str()); return TD_ENCCL; }
  auto f = (nccl_get_unique_id_fn)dlsym(h, "ncclGetUniqueId");
  if (!f) return TD_ENCCL;
  if (f(out256) != 0) return TD_ENCCL;
  if (f((char*)out256 + 128) != 0) return TD_ENCCL;
  return TD_OK;
}
