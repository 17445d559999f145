// controller.cpp -- TD-Pipe control plane (see controller.h for citations).
// Mirrors the step order of SURVEY.md §8(c) S0-S12; the decision log (S12) must
// be byte-identical to the reference scheduler's (tests/test_sched_parity.py).
#include "controller.h"

#include <algorithm>
#include <cstdio>

namespace tdp {

static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

Controller::Controller(const SchedOptions& o, const std::vector<Req>& reqs,
                       const std::vector<int64_t>& tdec, const std::vector<int64_t>& tpre,
                       bool keep_log)
    : opt_(o), reqs_(reqs), tdec_(tdec), tpre_(tpre), keep_log_(keep_log) {
  for (auto& r : reqs_) r.P = std::max(r.P, 1);
  for (size_t i = 0; i < reqs_.size(); ++i) pending_fresh_.push_back((int)i);
  const int s = opt_.fp_stride;
  int64_t maxP = 1;
  for (auto& r : reqs_) maxP = std::max<int64_t>(maxP, r.P);
  const int64_t H = std::max<int64_t>(opt_.fp_horizon, s * ceil_div(maxP, s));
  for (int64_t fp = s; fp <= H; fp += s) fps_.push_back((int)fp);
  const int64_t n = (int64_t)reqs_.size();
  if (n) {
    int64_t sl = 0, sp = 0;
    for (auto& r : reqs_) { sl += r.L; sp += r.P; }
    ctx_rep_ = std::max<int64_t>(1, sl / n + (sp / n) / 2);
  }
  b_mem_ = std::max<int64_t>(1, (opt_.C * opt_.B) / ((int64_t)opt_.W * ctx_rep_));
  if (tdec_.size() > 1) {
    const int64_t bmax = (int64_t)tdec_.size() - 1;
    int64_t best = 1;
    for (int64_t b = 1; b <= std::min(b_mem_, bmax); ++b)
      if ((__int128)b * tdec_[best] >= (__int128)best * tdec_[b]) best = b;
    Bp_ = best;
  }
}

// ------------------------------------------------------------------- utils
void Controller::emit(const std::string& s) {
  if (keep_log_) { log_ += s; log_ += '\n'; }
}

void Controller::emit_ids(const char* head, const std::vector<int64_t>& nums) {
  if (!keep_log_) return;
  log_ += head;
  char buf[32];
  for (int64_t v : nums) {
    snprintf(buf, sizeof buf, " %lld", (long long)v);
    log_ += buf;
  }
  log_ += '\n';
}

std::vector<int> Controller::pending_list() const {
  std::vector<int> v(pending_evicted_.begin(), pending_evicted_.end());
  v.insert(v.end(), pending_fresh_.begin(), pending_fresh_.end());
  return v;
}

int64_t Controller::tdec(int64_t b) const {
  b = std::min<int64_t>(std::max<int64_t>(b, 1), (int64_t)tdec_.size() - 1);
  return tdec_[b];
}
int64_t Controller::tpre(int64_t k) const {
  k = std::min<int64_t>(std::max<int64_t>(k, 1), (int64_t)tpre_.size() - 1);
  return tpre_[k];
}

int32_t Controller::alloc_one() {
  if (!free_heap_.empty()) { int32_t b = free_heap_.top(); free_heap_.pop(); return b; }
  return (int32_t)(watermark_++);
}
void Controller::release(const std::vector<int32_t>& b) {
  for (int32_t x : b) free_heap_.push(x);
}

// -------------------------------------------------------------- Alg.1 S2/S3
// UpdateUsage: for futurePoint <= predictLen,
// kvUsage[futurePoint] += blocks(inputLen + futurePoint); predictLen :=
// remaining predicted decode steps max(P-1-d, 0), inputLen := L + d  [R1,R2].
void Controller::update_usage(std::vector<int64_t>& U, const Req& r) const {
  const int64_t rem = std::max(r.P - 1 - r.d, 0);
  for (size_t i = 0; i < fps_.size(); ++i)
    if (fps_[i] <= rem) U[i] += ceil_div((int64_t)r.L + r.d + fps_[i], opt_.B);
}

std::vector<int64_t> Controller::rebuild_usage() const {
  std::vector<int64_t> U(fps_.size(), 0);
  for (int rid : live_) update_usage(U, reqs_[rid]);   // a sum: order irrelevant
  return U;
}

int64_t Controller::max_usage(const std::vector<int64_t>& U) const {
  int64_t m = 0;
  for (int64_t u : U) if (u > m) m = u;
  return m;
}

// CheckSwitch: switch to decode iff maxUsage > kvCapacity.
bool Controller::check_switch(const std::vector<int64_t>& U) const { return max_usage(U) > opt_.C; }

// getPrefillBatch [R5]: FIFO greedy under the token budget,
// max_seqs, and the now-free guard sum ceil(L/B) <= free blocks.
std::vector<int> Controller::form_prefill_batch(const std::vector<int>& pending, int64_t limit) const {
  std::vector<int> batch;
  int64_t tok = 0, need = 0;
  for (int rid : pending) {
    const Req& r = reqs_[rid];
    if (!batch.empty() && tok + r.L > opt_.budget) break;
    if ((int64_t)batch.size() >= opt_.max_seqs) break;
    const int64_t nb = ceil_div(r.L, opt_.B);
    if (need + nb > limit) break;
    batch.push_back(rid);
    tok += r.L;
    need += nb;
    if (tok >= opt_.budget) break;
  }
  return batch;
}

void Controller::add_usage_fresh(std::vector<int64_t>& U, const std::vector<int>& batch) const {
  for (int rid : batch) {
    const Req& r = reqs_[rid];
    const int64_t rem = std::max(r.P - 1, 0);
    for (size_t i = 0; i < fps_.size(); ++i)
      if (fps_[i] <= rem) U[i] += ceil_div((int64_t)r.L + fps_[i], opt_.B);
  }
}

void Controller::pop_pending(const std::vector<int>& batch) {
  for (int rid : batch) {
    if (!pending_evicted_.empty() && pending_evicted_.front() == rid) pending_evicted_.erase(pending_evicted_.begin());
    else pending_fresh_.pop_front();
  }
}

// SchedulePrefill loop, eager at one logical instant (S4).
int Controller::prefill_phase() {
  std::vector<int64_t> U = rebuild_usage();
  int launched = 0;
  const char* reason = "queue_empty";
  while (true) {
    if (pending_empty()) { reason = "queue_empty"; break; }
    std::vector<int> batch = form_prefill_batch(pending_list(), free_blocks());
    if (batch.empty()) { reason = "now_full"; break; }
    if (opt_.check_before_launch && (launched > 0 || !live_.empty())) {
      std::vector<int64_t> U2 = U;
      add_usage_fresh(U2, batch);
      if (check_switch(U2)) { reason = "forecast_pre"; break; }
    }
    pop_pending(batch);
    if (int rc = launch_prefill(batch, -1)) return rc;      // getPrefillBatch().Launch()
    ++launched;
    for (int rid : batch) update_usage(U, reqs_[rid]);     // UpdateUsage per request
    if (opt_.p2d_kv_permille) {                            // ablation: KV occupancy ratio
      if ((opt_.C - free_blocks()) * 1000 >= (int64_t)opt_.p2d_kv_permille * opt_.C) { reason = "kv_ratio"; break; }
    } else if (check_switch(U)) {                          // CheckSwitch
      reason = "forecast";
      break;
    }
  }
  stats_.p2d++;
  char buf[128];
  snprintf(buf, sizeof buf, "S P2D %s %lld %lld", reason, (long long)max_usage(U), (long long)opt_.C);
  emit(buf);
  return 0;
}

std::vector<int64_t> Controller::dry_run_prefill() const {
  std::vector<int64_t> U = rebuild_usage();
  std::vector<int> pending = pending_list();
  int64_t free = free_blocks();
  std::vector<int64_t> ks;
  int launched = 0;
  size_t off = 0;
  while (off < pending.size()) {
    std::vector<int> rest(pending.begin() + off, pending.end());
    std::vector<int> batch = form_prefill_batch(rest, free);
    if (batch.empty()) break;
    if (opt_.check_before_launch && (launched > 0 || !live_.empty())) {
      std::vector<int64_t> U2 = U;
      add_usage_fresh(U2, batch);
      if (check_switch(U2)) break;
    }
    off += batch.size();
    int64_t k = 0;
    for (int rid : batch) { free -= ceil_div(reqs_[rid].L, opt_.B); k += reqs_[rid].L; }
    ks.push_back(k);
    ++launched;
    add_usage_fresh(U, batch);
    if (opt_.p2d_kv_permille) {
      if ((opt_.C - free) * 1000 >= (int64_t)opt_.p2d_kv_permille * opt_.C) break;
    } else if (check_switch(U)) {
      break;
    }
  }
  return ks;
}

int Controller::launch_prefill(const std::vector<int>& batch, int slot) {
  for (int rid : batch) {
    Req& r = reqs_[rid];
    const int64_t k = ceil_div(r.L, opt_.B);
    std::vector<int64_t> line{rid};
    for (int64_t i = 0; i < k; ++i) { int32_t b = alloc_one(); r.blocks.push_back(b); line.push_back(b); }
    emit_ids("A", line);
  }
  MicroBatch mb;
  mb.mid = mb_counter_++;
  mb.kind = 'P';
  mb.slot = slot;
  mb.epoch = epoch_;
  for (int rid : batch) {
    Req& r = reqs_[rid];
    r.adm = adm_counter_++;
    r.in_flight = true;
    r.g = 0;
    r.d = 0;
    live_.insert(rid);
    mb.members.push_back(rid);
    mb.q_start.push_back(0);
    mb.q_len.push_back(r.L);
    stats_.prompt_tokens += r.L;
  }
  std::vector<int64_t> line{mb.mid, (int64_t)batch.size()};
  for (int rid : batch) line.push_back(rid);
  emit_ids("P", line);
  stats_.n_mb++;
  stats_.n_prefill++;
  inflight_.push_back(mb);
  return ex_ ? ex_->launch(inflight_.back(), reqs_) : 0;
}

// ------------------------------------------------------------ S5 formation
void Controller::form_decode() {
  epoch_++;
  pool_.clear();
  std::vector<int> members(live_.begin(), live_.end());
  std::sort(members.begin(), members.end(), [&](int a, int b) { return reqs_[a].adm < reqs_[b].adm; });
  cohort_n_ = (int64_t)members.size();
  cohort_done_ = 0;
  for (auto& r : reqs_) r.slot = -1;
  slots_.clear();
  const int n = (int)members.size();
  if (n == 0) return;
  const int Wf = std::min(opt_.W, n);
  const int q = n / Wf, rm = n % Wf;
  int idx = 0;
  for (int i = 0; i < Wf; ++i) {
    const int sz = q + (i < rm ? 1 : 0);
    Slot sl;
    sl.idx = i;
    sl.members.assign(members.begin() + idx, members.begin() + idx + sz);
    idx += sz;
    for (int rid : sl.members) reqs_[rid].slot = i;
    std::vector<int64_t> line{i, sz};
    for (int rid : sl.members) line.push_back(rid);
    emit_ids("G", line);
    slots_.push_back(std::move(sl));
  }
}

int Controller::try_launch_formed() {
  for (auto& sl : slots_) {
    if (sl.retired || sl.launched) continue;
    bool busy = false;
    for (int rid : sl.members) if (reqs_[rid].in_flight) { busy = true; break; }
    if (busy) break;
    if (int rc = launch_decode(sl)) return rc;
    if (!(sl.retired || sl.launched)) break;
  }
  return 0;
}

// ------------------------------------------------------------ S8 eviction
// Recompute on overflow: free the KV, prompt := prompt ++ generated.
void Controller::evict(int rid) {
  Req& r = reqs_[rid];
  release(r.blocks);
  std::vector<int64_t> line{rid};
  for (int32_t b : r.blocks) line.push_back(b);
  emit_ids("E", line);
  r.blocks.clear();
  r.L += r.g;
  r.N -= r.g;
  r.P = std::max(r.P - r.g, 1);
  r.g = 0;
  r.d = 0;
  live_.erase(rid);
  const int64_t old = r.adm;
  r.adm = -1;
  r.slot = -1;
  size_t pos = 0;
  while (pos < pending_evicted_.size() && reqs_[pending_evicted_[pos]].evict_key < old) ++pos;
  r.evict_key = old;
  pending_evicted_.insert(pending_evicted_.begin() + pos, rid);
  stats_.evicted++;
}

int64_t Controller::decode_need(const std::vector<int>& members) const {
  int64_t need = 0;
  for (int rid : members) {
    const Req& r = reqs_[rid];
    need += std::max<int64_t>(0, ceil_div((int64_t)r.L + r.d + 1, opt_.B) - (int64_t)r.blocks.size());
  }
  return need;
}

void Controller::ensure_blocks(Slot& sl) {
  while (!sl.members.empty() && decode_need(sl.members) > free_blocks()) {
    int victim = -1;
    int64_t best = -1;
    for (int rid : sl.members) if (reqs_[rid].adm > best) { best = reqs_[rid].adm; victim = rid; }
    for (int rid : pool_) if (reqs_[rid].adm > best) { best = reqs_[rid].adm; victim = rid; }
    auto it = std::find(sl.members.begin(), sl.members.end(), victim);
    if (it != sl.members.end()) sl.members.erase(it);
    else pool_.erase(std::find(pool_.begin(), pool_.end(), victim));
    evict(victim);
  }
}

int Controller::launch_decode(Slot& sl) {
  ensure_blocks(sl);
  if (sl.members.empty()) { retire(sl); return 0; }
  for (int rid : sl.members) {
    Req& r = reqs_[rid];
    const int64_t k = ceil_div((int64_t)r.L + r.d + 1, opt_.B) - (int64_t)r.blocks.size();
    if (k > 0) {
      std::vector<int64_t> line{rid};
      for (int64_t i = 0; i < k; ++i) { int32_t b = alloc_one(); r.blocks.push_back(b); line.push_back(b); }
      emit_ids("A", line);
    }
  }
  MicroBatch mb;
  mb.mid = mb_counter_++;
  mb.kind = 'D';
  mb.slot = sl.idx;
  mb.epoch = epoch_;
  for (int rid : sl.members) {
    Req& r = reqs_[rid];
    mb.members.push_back(rid);
    mb.q_start.push_back(r.L + r.d);
    mb.q_len.push_back(1);
    r.in_flight = true;
  }
  sl.launched = true;
  sl.inflight = true;
  std::vector<int64_t> line{mb.mid, sl.idx, (int64_t)sl.members.size()};
  for (int rid : sl.members) line.push_back(rid);
  emit_ids("D", line);
  stats_.n_mb++;
  stats_.n_decode++;
  inflight_.push_back(mb);
  return ex_ ? ex_->launch(inflight_.back(), reqs_) : 0;
}

void Controller::retire(Slot& sl) {
  if (!sl.retired) {
    sl.retired = true;
    emit_ids("X", {sl.idx});
  }
}

// ------------------------------------------------------------ S7 stealing
// Inter-batch work stealing, pool counted [R7].
void Controller::steal_refill(Slot& sl) {
  int64_t n_live = 0, n_others = 0;
  for (auto& s : slots_) if (&s != &sl && !s.retired) { n_live += (int64_t)s.members.size(); n_others++; }
  const int64_t rem = (int64_t)sl.members.size();
  n_live += rem + (int64_t)pool_.size();
  const int64_t Wa = n_others + 1;
  const int64_t q = n_live / Wa, s_ = n_live % Wa;
  int64_t A = 0;
  for (auto& s : slots_) if (&s != &sl && !s.retired && (int64_t)s.members.size() > q) A++;
  const int64_t target = q + (A < s_ ? 1 : 0);
  if (rem > target) {
    const int64_t k = rem - target;
    std::vector<int64_t> line{sl.idx};
    for (size_t i = sl.members.size() - (size_t)k; i < sl.members.size(); ++i) {
      const int rid = sl.members[i];
      reqs_[rid].slot = -1;
      pool_.push_back(rid);
      line.push_back(rid);
    }
    sl.members.resize(sl.members.size() - (size_t)k);
    stats_.stolen += k;
    emit_ids("W", line);
  } else if (rem < target && !pool_.empty()) {
    const int64_t k = std::min<int64_t>(target - rem, (int64_t)pool_.size());
    std::vector<int64_t> line{sl.idx};
    for (int64_t i = 0; i < k; ++i) {
      const int rid = pool_.front();
      pool_.pop_front();
      reqs_[rid].slot = sl.idx;
      sl.members.push_back(rid);
      line.push_back(rid);
    }
    stats_.refilled += k;
    emit_ids("U", line);
  }
}

// ------------------------------------------------------------ S9/S10 rule
// Eq.1 spatial = Achieved/Peak; Eq.2 temporal = 1 - bubble/total; switch to
// prefill iff spatial < temporal, exact integers.
bool Controller::decide_switch(Slot& sl) {
  std::vector<int64_t> ks = dry_run_prefill();
  if (ks.empty()) return false;
  if (opt_.d2p_finish_permille) {   // ablation: request-finish ratio of the decode cohort
    if (cohort_done_ * 1000 >= (int64_t)opt_.d2p_finish_permille * cohort_n_) {
      emit_ids("S D2P finish_ratio", {cohort_done_, cohort_n_});
      return true;
    }
    return false;
  }
  const int64_t bs = (int64_t)sl.members.size();
  int64_t sum_pre = 0, max_pre = 0;
  for (int64_t k : ks) { const int64_t t = tpre(k); sum_pre += t; max_pre = std::max(max_pre, t); }
  char buf[256];
  if (bs == 0) {
    snprintf(buf, sizeof buf, "S D2P 0 0 %lld %lld 0 %lld", (long long)tdec(Bp_), (long long)Bp_, (long long)sum_pre);
    emit(buf);
    return true;
  }
  const int64_t tdb = tdec(bs), tdp = tdec(Bp_);
  const int64_t bubble = (int64_t)opt_.eq2_bubble_scale * std::max<int64_t>(0, max_pre - tdb);
  const int64_t total = sum_pre + (int64_t)opt_.W * tdb + bubble;
  if ((__int128)bs * tdp * total < (__int128)Bp_ * tdb * (total - bubble)) {
    snprintf(buf, sizeof buf, "S D2P %lld %lld %lld %lld %lld %lld", (long long)bs, (long long)tdb,
             (long long)tdp, (long long)Bp_, (long long)bubble, (long long)total);
    emit(buf);
    return true;
  }
  return false;
}

// ------------------------------------------------------------ S6 returns
void Controller::finish(Req& r) {
  r.done = true;
  cohort_done_++;
  release(r.blocks);
  std::vector<int64_t> line{r.rid};
  for (int32_t b : r.blocks) line.push_back(b);
  emit_ids("F", line);
  r.blocks.clear();
  live_.erase(r.rid);
  auto pit = std::find(pool_.begin(), pool_.end(), r.rid);
  if (pit != pool_.end()) pool_.erase(pit);
  if (r.slot >= 0 && r.slot < (int)slots_.size()) {
    auto& m = slots_[r.slot].members;
    auto it = std::find(m.begin(), m.end(), r.rid);
    if (it != m.end()) m.erase(it);
  }
  r.slot = -1;
}

int Controller::on_return(const MicroBatch& mb) {
  {
    std::vector<int64_t> line{mb.mid, (int64_t)mb.members.size()};
    for (int rid : mb.members) line.push_back(rid);
    emit_ids("R", line);
  }
  if (ex_) if (int rc = ex_->returned(mb)) return rc;
  for (int rid : mb.members) {
    Req& r = reqs_[rid];
    r.in_flight = false;
    r.g++;
    r.n_out++;
    if (mb.kind == 'D') r.d++;
    if (r.g == r.N) finish(r);
  }
  const bool current = mb.kind == 'D' && mb.epoch == epoch_;
  if (!current) {
    for (auto& sl : slots_)
      if (!sl.retired && !sl.launched && sl.members.empty()) retire(sl);
    return 0;
  }
  Slot& sl = slots_[mb.slot];
  sl.inflight = false;
  if (opt_.steal && opt_.W > 1) steal_refill(sl);
  if (!pending_empty() && decide_switch(sl)) {
    stats_.d2p++;
    if (int rc = prefill_phase()) return rc;
    form_decode();
    return 0;
  }
  if (sl.members.empty()) { retire(sl); return 0; }
  return launch_decode(sl);
}

int Controller::run_tdpipe() {
  if (reqs_.empty()) return 0;
  if (int rc = prefill_phase()) return rc;
  form_decode();
  if (int rc = try_launch_formed()) return rc;
  while (!inflight_.empty()) {
    MicroBatch mb = std::move(inflight_.front());
    inflight_.pop_front();
    if (int rc = on_return(mb)) return rc;
    if (int rc = try_launch_formed()) return rc;
    bool any_active = false;
    for (auto& s : slots_) if (!s.retired) { any_active = true; break; }
    if (!any_active && (!pending_empty() || !live_.empty())) {
      emit("S D2P idle");
      stats_.d2p++;
      if (int rc = prefill_phase()) return rc;
      form_decode();
      if (int rc = try_launch_formed()) return rc;
    }
  }
  if (!pending_empty() || !live_.empty()) { error = "scheduler stalled"; return -6; }
  return 0;
}

// ------------------------------------------------------------ S11 baselines
// Naive phase-interleaved PP+SB: W virtual engines, request r on engine r mod W,
// per-engine KV quota C/W.  ALT: prefill only if the engine's previous
// micro-batch was not a prefill (or it has nothing to decode); PRIO: whenever
// admissible.  Own-quota eviction of the most recently admitted running request.
int Controller::run_baseline() {
  const int W = opt_.W;
  std::vector<int64_t> quota(W), used(W, 0);
  for (int e = 0; e < W; ++e) quota[e] = opt_.C / W + (e < opt_.C % W ? 1 : 0);
  std::vector<std::vector<int>> q_ev(W), running(W);
  std::vector<std::deque<int>> q_fr(W);
  for (auto& r : reqs_) q_fr[r.rid % W].push_back(r.rid);
  std::vector<char> last(W, '-');
  for (auto& r : reqs_)
    if (ceil_div((int64_t)r.L + r.N, opt_.B) > quota[r.rid % W]) {
      error = "request exceeds its engine's KV quota";
      return -5;
    }

  auto issue = [&](int e) -> int {
    while (true) {
      std::vector<int> pend(q_ev[e].begin(), q_ev[e].end());
      pend.insert(pend.end(), q_fr[e].begin(), q_fr[e].end());
      std::vector<int> batch;
      if (!pend.empty()) batch = form_prefill_batch(pend, quota[e] - used[e]);
      bool do_p = !batch.empty();
      if (opt_.policy == kPPSBAlt) do_p = do_p && (last[e] != 'P' || running[e].empty());
      if (do_p) {
        for (int rid : batch) {
          if (!q_ev[e].empty() && q_ev[e].front() == rid) q_ev[e].erase(q_ev[e].begin());
          else q_fr[e].pop_front();
        }
        if (int rc = launch_prefill(batch, e)) return rc;
        for (int rid : batch) used[e] += (int64_t)reqs_[rid].blocks.size();
        running[e].insert(running[e].end(), batch.begin(), batch.end());
        last[e] = 'P';
        return 0;
      }
      if (!running[e].empty()) {
        while (!running[e].empty()) {
          if (decode_need(running[e]) <= quota[e] - used[e]) break;
          int victim = -1;
          int64_t best = -1;
          for (int rid : running[e]) if (reqs_[rid].adm > best) { best = reqs_[rid].adm; victim = rid; }
          running[e].erase(std::find(running[e].begin(), running[e].end(), victim));
          Req& r = reqs_[victim];
          used[e] -= (int64_t)r.blocks.size();
          const int64_t old = r.adm;
          release(r.blocks);
          std::vector<int64_t> line{victim};
          for (int32_t b : r.blocks) line.push_back(b);
          emit_ids("E", line);
          r.blocks.clear();
          r.L += r.g;
          r.N -= r.g;
          r.P = std::max(r.P - r.g, 1);
          r.g = r.d = 0;
          r.adm = -1;
          live_.erase(victim);
          size_t pos = 0;
          while (pos < q_ev[e].size() && reqs_[q_ev[e][pos]].evict_key < old) ++pos;
          r.evict_key = old;
          q_ev[e].insert(q_ev[e].begin() + pos, victim);
          stats_.evicted++;
        }
        if (running[e].empty()) { last[e] = '-'; continue; }
        for (int rid : running[e]) {
          Req& r = reqs_[rid];
          const int64_t k = ceil_div((int64_t)r.L + r.d + 1, opt_.B) - (int64_t)r.blocks.size();
          if (k > 0) {
            std::vector<int64_t> line{rid};
            for (int64_t i = 0; i < k; ++i) { int32_t b = alloc_one(); r.blocks.push_back(b); line.push_back(b); }
            used[e] += k;
            emit_ids("A", line);
          }
        }
        MicroBatch mb;
        mb.mid = mb_counter_++;
        mb.kind = 'D';
        mb.slot = e;
        mb.epoch = 0;
        for (int rid : running[e]) {
          Req& r = reqs_[rid];
          mb.members.push_back(rid);
          mb.q_start.push_back(r.L + r.d);
          mb.q_len.push_back(1);
          r.in_flight = true;
        }
        std::vector<int64_t> line{mb.mid, e, (int64_t)mb.members.size()};
        for (int rid : mb.members) line.push_back(rid);
        emit_ids("D", line);
        stats_.n_mb++;
        stats_.n_decode++;
        inflight_.push_back(mb);
        last[e] = 'D';
        return ex_ ? ex_->launch(inflight_.back(), reqs_) : 0;
      }
      return 0;  // engine idle
    }
  };

  for (int e = 0; e < W; ++e) if (int rc = issue(e)) return rc;
  while (!inflight_.empty()) {
    MicroBatch mb = std::move(inflight_.front());
    inflight_.pop_front();
    const int e = mb.slot;
    {
      std::vector<int64_t> line{mb.mid, (int64_t)mb.members.size()};
      for (int rid : mb.members) line.push_back(rid);
      emit_ids("R", line);
    }
    if (ex_) if (int rc = ex_->returned(mb)) return rc;
    for (int rid : mb.members) {
      Req& r = reqs_[rid];
      r.in_flight = false;
      r.g++;
      r.n_out++;
      if (mb.kind == 'D') r.d++;
      if (r.g == r.N) {
        used[e] -= (int64_t)r.blocks.size();
        r.done = true;
        release(r.blocks);
        std::vector<int64_t> line{rid};
        for (int32_t b : r.blocks) line.push_back(b);
        emit_ids("F", line);
        r.blocks.clear();
        live_.erase(rid);
        running[e].erase(std::find(running[e].begin(), running[e].end(), rid));
      }
    }
    if (int rc = issue(e)) return rc;
  }
  for (auto& r : reqs_) if (!r.done) { error = "baseline stalled"; return -6; }
  return 0;
}

// ------------------------------------------------------------ PP+HB [R23]
// Hybrid batching with chunked prefill: the
// PP+SB engine layout (W virtual engines, r mod W, quota C/W); each micro-batch
// = the engine's decoding requests (one token each, admission order) + prefill
// chunks up to hb_tokens (partially prefilled prompts first, then pending
// ones, evicted before fresh); a chunk is min(remaining prompt, budget left,
// tokens whose blocks fit).  The chunk completing a prompt yields the first
// token.  Mirrors oracle/scheduler.py RefScheduler._run_hybrid line by line.
int Controller::run_hybrid() {
  const int W = opt_.W;
  const int T = std::max(opt_.hb_tokens, 1);
  std::vector<int64_t> quota(W), used(W, 0);
  for (int e = 0; e < W; ++e) quota[e] = opt_.C / W + (e < opt_.C % W ? 1 : 0);
  std::vector<std::vector<int>> q_ev(W), running(W), filling(W);
  std::vector<std::deque<int>> q_fr(W);
  for (auto& r : reqs_) q_fr[r.rid % W].push_back(r.rid);
  for (auto& r : reqs_)
    if (ceil_div((int64_t)r.L + r.N, opt_.B) > quota[r.rid % W]) {
      error = "request exceeds its engine's KV quota";
      return -5;
    }
  auto contains = [](const std::vector<int>& v, int x) { return std::find(v.begin(), v.end(), x) != v.end(); };
  auto max_adm = [&](const std::vector<int>& v) {
    int victim = -1;
    int64_t best = -2;
    for (int rid : v) if (reqs_[rid].adm > best) { best = reqs_[rid].adm; victim = rid; }
    return victim;
  };
  auto evict = [&](int e, int victim) {
    Req& r = reqs_[victim];
    used[e] -= (int64_t)r.blocks.size();
    const int64_t old = r.adm;
    release(r.blocks);
    std::vector<int64_t> line{victim};
    for (int32_t b : r.blocks) line.push_back(b);
    emit_ids("E", line);
    r.blocks.clear();
    auto& from = contains(running[e], victim) ? running[e] : filling[e];
    from.erase(std::find(from.begin(), from.end(), victim));
    r.L += r.g;
    r.N -= r.g;
    r.P = std::max(r.P - r.g, 1);
    r.g = r.d = r.pf = 0;
    r.adm = -1;
    live_.erase(victim);
    size_t pos = 0;
    while (pos < q_ev[e].size() && reqs_[q_ev[e][pos]].evict_key < old) ++pos;
    r.evict_key = old;
    q_ev[e].insert(q_ev[e].begin() + pos, victim);
    stats_.evicted++;
  };
  struct Chunk { int rid, q0, ql; };
  auto plan = [&](int e, std::vector<int>& dec, std::vector<Chunk>& chunks) {
    dec = running[e];
    chunks.clear();
    int64_t avail = quota[e] - used[e] - decode_need(dec);
    int64_t budget = T - (int64_t)dec.size();
    std::vector<int> cands(filling[e]);
    cands.insert(cands.end(), q_ev[e].begin(), q_ev[e].end());
    cands.insert(cands.end(), q_fr[e].begin(), q_fr[e].end());
    for (int rid : cands) {
      if (budget <= 0) break;
      const Req& r = reqs_[rid];
      const int64_t fit = ((int64_t)r.blocks.size() + avail) * opt_.B - r.pf;
      const int64_t take = std::min<int64_t>({(int64_t)r.L - r.pf, budget, fit});
      if (take <= 0) break;
      avail -= ceil_div((int64_t)r.pf + take, opt_.B) - (int64_t)r.blocks.size();
      chunks.push_back({rid, r.pf, (int)take});
      budget -= take;
    }
  };
  auto issue = [&](int e) -> int {
    while (!running[e].empty() && decode_need(running[e]) > quota[e] - used[e]) {
      std::vector<int> cands(running[e]);
      cands.insert(cands.end(), filling[e].begin(), filling[e].end());
      evict(e, max_adm(cands));
    }
    std::vector<int> dec;
    std::vector<Chunk> chunks;
    plan(e, dec, chunks);
    while (dec.empty() && chunks.empty() && !filling[e].empty()) {
      evict(e, max_adm(filling[e]));
      plan(e, dec, chunks);
    }
    if (dec.empty() && chunks.empty()) return 0;   // engine idle
    auto grow = [&](int rid, int64_t tokens) {
      Req& r = reqs_[rid];
      const int64_t k = ceil_div(tokens, opt_.B) - (int64_t)r.blocks.size();
      if (k > 0) {
        std::vector<int64_t> line{rid};
        for (int64_t i = 0; i < k; ++i) { int32_t b = alloc_one(); r.blocks.push_back(b); line.push_back(b); }
        used[e] += k;
        emit_ids("A", line);
      }
    };
    for (int rid : dec) grow(rid, (int64_t)reqs_[rid].L + reqs_[rid].d + 1);
    for (const Chunk& c : chunks) {
      Req& r = reqs_[c.rid];
      if (r.pf == 0 && !contains(filling[e], c.rid)) {   // admission
        if (!q_ev[e].empty() && q_ev[e].front() == c.rid) q_ev[e].erase(q_ev[e].begin());
        else q_fr[e].pop_front();
        r.adm = adm_counter_++;
        r.g = r.d = 0;
        live_.insert(c.rid);
        filling[e].push_back(c.rid);
      }
      grow(c.rid, (int64_t)c.q0 + c.ql);
    }
    MicroBatch mb;
    mb.mid = mb_counter_++;
    mb.kind = 'H';
    mb.slot = e;
    mb.epoch = 0;
    for (int rid : dec) {
      mb.members.push_back(rid);
      mb.q_start.push_back(reqs_[rid].L + reqs_[rid].d);
      mb.q_len.push_back(1);
    }
    for (const Chunk& c : chunks) {
      mb.members.push_back(c.rid);
      mb.q_start.push_back(c.q0);
      mb.q_len.push_back(c.ql);
    }
    for (int rid : mb.members) reqs_[rid].in_flight = true;
    if (keep_log_) {
      std::string line = "H " + std::to_string(mb.mid) + " " + std::to_string(e) + " " + std::to_string(dec.size()) +
                         " " + std::to_string(chunks.size());
      for (int rid : dec) line += " " + std::to_string(rid);
      for (const Chunk& c : chunks)
        line += " " + std::to_string(c.rid) + ":" + std::to_string(c.q0) + ":" + std::to_string(c.ql);
      emit(line);
    }
    stats_.n_mb++;
    if (dec.empty()) stats_.n_prefill++;
    else stats_.n_decode++;
    for (const Chunk& c : chunks) stats_.prompt_tokens += c.ql;
    inflight_.push_back(mb);
    return ex_ ? ex_->launch(inflight_.back(), reqs_) : 0;
  };

  for (int e = 0; e < W; ++e) if (int rc = issue(e)) return rc;
  while (!inflight_.empty()) {
    MicroBatch mb = std::move(inflight_.front());
    inflight_.pop_front();
    const int e = mb.slot;
    {
      std::vector<int64_t> line{mb.mid, (int64_t)mb.members.size()};
      for (int rid : mb.members) line.push_back(rid);
      emit_ids("R", line);
    }
    if (ex_) if (int rc = ex_->returned(mb)) return rc;
    for (size_t i = 0; i < mb.members.size(); ++i) {
      const int rid = mb.members[i];
      Req& r = reqs_[rid];
      r.in_flight = false;
      if (contains(running[e], rid)) {        // decode token
        r.g++;
        r.n_out++;
        r.d++;
      } else {                                // prefill chunk
        r.pf = mb.q_start[i] + mb.q_len[i];
        if (r.pf < r.L) continue;
        filling[e].erase(std::find(filling[e].begin(), filling[e].end(), rid));
        running[e].push_back(rid);            // prompt complete: first token
        r.g++;
        r.n_out++;
      }
      if (r.g == r.N) {
        used[e] -= (int64_t)r.blocks.size();
        r.done = true;
        release(r.blocks);
        std::vector<int64_t> line{rid};
        for (int32_t b : r.blocks) line.push_back(b);
        emit_ids("F", line);
        r.blocks.clear();
        live_.erase(rid);
        running[e].erase(std::find(running[e].begin(), running[e].end(), rid));
      }
    }
    if (int rc = issue(e)) return rc;
  }
  for (auto& r : reqs_) if (!r.done) { error = "hybrid baseline stalled"; return -6; }
  return 0;
}

int Controller::run(ExecHooks* ex) {
  ex_ = ex;
  if (opt_.policy == kPPHB) return run_hybrid();
  return opt_.policy == kTDPipe ? run_tdpipe() : run_baseline();
}

}  // namespace tdp
