// ps_pipeline.cu — ps_pipeline_run: Algorithm 1 over k
// stages.  AR and synchronous (tiered) SD are driven from the calling thread;
// PIPESPEC runs one host thread per stage.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pipespec.h"

namespace {
long long now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

ps_status tokens_of(ps_stage* s, std::vector<int32_t>& v) {
  int64_t n = 0;
  ps_status st = ps_stage_tokens(s, nullptr, 0, &n);
  if (st != PS_OK) return st;
  v.resize((size_t)n);
  return ps_stage_tokens(s, v.data(), n, &n);
}

// m greedy tokens of stage i given context ctx (stage i is left holding ctx ++ out):
// stage 0 drafts autoregressively; stage i>0 runs sync SD with stage i-1.
ps_status produce(ps_stage* const* S, int i, const std::vector<int32_t>& ctx, int m, const ps_run_opts* o,
                  std::vector<int32_t>& out, ps_run_stats* stt) {
  ps_status st = ps_resync(S[i], ctx.data(), (int32_t)ctx.size());   // rollback cascade, lazy KV catch-up
  if (st != PS_OK) return st;
  out.clear();
  const int gamma = (i > 0 && o->gamma) ? o->gamma[i] : 0;
  while ((int)out.size() < m) {
    if (i == 0 || gamma == 0) {
      int32_t t;
      long long t0 = now_ns();
      if ((st = ps_draft(S[i], 1, &t)) != PS_OK) return st;
      if (stt && i < 8) { stt->steps[i]++; stt->busy_ns[i] += now_ns() - t0; }
      out.push_back(t);
      continue;
    }
    std::vector<int32_t> cur = ctx;
    cur.insert(cur.end(), out.begin(), out.end());
    std::vector<int32_t> d;
    if ((st = produce(S, i - 1, cur, gamma, o, d, stt)) != PS_OK) return st;
    int32_t a, nxt;
    long long t0 = now_ns();
    if ((st = ps_verify(S[i], d.data(), (int32_t)d.size(), &a, &nxt, nullptr)) != PS_OK) return st;
    if (stt && i < 8) {
      stt->steps[i]++; stt->verify_steps[i]++; stt->busy_ns[i] += now_ns() - t0;
      if (a < (int)d.size()) stt->rollbacks[i - 1]++;
    }
    out.insert(out.end(), d.begin(), d.begin() + a);
    out.push_back(nxt);
  }
  out.resize(m);
  return PS_OK;
}
}  // namespace

// ---------------------------------------------------------------- async PipeSpec
// Algorithm 1 with one host thread per stage.  Shared state (the
// committed buffers O_i, epochs, pending resync targets) lives under one mutex;
// every device call runs outside it on the stage's own stream.
//  * stage 0 drafts one token per step ("Generate next token, append to O_0")
//    while it is less than max_lead tokens ahead of stage 1;
//  * stage i>0 takes window = O_{i-1}[n : n + min(avail, gamma_i)] when at least
//    max(1, lookahead_i) valid drafts exist, else an AR step (lookahead 0) or
//    waits; verifies; publishes the accepted tokens + its own token; on a
//    mismatch (a < w, or the drafter disagreeing at its pending position)
//    every stage j < i is resynced to O_i (reading R2) and its epoch bumped, so
//    a stale in-flight result is discarded (reading R9).
namespace {
struct Shared {
  std::mutex mu;
  std::condition_variable cv;
  std::vector<std::vector<int32_t>> O;        // committed buffer per stage
  std::vector<unsigned> epoch;
  std::vector<int> pending;                    // 1: resync to O of `target_of`
  std::vector<std::vector<int32_t>> target;
  bool done = false;
  ps_status err = PS_OK;
  std::string err_msg;
};

bool extends(const std::vector<int32_t>& a, const std::vector<int32_t>& b) {   // a extends b
  return a.size() >= b.size() && std::equal(b.begin(), b.end(), a.begin());
}

// resync every stage j < i to O_i (caller holds the lock)
void post_rollback(Shared& sh, int i, ps_run_stats* stt) {
  for (int j = i - 1; j >= 0; --j) {
    if (extends(sh.O[j], sh.O[i])) continue;             // already consistent
    sh.target[j] = sh.O[i];
    sh.pending[j] = 1;
    sh.O[j] = sh.O[i];                                    // the committed view is resynced now
    ++sh.epoch[j];
    if (j < 8) stt->rollbacks[j]++;
  }
}
}  // namespace

static ps_status pipespec_async(ps_stage* const* S, int k, int n_prompt, const ps_run_opts* o,
                                std::vector<int32_t>& gen, ps_run_stats* stt) {
  const int K = k - 1;
  Shared sh;
  sh.O.resize(k);
  sh.epoch.assign(k, 0);
  sh.pending.assign(k, 0);
  sh.target.resize(k);
  for (int i = 0; i < k; ++i) {
    if (tokens_of(S[i], sh.O[i]) != PS_OK) return PS_E_CUDA;
  }
  int max_gamma = 1;
  for (int i = 1; i < k; ++i) max_gamma = std::max(max_gamma, o->gamma ? o->gamma[i] : 8);
  int max_look = 0;
  for (int i = 1; i < k; ++i) max_look = std::max(max_look, o->lookahead ? o->lookahead[i] : 0);
  const int max_lead = std::max(o->max_lead, std::max(2 * max_gamma + 2, max_look + 1));
  const size_t target_len = (size_t)n_prompt + (size_t)o->max_new_tokens;
  auto finished = [&]() {
    const auto& OK = sh.O[K];
    if (OK.size() >= target_len) return true;
    return o->eos_id >= 0 && std::find(OK.begin() + n_prompt, OK.end(), o->eos_id) != OK.end();
  };
  auto fail_all = [&](ps_status st) {
    std::lock_guard<std::mutex> g(sh.mu);
    if (sh.err == PS_OK) { sh.err = st; sh.err_msg = ps_last_error(); }
    sh.done = true;
    sh.cv.notify_all();
  };

  auto worker = [&](int i) {
    ps_stage* me = S[i];
    const int gamma = (i > 0 && o->gamma) ? o->gamma[i] : 8;
    const int look = (i > 0 && o->lookahead) ? o->lookahead[i] : 0;
    std::vector<int32_t> mine, window, resync_to;
    for (;;) {
      unsigned ep;
      bool do_resync = false;
      int kind = 0;   // 0 draft, 1 verify, 2 AR
      {
        std::unique_lock<std::mutex> lk(sh.mu);
        for (;;) {
          if (sh.done) return;
          if (sh.pending[i]) {                        // apply a rollback posted by a later stage
            resync_to = sh.target[i];
            sh.pending[i] = 0;
            do_resync = true;
            break;
          }
          if (i < K && sh.O[i].size() >= sh.O[i + 1].size() + (size_t)max_lead) {   // bounded draft ring
            sh.cv.wait(lk);
            continue;
          }
          if (i == 0) { kind = 0; break; }
          mine = sh.O[i];
          const auto& P = sh.O[i - 1];
          const size_t n = mine.size();
          if (P.size() >= n && P[n - 1] != mine[n - 1]) {   // drafter disagrees at my pending token
            post_rollback(sh, i, stt);
            sh.cv.notify_all();
          }
          const auto& P2 = sh.O[i - 1];
          size_t avail = 0;
          if (P2.size() > n && std::equal(mine.begin(), mine.end(), P2.begin())) avail = P2.size() - n;
          if (avail >= (size_t)std::max(1, look)) {
            const size_t w = std::min(avail, (size_t)gamma);
            window.assign(P2.begin() + n, P2.begin() + n + w);
            kind = 1;
            break;
          }
          if (look == 0) { window.clear(); kind = 2; break; }
          sh.cv.wait(lk);
        }
        ep = sh.epoch[i];
      }
      if (do_resync) {
        if (ps_resync(me, resync_to.data(), (int32_t)resync_to.size()) != PS_OK) return fail_all(PS_E_CUDA);
        continue;
      }
      // ---- device work, outside the lock
      const long long t0 = now_ns();
      int32_t a = 0, nxt = 0;
      ps_status st;
      if (kind == 0) st = ps_draft(me, 1, &nxt);
      else st = ps_verify(me, window.data(), (int32_t)window.size(), &a, &nxt, nullptr);
      if (st != PS_OK) return fail_all(st);
      const long long dt = now_ns() - t0;
      std::vector<int32_t> now;
      if (tokens_of(me, now) != PS_OK) return fail_all(PS_E_CUDA);
      {
        std::lock_guard<std::mutex> g(sh.mu);
        if (i < 8) { stt->steps[i]++; stt->busy_ns[i] += dt; if (kind == 1) stt->verify_steps[i]++; }
        if (sh.done) return;
        if (sh.epoch[i] != ep) continue;              // rolled back meanwhile: result is stale
        sh.O[i] = now;
        if (kind == 1 && i == K) stt->accept_hist[std::min(a + 1, 63)]++;
        if (kind == 1 && a < (int)window.size()) post_rollback(sh, i, stt);
        if (i == K && finished()) sh.done = true;
        sh.cv.notify_all();
      }
    }
  };
  std::vector<std::thread> th;
  for (int i = 0; i < k; ++i) th.emplace_back(worker, i);
  for (auto& t : th) t.join();
  if (sh.err != PS_OK) return sh.err;
  gen.assign(sh.O[K].begin() + n_prompt, sh.O[K].end());
  return PS_OK;
}

extern "C" ps_status ps_pipeline_run(ps_stage* const* S, int32_t k, const int32_t* prompt, int32_t n_prompt,
                                     const ps_run_opts* o, int32_t* out, int32_t* out_len, ps_run_stats* stats) {
  if (!S || k < 1 || k > 8 || !prompt || n_prompt < 1 || !o || !out || !out_len) return PS_E_INVALID;
  if (o->max_new_tokens < 1) return PS_E_INVALID;
  ps_run_stats local;
  ps_run_stats* stt = stats ? stats : &local;
  memset(stt, 0, sizeof *stt);
  const int K = k - 1;
  ps_status st;
  std::vector<int32_t> prm(prompt, prompt + n_prompt);
  for (int i = 0; i < k; ++i)
    if ((st = ps_prefill(S[i], prm.data(), n_prompt)) != PS_OK) return st;
  std::vector<int32_t> gen;
  const long long t_start = now_ns();
  auto done = [&]() {
    if ((int)gen.size() >= o->max_new_tokens) return true;
    return o->eos_id >= 0 && std::find(gen.begin(), gen.end(), o->eos_id) != gen.end();
  };
  if (o->mode == PS_MODE_AR || K == 0) {
    while (!done()) {
      int32_t t;
      long long t0 = now_ns();
      if ((st = ps_draft(S[K], 1, &t)) != PS_OK) return st;
      stt->steps[K]++;
      stt->busy_ns[K] += now_ns() - t0;
      gen.push_back(t);
    }
  } else if (o->mode == PS_MODE_SYNC_SD) {
    const int gamma = o->gamma ? o->gamma[K] : 8;
    std::vector<int32_t> ctx;
    while (!done()) {
      if ((st = tokens_of(S[K], ctx)) != PS_OK) return st;
      std::vector<int32_t> d;
      if ((st = produce(S, K - 1, ctx, gamma, o, d, stt)) != PS_OK) return st;
      int32_t a, nxt;
      long long t0 = now_ns();
      if ((st = ps_verify(S[K], d.data(), (int32_t)d.size(), &a, &nxt, nullptr)) != PS_OK) return st;
      stt->steps[K]++;
      stt->verify_steps[K]++;
      stt->busy_ns[K] += now_ns() - t0;
      if (a < (int)d.size()) stt->rollbacks[K - 1]++;
      stt->accept_hist[std::min(a + 1, 63)]++;
      gen.insert(gen.end(), d.begin(), d.begin() + a);
      gen.push_back(nxt);
    }
  } else if (o->mode == PS_MODE_PIPESPEC) {
    if ((st = pipespec_async(S, k, n_prompt, o, gen, stt)) != PS_OK) return st;
  } else {
    return PS_E_INVALID;
  }
  stt->wall_ns = now_ns() - t_start;
  if (o->eos_id >= 0) {
    auto it = std::find(gen.begin(), gen.end(), o->eos_id);
    if (it != gen.end()) gen.erase(it + 1, gen.end());
  }
  if ((int)gen.size() > o->max_new_tokens) gen.resize(o->max_new_tokens);
  std::copy(gen.begin(), gen.end(), out);
  *out_len = (int32_t)gen.size();
  stt->tokens = *out_len;
  return PS_OK;
}
