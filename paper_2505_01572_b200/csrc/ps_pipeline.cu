// ps_pipeline.cu — ps_pipeline_run: Algorithm 1 over k
// stages.  AR and synchronous (tiered) SD are driven from the calling thread;
// PIPESPEC runs one host thread per stage.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstring>
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
  } else {
    return PS_E_INVALID;   // PS_MODE_PIPESPEC: see ps_pipeline_async (next build step)
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
