// ps_pipeline.cu — ps_pipeline_run: Algorithm 1 over k
// stages.  AR and synchronous (tiered) SD are driven from the calling thread;
// PIPESPEC runs one host thread per stage over the board of ps_board.h, or one
// process per stage (ps_pipeline_run_rank) over the same board in shared
// memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/pipespec.h"
#include "ps_board.h"

ps_status fail(ps_status code, const char* fmt, ...);   // ps_stage.cu: thread-local message

namespace {
ps_status tokens_of(ps_stage* s, std::vector<int32_t>& v) {
  int64_t n = 0;
  ps_status st = ps_stage_tokens(s, nullptr, 0, &n);
  if (st != PS_OK) return st;
  v.resize((size_t)n);
  return ps_stage_tokens(s, v.data(), n, &n);
}

// Event log of the synchronous modes (same entries as the board's).
struct SyncLog {
  const ps_run_opts* o;
  ps_run_stats* st;
  long long t_start;
  int64_t n = 0;
  void add(int stage, int kind, int64_t len, int w, int a, int next, int origin, const int32_t* window) {
    if (!o->event_log || n >= o->event_cap) {
      if (o->event_log) st->events_dropped++;
      return;
    }
    ps_event& e = o->event_log[n++];
    memset(&e, 0, sizeof e);
    e.t_ns = now_ns() - t_start;
    e.stage = stage;
    e.kind = kind;
    e.n = (int32_t)len;
    e.w = w;
    e.a = a;
    e.next = next;
    e.origin = origin;
    for (int j = 0; j < w && j < 32; ++j) e.window[j] = window[j];
  }
};

// One AR step of stage i (a draft step for i = 0).
ps_status ar_step(ps_stage* const* S, int i, const ps_run_opts* o, ps_run_stats* stt, SyncLog& lg, int32_t* t) {
  int64_t n = 0;
  ps_status st = ps_stage_tokens(S[i], nullptr, 0, &n);
  if (st != PS_OK) return st;
  const long long t0 = now_ns();
  if ((st = ps_draft(S[i], 1, t)) != PS_OK) return st;
  pad_step(o, i, t0);
  stt->steps[i]++;
  stt->busy_ns[i] += now_ns() - t0;
  lg.add(i, i == 0 ? PS_EV_DRAFT : PS_EV_AR, n, 0, 0, *t, -1, nullptr);
  return PS_OK;
}

// m AR steps of stage i in one ps_draft call (its forwards chained on the
// device, include/pipespec.h); per-step events and stats as m ar_step calls.
// Stages with a virtual latency (padded per step) take them one by one.
ps_status ar_steps(ps_stage* const* S, int i, const ps_run_opts* o, ps_run_stats* stt, SyncLog& lg, int m,
                   std::vector<int32_t>& out) {
  if (m <= 1 || (o->virtual_ns && o->virtual_ns[i] > 0)) {
    for (int j = 0; j < m; ++j) {
      int32_t t;
      ps_status st = ar_step(S, i, o, stt, lg, &t);
      if (st != PS_OK) return st;
      out.push_back(t);
    }
    return PS_OK;
  }
  int64_t n = 0;
  ps_status st = ps_stage_tokens(S[i], nullptr, 0, &n);
  if (st != PS_OK) return st;
  const long long t0 = now_ns();
  std::vector<int32_t> t(m);
  if ((st = ps_draft(S[i], m, t.data())) != PS_OK) return st;
  stt->steps[i] += m;
  stt->busy_ns[i] += now_ns() - t0;
  for (int j = 0; j < m; ++j) {
    lg.add(i, i == 0 ? PS_EV_DRAFT : PS_EV_AR, n + j, 0, 0, t[j], -1, nullptr);
    out.push_back(t[j]);
  }
  return PS_OK;
}

// One verify step of stage i over window d.
ps_status verify_step(ps_stage* const* S, int i, const std::vector<int32_t>& d, const ps_run_opts* o,
                      ps_run_stats* stt, SyncLog& lg, int32_t* a, int32_t* nxt) {
  int64_t n = 0;
  ps_status st = ps_stage_tokens(S[i], nullptr, 0, &n);
  if (st != PS_OK) return st;
  const long long t0 = now_ns();
  if ((st = ps_verify(S[i], d.data(), (int32_t)d.size(), a, nxt, nullptr)) != PS_OK) return st;
  pad_step(o, i, t0);
  stt->steps[i]++;
  stt->verify_steps[i]++;
  stt->busy_ns[i] += now_ns() - t0;
  if (*a < (int)d.size()) stt->rollbacks[i - 1]++;
  lg.add(i, PS_EV_VERIFY, n, (int)d.size(), *a, *nxt, -1, d.data());
  return PS_OK;
}

// m greedy tokens of stage i given context ctx = O_{i+1} (stage i is left
// holding ctx ++ out): stage 0 drafts autoregressively; stage i>0 runs sync SD
// with stage i-1 (tiered synchronous speculative decoding).
ps_status produce(ps_stage* const* S, int i, const std::vector<int32_t>& ctx, int m, const ps_run_opts* o,
                  std::vector<int32_t>& out, ps_run_stats* stt, SyncLog& lg) {
  ps_status st = ps_resync(S[i], ctx.data(), (int32_t)ctx.size());   // rollback cascade, lazy KV catch-up
  if (st != PS_OK) return st;
  lg.add(i, PS_EV_RESYNC, (int64_t)ctx.size(), 0, 0, 0, i + 1, nullptr);
  out.clear();
  const int gamma = i > 0 ? opt_gamma(o, i) : 0;
  while ((int)out.size() < m) {
    if (i == 0 || gamma == 0) {
      if ((st = ar_steps(S, i, o, stt, lg, m - (int)out.size(), out)) != PS_OK) return st;
      continue;
    }
    std::vector<int32_t> cur = ctx;
    cur.insert(cur.end(), out.begin(), out.end());
    std::vector<int32_t> d;
    if ((st = produce(S, i - 1, cur, gamma, o, d, stt, lg)) != PS_OK) return st;
    int32_t a, nxt;
    if ((st = verify_step(S, i, d, o, stt, lg, &a, &nxt)) != PS_OK) return st;
    out.insert(out.end(), d.begin(), d.begin() + a);
    out.push_back(nxt);
  }
  out.resize(m);
  return PS_OK;
}

ps_status real_draft1(void* s, int32_t* t) { return ps_draft((ps_stage*)s, 1, t); }
ps_status real_verify(void* s, const int32_t* w, int32_t n, int32_t* a, int32_t* nx) {
  // asynchronous pass + wait: the host thread is free between the launch and
  // the commit (ps_verify_async / ps_verify_wait, include/pipespec.h)
  ps_verify_ticket tk;
  ps_status st = ps_verify_async((ps_stage*)s, w, n, &tk);
  if (st != PS_OK) return st;
  return ps_verify_wait((ps_stage*)s, a, nx);
}
ps_status real_resync(void* s, const int32_t* t, int32_t n) { return ps_resync((ps_stage*)s, t, n); }
ps_status real_tokens(void* s, std::vector<int32_t>& v) { return tokens_of((ps_stage*)s, v); }
StageOps real_ops(ps_stage* s) { return StageOps{s, real_draft1, real_verify, real_resync, real_tokens}; }

const std::string& last_error_str() {
  static thread_local std::string s;
  s = ps_last_error();
  return s;
}

// Validate the per-stage windows of the speculative modes: 1 <= gamma_i <=
// max_window of stage i.  S holds all k stages, or (rank >= 1) only stage `rank`.
ps_status check_gammas(ps_stage* const* S, int k, const ps_run_opts* o, int rank = -1) {
  if (o->mode == PS_MODE_AR) return PS_OK;
  for (int i = 1; i < k; ++i) {
    if (rank >= 0 && i != rank) continue;
    ps_stage_info inf;
    ps_status st = ps_stage_get_info(S[rank >= 0 ? 0 : i], &inf);
    if (st != PS_OK) return st;
    const int g = opt_gamma(o, i);
    if (g < 1 || g > inf.max_window)
      return fail(PS_E_INVALID, "gamma[%d] = %d not in [1, max_window = %d]", i, g, (int)inf.max_window);
  }
  return PS_OK;
}

void fwd_totals(ps_stage* s, double* ms, int64_t* n) {
  ps_stage_info inf;
  if (ps_stage_get_info(s, &inf) == PS_OK) { *ms = inf.sum_fwd_ms; *n = inf.n_fwd; }
}
}  // namespace

extern "C" ps_status ps_pipeline_run(ps_stage* const* S, int32_t k, const int32_t* prompt, int32_t n_prompt,
                                     const ps_run_opts* o, int32_t* out, int32_t* out_len, ps_run_stats* stats) {
  if (!S || k < 1 || k > 8 || !prompt || n_prompt < 1 || !o || !out || !out_len)
    return fail(PS_E_INVALID, "ps_pipeline_run: NULL argument or k not in 1..8");
  if (o->max_new_tokens < 1) return fail(PS_E_INVALID, "max_new_tokens < 1");
  if (o->mode != PS_MODE_AR && o->mode != PS_MODE_SYNC_SD && o->mode != PS_MODE_PIPESPEC)
    return fail(PS_E_INVALID, "unknown mode %d", o->mode);
  if (o->event_log && o->event_cap < 0) return fail(PS_E_INVALID, "event_cap < 0");
  ps_status st;
  if ((st = check_gammas(S, k, o)) != PS_OK) return st;
  ps_run_stats local;
  ps_run_stats* stt = stats ? stats : &local;
  memset(stt, 0, sizeof *stt);
  const int K = k - 1;
  std::vector<int32_t> prm(prompt, prompt + n_prompt);
  for (int i = 0; i < k; ++i)
    if ((st = ps_prefill(S[i], prm.data(), n_prompt)) != PS_OK) return st;
  if (o->alpha && K > 0) {
    // synthetic acceptance (reading R24): the target stream S is M_K's own AR
    // decode, then every stage i < K emits the chained override token
    std::vector<int32_t> tgt(o->max_new_tokens);
    if ((st = ps_draft(S[K], o->max_new_tokens, tgt.data())) != PS_OK) return st;
    for (int i = 0; i < K; ++i)
      if ((st = ps_set_synthetic(S[i], tgt.data(), o->max_new_tokens, n_prompt, i, K, o->alpha + i, o->seed)) != PS_OK)
        return st;
    if ((st = ps_kv_rollback(S[K], n_prompt)) != PS_OK) return st;
  }
  double ms0[8] = {};
  int64_t n0[8] = {};
  for (int i = 0; i < k; ++i) fwd_totals(S[i], &ms0[i], &n0[i]);
  std::vector<int32_t> gen;
  const long long t_start = now_ns();
  SyncLog lg{o, stt, t_start};
  auto done = [&]() {
    if ((int)gen.size() >= o->max_new_tokens) return true;
    return o->eos_id >= 0 && std::find(gen.begin(), gen.end(), o->eos_id) != gen.end();
  };
  if (o->mode == PS_MODE_AR || K == 0) {
    if (o->eos_id < 0) {                 // no early stop: one chained ps_draft
      if ((st = ar_steps(S, K, o, stt, lg, o->max_new_tokens, gen)) != PS_OK) return st;
    }
    while (!done()) {
      int32_t t;
      if ((st = ar_step(S, K, o, stt, lg, &t)) != PS_OK) return st;
      gen.push_back(t);
    }
    stt->n_events = lg.n;
  } else if (o->mode == PS_MODE_SYNC_SD) {
    std::vector<int32_t> ctx;
    while (!done()) {
      if ((st = tokens_of(S[K], ctx)) != PS_OK) return st;
      std::vector<int32_t> d;
      if ((st = produce(S, K - 1, ctx, opt_gamma(o, K), o, d, stt, lg)) != PS_OK) return st;
      int32_t a, nxt;
      if ((st = verify_step(S, K, d, o, stt, lg, &a, &nxt)) != PS_OK) return st;
      stt->accept_hist[std::min(a + 1, 63)]++;
      gen.insert(gen.end(), d.begin(), d.begin() + a);
      gen.push_back(nxt);
    }
    stt->n_events = lg.n;
  } else {
    const int cap = n_prompt + o->max_new_tokens + std::max(o->max_lead, 0) + 4 * 64 + 64;
    const int ev_cap = o->event_log ? std::max(o->event_cap, 0) : 0;
    std::vector<uint8_t> mem;
    Board* b = board_on_heap(mem, k, cap, ev_cap);
    std::vector<StageOps> ops;
    for (int i = 0; i < k; ++i) ops.push_back(real_ops(S[i]));
    st = run_board_threads(b, ops.data(), k, n_prompt, o, gen, stt, last_error_str);
    std::string msg = b->err_msg;
    board_destroy(b);
    if (st != PS_OK) return fail(st, "%s", msg.c_str());   // a worker's error, on the caller's thread
  }
  stt->wall_ns = now_ns() - t_start;
  for (int i = 0; i < k; ++i) {
    double ms = 0;
    int64_t n = 0;
    fwd_totals(S[i], &ms, &n);
    stt->fwd_ns[i] = (int64_t)((ms - ms0[i]) * 1e6);
    stt->n_fwd[i] = n - n0[i];
  }
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

extern "C" ps_status ps_board_create(const char* name, int32_t k, int32_t capacity) {
  if (!name || k < 1 || k > 8 || capacity < 2) return fail(PS_E_INVALID, "ps_board_create: bad arguments");
  ps_status st = board_create_shm(name, k, capacity);
  if (st != PS_OK) return fail(st, "cannot create shared-memory board %s", name);
  return PS_OK;
}

extern "C" ps_status ps_board_unlink(const char* name) {
  if (!name) return fail(PS_E_INVALID, "NULL board name");
  return shm_unlink(name) == 0 ? PS_OK : fail(PS_E_INVALID, "cannot unlink board %s", name);
}

// ---------------------------------------------------------------- tensor-parallel stage groups
// A stage M_rank that is tensor parallel over n ranks driven by THIS process
// (one host thread per member, ps_tp_connect_local): every board step runs on
// all members concurrently; the members agree bit for bit, the leader's
// result is the stage's.
namespace {
struct Group {
  std::vector<ps_stage*> st;
};
template <class F>
ps_status all_members(Group* g, F f) {
  const int n = (int)g->st.size();
  if (n == 1) return f(0);
  std::vector<ps_status> r(n, PS_OK);
  std::vector<std::string> err(n);
  std::vector<std::thread> th;
  for (int i = 1; i < n; ++i)
    th.emplace_back([&, i] {
      r[i] = f(i);
      if (r[i] != PS_OK) err[i] = ps_last_error();
    });
  r[0] = f(0);
  if (r[0] != PS_OK) err[0] = ps_last_error();
  for (auto& t : th) t.join();
  for (int i = 0; i < n; ++i)
    if (r[i] != PS_OK) return fail(r[i], "tensor-parallel member %d: %s", i, err[i].c_str());
  return PS_OK;
}
ps_status grp_draft1(void* c, int32_t* t) {
  Group* g = (Group*)c;
  std::vector<int32_t> tt(g->st.size());
  ps_status st = all_members(g, [&](int i) { return ps_draft(g->st[i], 1, &tt[i]); });
  if (st != PS_OK) return st;
  for (size_t i = 1; i < tt.size(); ++i)
    if (tt[i] != tt[0]) return fail(PS_E_CUDA, "tensor-parallel members disagree (%d vs %d)", tt[i], tt[0]);
  *t = tt[0];
  return PS_OK;
}
ps_status grp_verify(void* c, const int32_t* w, int32_t n, int32_t* a, int32_t* nx) {
  Group* g = (Group*)c;
  std::vector<int32_t> aa(g->st.size()), nn(g->st.size());
  ps_status st = all_members(g, [&](int i) {
    ps_verify_ticket tk;
    ps_status s2 = ps_verify_async(g->st[i], w, n, &tk);
    return s2 != PS_OK ? s2 : ps_verify_wait(g->st[i], &aa[i], &nn[i]);
  });
  if (st != PS_OK) return st;
  for (size_t i = 1; i < aa.size(); ++i)
    if (aa[i] != aa[0] || nn[i] != nn[0]) return fail(PS_E_CUDA, "tensor-parallel members disagree on (a, next)");
  *a = aa[0];
  *nx = nn[0];
  return PS_OK;
}
ps_status grp_resync(void* c, const int32_t* t, int32_t n) {
  Group* g = (Group*)c;
  return all_members(g, [&](int i) { return ps_resync(g->st[i], t, n); });
}
ps_status grp_tokens(void* c, std::vector<int32_t>& v) { return tokens_of(((Group*)c)->st[0], v); }
}  // namespace

extern "C" ps_status ps_pipeline_run_rank_group(ps_stage* const* group, int32_t n, int32_t rank, int32_t k,
                                                const char* board, const int32_t* prompt, int32_t n_prompt,
                                                const ps_run_opts* o, int32_t* out, int32_t* out_len,
                                                ps_run_stats* stats) {
  if (!group || n < 1 || n > 8 || !board || !prompt || n_prompt < 1 || !o || !out || !out_len ||
      o->max_new_tokens < 1)
    return fail(PS_E_INVALID, "ps_pipeline_run_rank_group: bad argument");
  for (int i = 0; i < n; ++i)
    if (!group[i]) return fail(PS_E_INVALID, "NULL group member %d", i);
  if (o->mode != PS_MODE_PIPESPEC) return fail(PS_E_INVALID, "per-rank runs are PS_MODE_PIPESPEC only");
  if (o->alpha) return fail(PS_E_INVALID, "per-rank runs take their synthetic override from ps_set_synthetic");
  ps_status st;
  if (rank > 0 && (st = check_gammas(group, k, o, rank)) != PS_OK) return st;
  Group g{std::vector<ps_stage*>(group, group + n)};
  if ((st = all_members(&g, [&](int i) { return ps_prefill(g.st[i], prompt, n_prompt); })) != PS_OK) return st;
  ps_run_stats local;
  ps_run_stats* stt = stats ? stats : &local;
  memset(stt, 0, sizeof *stt);
  double ms0 = 0;
  int64_t n0 = 0;
  fwd_totals(group[0], &ms0, &n0);
  std::string err;
  const StageOps ops = n == 1 ? real_ops(group[0]) : StageOps{&g, grp_draft1, grp_verify, grp_resync, grp_tokens};
  st = run_rank(ops, rank, k, board, n_prompt, o, out, out_len, stt, last_error_str, &err);
  if (st != PS_OK) return fail(st, "%s", err.c_str());
  if (rank >= 0 && rank < 8) {
    double ms = 0;
    int64_t nf = 0;
    fwd_totals(group[0], &ms, &nf);
    stt->fwd_ns[rank] = (int64_t)((ms - ms0) * 1e6);
    stt->n_fwd[rank] = nf - n0;
  }
  return PS_OK;
}

extern "C" ps_status ps_pipeline_run_rank(ps_stage* stage, int32_t rank, int32_t k, const char* board,
                                          const int32_t* prompt, int32_t n_prompt, const ps_run_opts* o,
                                          int32_t* out, int32_t* out_len, ps_run_stats* stats) {
  return ps_pipeline_run_rank_group(&stage, 1, rank, k, board, prompt, n_prompt, o, out, out_len, stats);
}
