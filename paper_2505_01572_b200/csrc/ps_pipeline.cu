// ps_pipeline.cu — ps_pipeline_run: Algorithm 1 over k
// stages.  AR and synchronous (tiered) SD are driven from the calling thread;
// PIPESPEC runs one host thread per stage.
#include <cuda_runtime.h>

#include <fcntl.h>
#include <pthread.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

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
#include "../../include/pipespec_test.h"

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
// Algorithm 1 with one host thread (or process) per stage.  The
// shared state -- committed buffers O_i, epochs, pending resync targets -- is
// a flat "board" under one process-shared mutex, so the same code runs the
// stages as threads of one process (board on the heap, ps_pipeline_run) or as
// one process per GPU (board in POSIX shared memory, ps_pipeline_run_rank).
// Every device call runs outside the lock on the stage's own stream.
//  * stage 0 drafts one token per step ("Generate next token, append to O_0")
//    while it is less than max_lead tokens ahead of stage 1;
//  * stage i>0 takes window = O_{i-1}[n : n + min(avail, gamma_i)] when at least
//    max(1, lookahead_i) valid drafts exist, else an AR step (lookahead 0) or
//    waits; verifies; publishes the accepted tokens + its own token; on a
//    mismatch (a < w, or the drafter disagreeing at its pending position)
//    every stage j < i is resynced to O_i (reading R2) and its epoch bumped, so
//    a stale in-flight result is discarded (reading R9).
namespace {
constexpr uint32_t kBoardMagic = 0x50535042u;   // "PSPB"
constexpr long long kBoardTimeoutNs = 600ll * 1000 * 1000 * 1000;

struct Board {
  uint32_t magic;
  int32_t k, cap, n_prompt;
  pthread_mutex_t mu;
  pthread_cond_t cv;
  int32_t ready, done, err, pad;
  char err_msg[256];
  int64_t len[8], tlen[8];
  uint32_t epoch[8];
  int32_t pending[8];
  int64_t t_start;
  ps_run_stats stats;
  // followed by int32 O[8][cap], T[8][cap]
  int32_t* O(int i) { return reinterpret_cast<int32_t*>(this + 1) + (size_t)i * cap; }
  int32_t* T(int i) { return reinterpret_cast<int32_t*>(this + 1) + (size_t)(8 + i) * cap; }
};
size_t board_bytes(int cap) { return sizeof(Board) + (size_t)16 * cap * sizeof(int32_t); }

void board_init(Board* b, int k, int cap) {
  memset(b, 0, sizeof(Board));
  b->k = k;
  b->cap = cap;
  pthread_mutexattr_t ma;
  pthread_mutexattr_init(&ma);
  pthread_mutexattr_setpshared(&ma, PTHREAD_PROCESS_SHARED);
  pthread_mutex_init(&b->mu, &ma);
  pthread_mutexattr_destroy(&ma);
  pthread_condattr_t ca;
  pthread_condattr_init(&ca);
  pthread_condattr_setpshared(&ca, PTHREAD_PROCESS_SHARED);
  pthread_condattr_setclock(&ca, CLOCK_MONOTONIC);
  pthread_cond_init(&b->cv, &ca);
  pthread_condattr_destroy(&ca);
  __atomic_store_n(&b->magic, kBoardMagic, __ATOMIC_RELEASE);
}

struct Lock {
  Board* b;
  explicit Lock(Board* b_) : b(b_) { pthread_mutex_lock(&b->mu); }
  ~Lock() { pthread_mutex_unlock(&b->mu); }
};
// wait on the board (lock held) at most 50 ms: every waiter re-checks its
// predicate and the global deadline, so a dead peer process ends the run
void board_wait(Board* b) {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  ts.tv_nsec += 50 * 1000 * 1000;
  if (ts.tv_nsec >= 1000000000) { ts.tv_sec += 1; ts.tv_nsec -= 1000000000; }
  pthread_cond_timedwait(&b->cv, &b->mu, &ts);
}
void board_fail(Board* b, ps_status st, const char* msg) {   // lock held
  if (b->err == PS_OK) {
    b->err = st;
    snprintf(b->err_msg, sizeof b->err_msg, "%s", msg ? msg : "");
  }
  b->done = 1;
  pthread_cond_broadcast(&b->cv);
}

bool prefix_of(const int32_t* a, int64_t na, const int32_t* b, int64_t nb) {   // a extends b
  return na >= nb && std::equal(b, b + nb, a);
}

// resync every stage j < i to O_i (lock held)
void post_rollback(Board* b, int i) {
  for (int j = i - 1; j >= 0; --j) {
    if (prefix_of(b->O(j), b->len[j], b->O(i), b->len[i])) continue;   // already consistent
    std::copy(b->O(i), b->O(i) + b->len[i], b->T(j));
    b->tlen[j] = b->len[i];
    b->pending[j] = 1;
    std::copy(b->O(i), b->O(i) + b->len[i], b->O(j));   // the committed view is resynced now
    b->len[j] = b->len[i];
    ++b->epoch[j];
    b->stats.rollbacks[j]++;
  }
}

// What a worker calls on its stage (the real ps_stage, or a test double).
struct StageOps {
  void* ctx;
  ps_status (*draft1)(void*, int32_t*);
  ps_status (*verify)(void*, const int32_t*, int32_t, int32_t*, int32_t*);
  ps_status (*resync)(void*, const int32_t*, int32_t);
  ps_status (*tokens)(void*, std::vector<int32_t>&);
};
ps_status real_draft1(void* s, int32_t* t) { return ps_draft((ps_stage*)s, 1, t); }
ps_status real_verify(void* s, const int32_t* w, int32_t n, int32_t* a, int32_t* nx) {
  return ps_verify((ps_stage*)s, w, n, a, nx, nullptr);
}
ps_status real_resync(void* s, const int32_t* t, int32_t n) { return ps_resync((ps_stage*)s, t, n); }
ps_status real_tokens(void* s, std::vector<int32_t>& v) { return tokens_of((ps_stage*)s, v); }
StageOps real_ops(ps_stage* s) { return StageOps{s, real_draft1, real_verify, real_resync, real_tokens}; }

// Stage i's loop (Alg.1 lines 95-110 for i > 0, 98-100 for i = 0).
void board_worker(Board* b, int i, const StageOps& ops, const ps_run_opts* o, const std::string& (*errf)()) {
  const int k = b->k, K = k - 1;
  const int gamma = (i > 0 && o->gamma) ? o->gamma[i] : 8;
  const int look = (i > 0 && o->lookahead) ? o->lookahead[i] : 0;
  int max_gamma = 1, max_look = 0;
  for (int j = 1; j < k; ++j) {
    max_gamma = std::max(max_gamma, o->gamma ? o->gamma[j] : 8);
    max_look = std::max(max_look, o->lookahead ? o->lookahead[j] : 0);
  }
  const int64_t max_lead = std::max<int64_t>(o->max_lead, std::max(2 * max_gamma + 2, max_look + 1));
  const int64_t target_len = (int64_t)b->n_prompt + o->max_new_tokens;
  auto finished = [&]() {
    if (b->len[K] >= target_len) return true;
    return o->eos_id >= 0 && std::find(b->O(K) + b->n_prompt, b->O(K) + b->len[K], o->eos_id) != b->O(K) + b->len[K];
  };
  std::vector<int32_t> mine, window, resync_to, now;
  for (;;) {
    uint32_t ep;
    bool do_resync = false;
    int kind = 0;   // 0 draft, 1 verify, 2 AR
    {
      Lock lk(b);
      for (;;) {
        if (b->done) return;
        if (now_ns() - b->t_start > kBoardTimeoutNs) return board_fail(b, PS_E_STALE, "pipeline timed out");
        if (b->pending[i]) {                          // apply a rollback posted by a later stage
          resync_to.assign(b->T(i), b->T(i) + b->tlen[i]);
          b->pending[i] = 0;
          do_resync = true;
          break;
        }
        if (i < K && b->len[i] >= b->len[i + 1] + max_lead) { board_wait(b); continue; }   // bounded draft ring
        if (i == 0) { kind = 0; break; }
        const int64_t n = b->len[i];
        mine.assign(b->O(i), b->O(i) + n);
        if (b->len[i - 1] >= n && b->O(i - 1)[n - 1] != mine[n - 1]) {   // drafter disagrees at my pending token
          post_rollback(b, i);
          pthread_cond_broadcast(&b->cv);
        }
        int64_t avail = 0;
        if (b->len[i - 1] > n && std::equal(mine.begin(), mine.end(), b->O(i - 1))) avail = b->len[i - 1] - n;
        if (avail >= std::max(1, look)) {
          const int64_t w = std::min<int64_t>(avail, gamma);
          window.assign(b->O(i - 1) + n, b->O(i - 1) + n + w);
          kind = 1;
          break;
        }
        if (look == 0) { window.clear(); kind = 2; break; }
        board_wait(b);
      }
      ep = b->epoch[i];
    }
    if (do_resync) {
      ps_status st = ops.resync(ops.ctx, resync_to.data(), (int32_t)resync_to.size());
      if (st != PS_OK) { Lock lk(b); return board_fail(b, st, errf().c_str()); }
      continue;
    }
    // ---- device work, outside the lock
    const long long t0 = now_ns();
    int32_t a = 0, nxt = 0;
    ps_status st = kind == 0 ? ops.draft1(ops.ctx, &nxt)
                             : ops.verify(ops.ctx, window.data(), (int32_t)window.size(), &a, &nxt);
    if (st == PS_OK) st = ops.tokens(ops.ctx, now);
    if (st != PS_OK) { Lock lk(b); return board_fail(b, st, errf().c_str()); }
    const long long dt = now_ns() - t0;
    {
      Lock lk(b);
      b->stats.steps[i]++;
      b->stats.busy_ns[i] += dt;
      if (kind == 1) b->stats.verify_steps[i]++;
      if (b->done) return;
      if (b->epoch[i] != ep) continue;               // rolled back meanwhile: result is stale
      if ((int64_t)now.size() > b->cap) return board_fail(b, PS_E_CAPACITY, "token buffer beyond board capacity");
      std::copy(now.begin(), now.end(), b->O(i));
      b->len[i] = (int64_t)now.size();
      if (kind == 1 && i == K) b->stats.accept_hist[std::min(a + 1, 63)]++;
      if (kind == 1 && a < (int)window.size()) post_rollback(b, i);
      if (i == K && finished()) b->done = 1;
      pthread_cond_broadcast(&b->cv);
    }
  }
}

const std::string& last_error_str() {
  static thread_local std::string s;
  s = ps_last_error();
  return s;
}

// Generated tokens of O_K (lock not needed: every worker has returned).
void board_result(Board* b, const ps_run_opts* o, std::vector<int32_t>& gen) {
  const int K = b->k - 1;
  gen.assign(b->O(K) + b->n_prompt, b->O(K) + b->len[K]);
  (void)o;
}

ps_status run_board_threads(Board* b, const StageOps* ops, int k, const int32_t* prompt, int n_prompt,
                            const ps_run_opts* o, std::vector<int32_t>& gen, ps_run_stats* stt,
                            const std::string& (*errf)()) {
  b->n_prompt = n_prompt;
  for (int i = 0; i < k; ++i) {
    std::vector<int32_t> v;
    ps_status st = ops[i].tokens(ops[i].ctx, v);
    if (st != PS_OK) return st;
    if ((int64_t)v.size() > b->cap) return PS_E_CAPACITY;
    std::copy(v.begin(), v.end(), b->O(i));
    b->len[i] = (int64_t)v.size();
  }
  (void)prompt;
  b->t_start = now_ns();
  std::vector<std::thread> th;
  for (int i = 0; i < k; ++i) th.emplace_back(board_worker, b, i, std::cref(ops[i]), o, errf);
  for (auto& t : th) t.join();
  memcpy(stt->steps, b->stats.steps, sizeof stt->steps);
  memcpy(stt->verify_steps, b->stats.verify_steps, sizeof stt->verify_steps);
  memcpy(stt->rollbacks, b->stats.rollbacks, sizeof stt->rollbacks);
  memcpy(stt->busy_ns, b->stats.busy_ns, sizeof stt->busy_ns);
  memcpy(stt->accept_hist, b->stats.accept_hist, sizeof stt->accept_hist);
  if (b->err != PS_OK) return b->err;
  board_result(b, o, gen);
  return PS_OK;
}
}  // namespace

static ps_status pipespec_async(ps_stage* const* S, int k, int n_prompt, const ps_run_opts* o,
                                std::vector<int32_t>& gen, ps_run_stats* stt, const int32_t* prompt) {
  int cap = 0;
  for (int i = 0; i < k; ++i) {
    ps_stage_info inf;
    if (ps_stage_get_info(S[i], &inf) != PS_OK) return PS_E_INVALID;
  }
  cap = n_prompt + o->max_new_tokens + std::max(o->max_lead, 0) + 4 * 64 + 64;
  std::vector<uint8_t> mem(board_bytes(cap) + 64);
  Board* b = reinterpret_cast<Board*>((reinterpret_cast<uintptr_t>(mem.data()) + 63) & ~(uintptr_t)63);
  board_init(b, k, cap);
  std::vector<StageOps> ops;
  for (int i = 0; i < k; ++i) ops.push_back(real_ops(S[i]));
  ps_status st = run_board_threads(b, ops.data(), k, prompt, n_prompt, o, gen, stt, last_error_str);
  pthread_cond_destroy(&b->cv);
  pthread_mutex_destroy(&b->mu);
  return st;
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
    if ((st = pipespec_async(S, k, n_prompt, o, gen, stt, prm.data())) != PS_OK) return st;
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

// ---------------------------------------------------------------- one process per stage
// The board in POSIX shared memory: stage i runs in its own process (its own
// GPU), the processes exchange only the committed token buffers, epochs and
// rollback targets through the board (SURVEY §8(e) "across stages: tiny
// messages ... pinned-host mailboxes").
namespace {
Board* board_open(const char* name, size_t* bytes) {
  const int fd = shm_open(name, O_RDWR, 0600);
  if (fd < 0) return nullptr;
  struct stat sb;
  if (fstat(fd, &sb) != 0 || (size_t)sb.st_size < sizeof(Board)) { close(fd); return nullptr; }
  void* p = mmap(nullptr, (size_t)sb.st_size, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return nullptr;
  Board* b = (Board*)p;
  if (__atomic_load_n(&b->magic, __ATOMIC_ACQUIRE) != kBoardMagic || board_bytes(b->cap) > (size_t)sb.st_size) {
    munmap(p, (size_t)sb.st_size);
    return nullptr;
  }
  *bytes = (size_t)sb.st_size;
  return b;
}

ps_status run_rank(const StageOps& ops, int rank, int k, const char* name, int n_prompt, const ps_run_opts* o,
                   int32_t* out, int32_t* out_len, ps_run_stats* stt, const std::string& (*errf)()) {
  size_t bytes = 0;
  Board* b = board_open(name, &bytes);
  if (!b) return PS_E_INVALID;
  ps_status result = PS_OK;
  std::vector<int32_t> v;
  ps_status st = ops.tokens(ops.ctx, v);
  {
    Lock lk(b);
    if (b->k != k || rank < 0 || rank >= k) {
      board_fail(b, PS_E_INVALID, "rank / k do not match the board");
    } else if (st != PS_OK || (int64_t)v.size() > b->cap) {
      board_fail(b, st != PS_OK ? st : PS_E_CAPACITY, "stage tokens");
    } else {
      std::copy(v.begin(), v.end(), b->O(rank));
      b->len[rank] = (int64_t)v.size();
      b->n_prompt = n_prompt;
      if (++b->ready == k) b->t_start = now_ns();      // the last stage to arrive starts the clock
      pthread_cond_broadcast(&b->cv);
      const long long t0 = now_ns();
      while (b->ready < k && !b->done) {
        if (now_ns() - t0 > 120ll * 1000 * 1000 * 1000) { board_fail(b, PS_E_STALE, "peers did not attach"); break; }
        board_wait(b);
      }
    }
  }
  if (!b->done) board_worker(b, rank, ops, o, errf);
  {
    Lock lk(b);
    while (!b->done) board_wait(b);                  // another stage ended the run
    result = (ps_status)b->err;
    if (result == PS_OK) {
      std::vector<int32_t> gen;
      board_result(b, o, gen);
      if (o->eos_id >= 0) {
        auto it = std::find(gen.begin(), gen.end(), o->eos_id);
        if (it != gen.end()) gen.erase(it + 1, gen.end());
      }
      if ((int)gen.size() > o->max_new_tokens) gen.resize(o->max_new_tokens);
      std::copy(gen.begin(), gen.end(), out);
      *out_len = (int32_t)gen.size();
      if (stt) {
        *stt = b->stats;
        stt->tokens = *out_len;
        stt->wall_ns = now_ns() - b->t_start;
      }
    }
  }
  munmap(b, bytes);
  return result;
}
}  // namespace

extern "C" ps_status ps_board_create(const char* name, int32_t k, int32_t capacity) {
  if (!name || k < 1 || k > 8 || capacity < 2) return PS_E_INVALID;
  const int fd = shm_open(name, O_CREAT | O_RDWR | O_TRUNC, 0600);
  if (fd < 0) return PS_E_INVALID;
  const size_t bytes = board_bytes(capacity);
  if (ftruncate(fd, (off_t)bytes) != 0) { close(fd); return PS_E_INVALID; }
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return PS_E_INVALID;
  board_init((Board*)p, k, capacity);
  munmap(p, bytes);
  return PS_OK;
}

extern "C" ps_status ps_board_unlink(const char* name) {
  if (!name) return PS_E_INVALID;
  return shm_unlink(name) == 0 ? PS_OK : PS_E_INVALID;
}

extern "C" ps_status ps_pipeline_run_rank(ps_stage* stage, int32_t rank, int32_t k, const char* board,
                                          const int32_t* prompt, int32_t n_prompt, const ps_run_opts* o,
                                          int32_t* out, int32_t* out_len, ps_run_stats* stats) {
  if (!stage || !board || !prompt || n_prompt < 1 || !o || !out || !out_len || o->max_new_tokens < 1)
    return PS_E_INVALID;
  if (o->mode != PS_MODE_PIPESPEC) return PS_E_INVALID;
  ps_status st = ps_prefill(stage, prompt, n_prompt);
  if (st != PS_OK) return st;
  return run_rank(real_ops(stage), rank, k, board, n_prompt, o, out, out_len, stats, last_error_str);
}

// ---------------------------------------------------------------- protocol test double
// A closed-form "model" on the host, so the board protocol (threads and
// processes, rollbacks, epochs) is testable without a GPU.  Stage K:
//   next(c) = (c[-1] * 7919 + |c| * 104729 + 13) mod V;
// stage i < K agrees with stage i+1 with probability alpha (hash of seed, i,
// |c|), else emits another token.  Never used by the product path.
namespace {
struct FakeStage {
  int i, k, V;
  double alpha;
  uint64_t seed;
  int sleep_us;
  std::vector<int32_t> toks;
  static uint64_t mix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
  }
  int32_t next_at(int level, const std::vector<int32_t>& c) const {
    int64_t t = ((int64_t)c.back() * 7919 + (int64_t)c.size() * 104729 + 13) % V;
    for (int j = k - 2; j >= level; --j) {
      const uint64_t h = mix(seed ^ ((uint64_t)j << 48) ^ (uint64_t)c.size());
      if ((double)(h >> 11) >= alpha * 9007199254740992.0) t = (t + 1 + (int64_t)(mix(h) % (uint64_t)(V - 1))) % V;
    }
    return (int32_t)t;
  }
  void nap() const { if (sleep_us > 0) usleep((useconds_t)(sleep_us * (1 + 3 * i))); }   // later stages are slower
  static ps_status draft1(void* p, int32_t* t) {
    FakeStage* s = (FakeStage*)p;
    *t = s->next_at(s->i, s->toks);
    s->toks.push_back(*t);
    s->nap();
    return PS_OK;
  }
  static ps_status verify(void* p, const int32_t* w, int32_t n, int32_t* a, int32_t* nx) {
    FakeStage* s = (FakeStage*)p;
    std::vector<int32_t> c = s->toks;
    int j = 0;
    int32_t pred = s->next_at(s->i, c);
    while (j < n && pred == w[j]) {
      c.push_back(w[j]);
      ++j;
      pred = s->next_at(s->i, c);
    }
    c.push_back(pred);
    s->toks = c;
    *a = j;
    *nx = pred;
    s->nap();
    return PS_OK;
  }
  static ps_status resync(void* p, const int32_t* t, int32_t n) {
    ((FakeStage*)p)->toks.assign(t, t + n);
    return PS_OK;
  }
  static ps_status tokens(void* p, std::vector<int32_t>& v) {
    v = ((FakeStage*)p)->toks;
    return PS_OK;
  }
  StageOps ops() { return StageOps{this, draft1, verify, resync, tokens}; }
};
const std::string& fake_err() {
  static thread_local std::string s = "fake stage error";
  return s;
}
}  // namespace

extern "C" ps_status ps_test_fake_run_rank(int32_t rank, int32_t k, const char* board, const int32_t* prompt,
                                           int32_t n_prompt, const ps_run_opts* o, int32_t vocab, double alpha,
                                           uint64_t seed, int32_t sleep_us, int32_t* out, int32_t* out_len,
                                           ps_run_stats* stats) {
  if (!prompt || n_prompt < 1 || !o || vocab < 2 || k < 1 || k > 8) return PS_E_INVALID;
  FakeStage f{rank, k, vocab, alpha, seed, sleep_us, std::vector<int32_t>(prompt, prompt + n_prompt)};
  return run_rank(f.ops(), rank, k, board, n_prompt, o, out, out_len, stats, fake_err);
}

extern "C" ps_status ps_test_fake_pipeline(int32_t k, const int32_t* prompt, int32_t n_prompt, const ps_run_opts* o,
                                           int32_t vocab, double alpha, uint64_t seed, int32_t sleep_us,
                                           int32_t* out, int32_t* out_len, ps_run_stats* stats) {
  if (!prompt || n_prompt < 1 || !o || vocab < 2 || k < 1 || k > 8 || !out || !out_len) return PS_E_INVALID;
  std::vector<FakeStage> fs;
  for (int i = 0; i < k; ++i)
    fs.push_back(FakeStage{i, k, vocab, alpha, seed, sleep_us, std::vector<int32_t>(prompt, prompt + n_prompt)});
  std::vector<StageOps> ops;
  for (auto& f : fs) ops.push_back(f.ops());
  const int cap = n_prompt + o->max_new_tokens + std::max(o->max_lead, 0) + 4 * 64 + 64;
  std::vector<uint8_t> mem(board_bytes(cap) + 64);
  Board* b = reinterpret_cast<Board*>((reinterpret_cast<uintptr_t>(mem.data()) + 63) & ~(uintptr_t)63);
  board_init(b, k, cap);
  ps_run_stats local;
  ps_run_stats* stt = stats ? stats : &local;
  memset(stt, 0, sizeof *stt);
  std::vector<int32_t> gen;
  const long long t0 = now_ns();
  ps_status st = run_board_threads(b, ops.data(), k, prompt, n_prompt, o, gen, stt, fake_err);
  pthread_cond_destroy(&b->cv);
  pthread_mutex_destroy(&b->mu);
  if (st != PS_OK) return st;
  if ((int)gen.size() > o->max_new_tokens) gen.resize(o->max_new_tokens);
  std::copy(gen.begin(), gen.end(), out);
  *out_len = (int32_t)gen.size();
  stt->tokens = *out_len;
  stt->wall_ns = now_ns() - t0;
  return PS_OK;
}
