// ps_board.h — the async PipeSpec runtime's shared state and stage loop
// (Algorithm 1), shared by the product library
// (ps_pipeline.cu: real stages) and the test library (ps_testlib.cu: a
// closed-form host test double).  Internal header; not part of the ABI.
//
// The shared state -- committed buffers O_i, epochs, pending resync targets,
// the event log -- is a flat "board" under one process-shared robust mutex,
// so the same code runs the stages as threads of one process (board on the
// heap, ps_pipeline_run) or as one process per GPU (board in POSIX shared
// memory, ps_pipeline_run_rank).  Every device call runs outside the lock on
// the stage's own stream.
//  * stage 0 drafts one token per step ("Generate next token, append to O_0")
//    while it is less than max_lead tokens ahead of stage 1;
//  * stage i>0 takes window = O_{i-1}[n : n + min(avail, gamma_i)] when at least
//    max(1, lookahead_i) valid drafts exist, else an AR step (lookahead 0) or
//    waits; verifies; publishes the accepted tokens + its own token; on a
//    mismatch (a < w, or the drafter's buffer disagreeing with O_i[0:n]) every
//    stage j < i is resynced to O_i (reading R2) and its epoch bumped, so a
//    stale in-flight result is discarded (reading R9).
#pragma once
#include <errno.h>
#include <fcntl.h>
#include <pthread.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pipespec.h"

namespace {
inline long long now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

constexpr uint32_t kBoardMagic = 0x50535043u;   // "PSPC"
constexpr long long kBoardTimeoutNs = 600ll * 1000 * 1000 * 1000;

struct Board {
  uint32_t magic;
  int32_t k, cap, n_prompt;
  pthread_mutex_t mu;
  pthread_cond_t cv;
  int32_t ready, done, err, ev_cap;
  char err_msg[256];
  int64_t len[8], tlen[8];
  uint32_t epoch[8];
  int32_t pending[8];
  int64_t t_start;
  int64_t n_ev, ev_dropped;
  ps_run_stats stats;
  // followed by int32 O[8][cap], T[8][cap], then ps_event[ev_cap]
  int32_t* O(int i) { return reinterpret_cast<int32_t*>(this + 1) + (size_t)i * cap; }
  int32_t* T(int i) { return reinterpret_cast<int32_t*>(this + 1) + (size_t)(8 + i) * cap; }
  ps_event* EV() { return reinterpret_cast<ps_event*>(reinterpret_cast<int32_t*>(this + 1) + (size_t)16 * cap); }
};
inline size_t board_bytes(int cap, int ev_cap) {
  return sizeof(Board) + (size_t)16 * cap * sizeof(int32_t) + (size_t)ev_cap * sizeof(ps_event);
}

inline void board_init(Board* b, int k, int cap, int ev_cap) {
  memset(b, 0, sizeof(Board));
  b->k = k;
  b->cap = cap;
  b->ev_cap = ev_cap;
  pthread_mutexattr_t ma;
  pthread_mutexattr_init(&ma);
  pthread_mutexattr_setpshared(&ma, PTHREAD_PROCESS_SHARED);
  // robust: a stage process that dies holding the lock does not block its peers
  pthread_mutexattr_setrobust(&ma, PTHREAD_MUTEX_ROBUST);
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

inline void board_fail(Board* b, ps_status st, const char* msg) {   // lock held
  if (b->err == PS_OK) {
    b->err = st;
    snprintf(b->err_msg, sizeof b->err_msg, "%s", msg ? msg : "");
  }
  b->done = 1;
  pthread_cond_broadcast(&b->cv);
}

struct Lock {
  Board* b;
  explicit Lock(Board* b_) : b(b_) {
    const int rc = pthread_mutex_lock(&b->mu);
    if (rc == EOWNERDEAD) {               // the previous owner (a stage process) died
      pthread_mutex_consistent(&b->mu);
      board_fail(b, PS_E_STALE, "a stage process died holding the board lock");
    }
  }
  ~Lock() { pthread_mutex_unlock(&b->mu); }
};
// wait on the board (lock held) at most 50 ms: every waiter re-checks its
// predicate and the global deadline, so a dead peer process ends the run
inline void board_wait(Board* b) {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  ts.tv_nsec += 50 * 1000 * 1000;
  if (ts.tv_nsec >= 1000000000) { ts.tv_sec += 1; ts.tv_nsec -= 1000000000; }
  const int rc = pthread_cond_timedwait(&b->cv, &b->mu, &ts);
  if (rc == EOWNERDEAD) {
    pthread_mutex_consistent(&b->mu);
    board_fail(b, PS_E_STALE, "a stage process died holding the board lock");
  }
}

// Event log (lock held): entries in the order the committed buffers change.
inline void board_event(Board* b, int stage, int kind, int64_t n, int w, int a, int next, int origin,
                        const int32_t* window) {
  if (b->n_ev >= b->ev_cap) { b->ev_dropped++; return; }
  ps_event& e = b->EV()[b->n_ev++];
  memset(&e, 0, sizeof e);
  e.t_ns = now_ns() - b->t_start;
  e.stage = stage;
  e.kind = kind;
  e.n = (int32_t)n;
  e.w = w;
  e.a = a;
  e.next = next;
  e.origin = origin;
  for (int j = 0; j < w && j < 32; ++j) e.window[j] = window[j];
}

inline bool prefix_of(const int32_t* a, int64_t na, const int32_t* b, int64_t nb) {   // a extends b
  return na >= nb && std::equal(b, b + nb, a);
}

// resync every stage j < i to O_i (lock held)
inline void post_rollback(Board* b, int i) {
  for (int j = i - 1; j >= 0; --j) {
    if (prefix_of(b->O(j), b->len[j], b->O(i), b->len[i])) continue;   // already consistent
    std::copy(b->O(i), b->O(i) + b->len[i], b->T(j));
    b->tlen[j] = b->len[i];
    b->pending[j] = 1;
    std::copy(b->O(i), b->O(i) + b->len[i], b->O(j));   // the committed view is resynced now
    b->len[j] = b->len[i];
    ++b->epoch[j];
    b->stats.rollbacks[j]++;
    board_event(b, j, PS_EV_RESYNC, b->len[i], 0, 0, 0, i, nullptr);
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

inline int opt_gamma(const ps_run_opts* o, int i) { return o->gamma ? o->gamma[i] : 8; }

// Pad a step to the stage's virtual latency (ps_run_opts.virtual_ns).
inline void pad_step(const ps_run_opts* o, int i, long long t0) {
  if (!o->virtual_ns || o->virtual_ns[i] <= 0) return;
  const long long until = t0 + o->virtual_ns[i];
  for (long long t = now_ns(); t < until; t = now_ns())
    std::this_thread::sleep_for(std::chrono::nanoseconds(std::min(until - t, 200000ll)));
}

// Stage i's loop (Alg.1 lines 95-110 for i > 0, 98-100 for i = 0).
inline void board_worker(Board* b, int i, const StageOps& ops, const ps_run_opts* o,
                         const std::string& (*errf)()) {
  const int k = b->k, K = k - 1;
  const int gamma = i > 0 ? opt_gamma(o, i) : 8;
  const int look = (i > 0 && o->lookahead) ? o->lookahead[i] : 0;
  int max_gamma = 1, max_look = 0;
  for (int j = 1; j < k; ++j) {
    max_gamma = std::max(max_gamma, opt_gamma(o, j));
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
    int64_t n = 0;
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
        n = b->len[i];
        if (i == 0) { kind = 0; break; }
        mine.assign(b->O(i), b->O(i) + n);
        // The drafter's buffer disagrees with mine within O_i[0:n] -- at my
        // pending token, or earlier when a higher stage's rollback left O_{i-1}
        // on a short prefix of O_i from which the drafter diverged: resync it
        // (Alg.1, reading R2).
        const bool agree = b->len[i - 1] >= n && std::equal(mine.begin(), mine.end(), b->O(i - 1));
        if (b->len[i - 1] >= n && !agree) {
          post_rollback(b, i);
          pthread_cond_broadcast(&b->cv);
        }
        const int64_t avail = (agree && b->len[i - 1] > n) ? b->len[i - 1] - n : 0;
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
    pad_step(o, i, t0);
    const long long dt = now_ns() - t0;
    {
      Lock lk(b);
      b->stats.steps[i]++;
      b->stats.busy_ns[i] += dt;
      if (kind == 1) b->stats.verify_steps[i]++;
      if (b->done || b->epoch[i] != ep) {            // run over, or rolled back meanwhile: result is stale
        board_event(b, i, PS_EV_STALE, n, 0, 0, 0, kind == 0 ? PS_EV_DRAFT : kind == 1 ? PS_EV_VERIFY : PS_EV_AR,
                    nullptr);
        if (b->done) return;
        continue;
      }
      if ((int64_t)now.size() > b->cap) return board_fail(b, PS_E_CAPACITY, "token buffer beyond board capacity");
      std::copy(now.begin(), now.end(), b->O(i));
      b->len[i] = (int64_t)now.size();
      if (kind == 0) board_event(b, i, PS_EV_DRAFT, n, 0, 0, nxt, -1, nullptr);
      else board_event(b, i, kind == 1 ? PS_EV_VERIFY : PS_EV_AR, n, (int)window.size(), a, nxt, -1, window.data());
      if (kind == 1 && i == K) b->stats.accept_hist[std::min(a + 1, 63)]++;
      if (kind == 1 && a < (int)window.size()) post_rollback(b, i);
      if (i == K && finished()) b->done = 1;
      pthread_cond_broadcast(&b->cv);
    }
  }
}

// Generated tokens of O_K (lock not needed: every worker has returned).
inline void board_result(Board* b, std::vector<int32_t>& gen) {
  const int K = b->k - 1;
  gen.assign(b->O(K) + b->n_prompt, b->O(K) + b->len[K]);
}

// Copy the board's stats and event log to the caller (every worker returned).
inline void board_copy_out(Board* b, const ps_run_opts* o, ps_run_stats* stt) {
  if (!stt) return;
  memcpy(stt->steps, b->stats.steps, sizeof stt->steps);
  memcpy(stt->verify_steps, b->stats.verify_steps, sizeof stt->verify_steps);
  memcpy(stt->rollbacks, b->stats.rollbacks, sizeof stt->rollbacks);
  memcpy(stt->busy_ns, b->stats.busy_ns, sizeof stt->busy_ns);
  memcpy(stt->accept_hist, b->stats.accept_hist, sizeof stt->accept_hist);
  const int64_t m = o->event_log ? std::min<int64_t>(b->n_ev, std::max(o->event_cap, 0)) : 0;
  if (m > 0) memcpy(o->event_log, b->EV(), (size_t)m * sizeof(ps_event));
  stt->n_events = m;
  stt->events_dropped = b->ev_dropped + (b->n_ev - m);
}

inline ps_status run_board_threads(Board* b, const StageOps* ops, int k, int n_prompt, const ps_run_opts* o,
                                   std::vector<int32_t>& gen, ps_run_stats* stt, const std::string& (*errf)()) {
  b->n_prompt = n_prompt;
  for (int i = 0; i < k; ++i) {
    std::vector<int32_t> v;
    ps_status st = ops[i].tokens(ops[i].ctx, v);
    if (st != PS_OK) return st;
    if ((int64_t)v.size() > b->cap) return PS_E_CAPACITY;
    std::copy(v.begin(), v.end(), b->O(i));
    b->len[i] = (int64_t)v.size();
  }
  b->t_start = now_ns();
  std::vector<std::thread> th;
  for (int i = 0; i < k; ++i) th.emplace_back(board_worker, b, i, std::cref(ops[i]), o, errf);
  for (auto& t : th) t.join();
  board_copy_out(b, o, stt);
  if (b->err != PS_OK) return b->err;
  board_result(b, gen);
  return PS_OK;
}

// Heap board for the threads layout (freed by the owner of `mem`).
inline Board* board_on_heap(std::vector<uint8_t>& mem, int k, int cap, int ev_cap) {
  mem.assign(board_bytes(cap, ev_cap) + 64, 0);
  Board* b = reinterpret_cast<Board*>((reinterpret_cast<uintptr_t>(mem.data()) + 63) & ~(uintptr_t)63);
  board_init(b, k, cap, ev_cap);
  return b;
}
inline void board_destroy(Board* b) {
  pthread_cond_destroy(&b->cv);
  pthread_mutex_destroy(&b->mu);
}

// ---------------------------------------------------------------- one process per stage
// The board in POSIX shared memory: stage i runs in its own process (its own
// GPU), the processes exchange only the committed token buffers, epochs and
// rollback targets through the board (SURVEY §8(e) "across stages: tiny
// messages ... pinned-host mailboxes").
inline int board_ev_cap_for(int cap) { return 4 * cap; }

inline ps_status board_create_shm(const char* name, int k, int cap) {
  const int fd = shm_open(name, O_CREAT | O_RDWR | O_TRUNC, 0600);
  if (fd < 0) return PS_E_INVALID;
  const size_t bytes = board_bytes(cap, board_ev_cap_for(cap));
  if (ftruncate(fd, (off_t)bytes) != 0) { close(fd); return PS_E_INVALID; }
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return PS_E_INVALID;
  board_init((Board*)p, k, cap, board_ev_cap_for(cap));
  munmap(p, bytes);
  return PS_OK;
}

inline Board* board_open(const char* name, size_t* bytes) {
  const int fd = shm_open(name, O_RDWR, 0600);
  if (fd < 0) return nullptr;
  struct stat sb;
  if (fstat(fd, &sb) != 0 || (size_t)sb.st_size < sizeof(Board)) { close(fd); return nullptr; }
  void* p = mmap(nullptr, (size_t)sb.st_size, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return nullptr;
  Board* b = (Board*)p;
  if (__atomic_load_n(&b->magic, __ATOMIC_ACQUIRE) != kBoardMagic || board_bytes(b->cap, b->ev_cap) > (size_t)sb.st_size) {
    munmap(p, (size_t)sb.st_size);
    return nullptr;
  }
  *bytes = (size_t)sb.st_size;
  return b;
}

// Stage `rank` of a shared-memory board.  On error the board's message is
// copied to *err_out (the caller's thread-local error).
inline ps_status run_rank(const StageOps& ops, int rank, int k, const char* name, int n_prompt, const ps_run_opts* o,
                          int32_t* out, int32_t* out_len, ps_run_stats* stt, const std::string& (*errf)(),
                          std::string* err_out) {
  size_t bytes = 0;
  Board* b = board_open(name, &bytes);
  if (!b) {
    *err_out = std::string("cannot open board ") + name;
    return PS_E_INVALID;
  }
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
    if (result != PS_OK) {
      *err_out = b->err_msg;
    } else {
      std::vector<int32_t> gen;
      board_result(b, gen);
      if (o->eos_id >= 0) {
        auto it = std::find(gen.begin(), gen.end(), o->eos_id);
        if (it != gen.end()) gen.erase(it + 1, gen.end());
      }
      if ((int)gen.size() > o->max_new_tokens) gen.resize(o->max_new_tokens);
      std::copy(gen.begin(), gen.end(), out);
      *out_len = (int32_t)gen.size();
      if (stt) {
        const ps_run_stats keep = *stt;
        *stt = b->stats;
        memcpy(stt->fwd_ns, keep.fwd_ns, sizeof stt->fwd_ns);
        memcpy(stt->n_fwd, keep.n_fwd, sizeof stt->n_fwd);
        board_copy_out(b, o, stt);
        stt->tokens = *out_len;
        stt->wall_ns = now_ns() - b->t_start;
      }
    }
  }
  munmap(b, bytes);
  return result;
}
}  // namespace
