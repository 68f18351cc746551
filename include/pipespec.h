/*
 * pipespec.h — C ABI of the B200-native PipeSpec verify hot path.
 *
 * PipeSpec (arXiv 2505.01572) states the problem as
 *   "Require: Input prompt, Models [M_0...M_K];  Ensure: Generated sequence O_K"
 *   (Alg.1), greedy decoding.
 * Each model M_i is a *stage* that owns its token buffer O_i ("Let O_i be token
 * buffer for model i") and a paged KV cache.  The hot path is the
 * per-stage verification pass (Alg.1): one bf16 forward of M_i over
 * [pending token, d_0 .. d_{w-1}], greedy argmax per row, the longest matching
 * prefix a, append d[0:a] + correction/bonus token (reading R1 of DESIGN.md),
 * KV truncation (rollback) and the rejection signal to earlier stages.
 *
 * Conventions for every call:
 *  - All sizes are int32/int64; all structs are plain C.
 *  - Device pointers are CUDA device addresses on the stage's device; "host"
 *    pointers are ordinary (pageable or pinned) host memory.  A pointer that
 *    may be either is classified with cudaPointerGetAttributes.
 *  - Weights and the KV pool are BORROWED: the caller (e.g. PyTorch) owns them
 *    and keeps them alive until ps_stage_destroy.  The stage owns its token
 *    buffer, page table, scratch activations and CUDA graphs.
 *  - Errors: every call returns a ps_status; on error nothing observable
 *    changed (out-params untouched, buffer unchanged) and ps_last_error()
 *    returns a thread-local message.  No C++ exception crosses the ABI.
 *  - Threading: a stage is single-owner: one thread drives it;
 *    different stages may be driven concurrently from different threads.
 *  - Determinism: identical inputs give bit-identical results; the
 *    kernels are row-bucket invariant (fixed split order, absolute-position KV
 *    chunking, no floating-point atomics), so a verify over w drafts yields the
 *    same per-row logits as w+1 single-token steps.
 *  - There is no CPU fallback: without a usable sm_100a device every compute
 *    call returns PS_E_CUDA.
 */
#ifndef PIPESPEC_H_
#define PIPESPEC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t ps_status;
#define PS_OK          0
#define PS_E_INVALID  -1  /* bad argument / config (SPEC exit 2)              */
#define PS_E_CONTRACT -2  /* engine contract violated, e.g. rollback keep > len*/
#define PS_E_CAPACITY -3  /* out of KV pages or beyond max_seq                        */
#define PS_E_CUDA     -4  /* CUDA error or no sm_100a device                          */
#define PS_E_NCCL     -5  /* collective failure (tensor-parallel stages)              */
#define PS_E_STALE    -6  /* operation discarded by an epoch change (runtime)         */

/* Thread-local description of the last error on this thread ("" if none). */
const char* ps_last_error(void);

/* Library/ABI version (major*10000 + minor*100 + patch). */
int32_t ps_version(void);

/* Model shape (public HF LLaMA configs; reading R19).
 * Validated by ps_stage_create: n_heads % n_kv_heads == 0,
 * head_dim in {64,128}, d_model % 64 == 0, d_ffn % 64 == 0, vocab >= 2. */
typedef struct ps_model_shape {
  int32_t vocab, d_model, n_layers, n_heads, n_kv_heads, head_dim, d_ffn;
  float rms_eps, rope_theta;
  int32_t rope_kind;        /* 0 plain rotate-half, 1 llama3 frequency scaling */
  float rope_factor, lo_ff, hi_ff;
  int32_t rope_orig_max;
  int32_t tied_lm_head;     /* 1: lm_head == embed */
} ps_model_shape;

/* Per-layer weight slots, in this order (PyTorch nn.Linear layout [out,in]). */
enum { PS_WQ = 0, PS_WK, PS_WV, PS_WO, PS_WG, PS_WU, PS_WD, PS_N_ATTN, PS_N_MLP, PS_LAYER_SLOTS };

/* bf16 device pointers, row-major, 16-byte aligned.  `layers` is a HOST array
 * of n_layers*PS_LAYER_SLOTS device pointers.  Borrowed. */
typedef struct ps_weights {
  const void* embed;        /* [vocab, d_model]                       */
  const void* lm_head;      /* [vocab, d_model] (== embed when tied)  */
  const void* final_norm;   /* [d_model]                              */
  const void* const* layers;
} ps_weights;

/* Device placement.  Tensor parallelism inside a stage (
 * the paper only says the 70B was "split across 2 GPUs", reading R18):
 * tp_size in 1..8 ranks, each a stage of its own (one per GPU, or several on
 * one GPU with opts.max_ctas partitioning the SMs), created with the FULL
 * model shape and this rank's weight SHARDS (Megatron layout):
 *   wq/wk/wv: query / KV heads [r*H/T, (r+1)*H/T) rows;  wg/wu: d_ffn rows
 *   [r*F/T, ...);  wo, wd: the matching input COLUMNS (row-parallel);
 *   lm_head: vocabulary rows [r*V/T, (r+1)*V/T);  embed and the norm gains
 *   replicated.  Requires n_heads, n_kv_heads, vocab divisible by T, d_ffn by
 *   64*T, d_model by 128, use_megakernel = 1.
 * The O and down projections each end in an all-reduce of the [R, d] partials
 * and the lm_head in a max over the ranks' greedy keys; both run INSIDE the
 * megakernel over peer memory (no NCCL call): every rank publishes its
 * partial in its exchange buffer, then reads all T in rank order, so every
 * rank holds bit-identical activations and takes the same (a, next).  The
 * ranks of a group must run the same call sequence (ps_prefill / ps_verify /
 * ps_draft / ps_resync / ps_kv_rollback) concurrently, one host thread or
 * process each.  Before the first forward connect the group with
 * ps_tp_connect (one process per GPU, CUDA IPC handles) or
 * ps_tp_connect_local (ranks in one process).  nccl_comm is unused. */
typedef struct ps_placement {
  int32_t device;           /* CUDA ordinal */
  void* nccl_comm;          /* reserved, NULL */
  int32_t tp_rank, tp_size;
} ps_placement;

/* Stage options.  kv_pool: device buffer of kv_pool_bytes (>= the value of
 * ps_kv_pool_bytes for max_seq), borrowed; its layout is private to the
 * library ([page][layer][K|V][kv_head][page_size][head_dim] bf16).
 * stream: a cudaStream_t the stage enqueues all work on (NULL = a stream the
 * stage creates). */
typedef struct ps_stage_opts {
  int32_t max_seq;          /* max tokens in O_i (prompt + generated), >= 2   */
  int32_t max_window;       /* max w accepted by ps_verify, 0..31             */
  int32_t page_size;        /* tokens per KV page: 64, 128 or 256             */
  void* kv_pool;
  int64_t kv_pool_bytes;
  void* stream;
  int32_t use_graphs;       /* ignored (kept for layout stability): a forward
                               is ONE persistent kernel launch               */
  int32_t use_megakernel;   /* must be 1: the whole forward as one persistent
                               cooperative kernel (ps_mega.cuh)              */
  int32_t max_ctas;         /* megakernel CTAs (one per SM), 0 = every SM; a
                               smaller grid leaves SMs to concurrent stages  */
} ps_stage_opts;

typedef struct ps_stage ps_stage;

/* Bytes of KV pool a stage of this shape needs for max_seq tokens
 * (_tp: one rank of a tp_size group, which holds n_kv_heads / tp_size heads). */
int64_t ps_kv_pool_bytes(const ps_model_shape* shape, int32_t max_seq, int32_t page_size);
int64_t ps_kv_pool_bytes_tp(const ps_model_shape* shape, int32_t max_seq, int32_t page_size, int32_t tp_size);

/* Create a stage: validates the shape, builds TMA descriptors over the
 * borrowed weights, allocates scratch, and (optionally) captures graphs.
 * O_i starts empty; call ps_prefill before ps_draft / ps_verify. */
ps_status ps_stage_create(const ps_model_shape* shape, const ps_weights* weights,
                          const ps_placement* placement, const ps_stage_opts* opts,
                          ps_stage** out);
ps_status ps_stage_destroy(ps_stage* stage);

/* Tensor-parallel group wiring (see ps_placement).  PS_TP_HANDLE_BYTES is the
 * size of one exported handle: the cudaIpcMemHandle_t of the rank's exchange
 * buffer plus its rank, megakernel grid (CTAs), buffer size and shard shape.
 * ps_tp_handle writes this rank's handle; ps_tp_connect takes all tp_size
 * handles in rank order (host array [tp_size][PS_TP_HANDLE_BYTES], this
 * rank's own entry ignored), rejects a group whose ranks differ in grid or
 * shard shape (PS_E_INVALID: every rank waits for its peers' phase counters at
 * its own grid's target), and maps the peers' buffers, enabling peer access; ps_tp_connect_local links n stages created in THIS process (rank
 * order = array order, n == their tp_size).  A forward on an unconnected
 * tp_size > 1 stage returns PS_E_INVALID. */
#define PS_TP_HANDLE_BYTES 256
ps_status ps_tp_handle(ps_stage* stage, void* handle_out);
ps_status ps_tp_connect(ps_stage* stage, const void* handles);
ps_status ps_tp_connect_local(ps_stage* const* stages, int32_t n);

/* O_i := tokens[0:n] (host, n >= 1, every token < vocab, n <= max_seq).
 * Keeps the KV of the longest common prefix with the current O_i, then runs
 * the forward over the remaining positions so KV covers 0..n-2 and tokens[n-1]
 * is pending.  Serves as prefill, as catch-up after a resync, and as the
 * extend half of "rollback O_i to match O_j".
 * Path (ps_set_prefill_path): runs of >= 64 positions go in chunks of up to
 * 512 tokens through the prefill kernels (tcgen05 GEMMs with the tokens as
 * the M = 128 side, causal prefill attention; "the prefill phase
 * processes the initial input prompt") on single-GPU
 * stages; shorter runs, and tensor-parallel stages, use the decode
 * megakernel's 64-row bucket. */
ps_status ps_prefill(ps_stage* stage, const int32_t* tokens, int32_t n);

/* Prefill path of ps_prefill.  PS_PREFILL_AUTO (default): as described
 * there.  PS_PREFILL_ROWS: always the megakernel's 64-row bucket, whose KV is
 * bit-identical to KV written by decode forwards (row-bucket invariance); the
 * GEMM path's KV agrees with it within fp32 rounding (another summation order).
 * PS_E_INVALID for any other value. */
#define PS_PREFILL_AUTO 0
#define PS_PREFILL_ROWS 1
ps_status ps_set_prefill_path(ps_stage* stage, int32_t path);

/* Lazy form of ps_prefill for the rollback cascade ("Rollback O_i to match
 * O_j's last token"; reading R2): O_i := tokens[0:n] (host), keeping the
 * KV of the longest common prefix; the KV of the remaining positions is
 * computed by the next ps_draft / ps_verify as extra leading rows of that
 * forward (in 32-row chunks if more are pending).  No device work here. */
ps_status ps_resync(ps_stage* stage, const int32_t* tokens, int32_t n);

/* n_steps greedy autoregressive steps (rows = 1 each; Alg.1
 * "Generate next token, append to O_0"), appended to O_i; the tokens are
 * written to out_tokens[0:n_steps] (host).  Equals ps_verify with w = 0,
 * repeated.  With a synthetic-alpha override set (ps_set_synthetic), the
 * emitted token is the override's on-path token.  The forwards are launched
 * back to back in chains of up to 256, each taking its row token from the
 * previous one on the device (no host round trip per token; same results as
 * n single steps); a failure inside a chain leaves the tokens of the earlier
 * chains appended, O_i otherwise unchanged, and the stage's KV to be
 * recomputed by the next forward. */
ps_status ps_draft(ps_stage* stage, int32_t n_steps, int32_t* out_tokens);

/* Verification pass (Alg.1).  With len(O_i) = n, window[j] (host or
 * device, int32) is the draft for position n+j, 0 <= w <= max_window.  Rows
 * [x[n-1], d_0..d_{w-1}] at positions n-1..n-1+w are forwarded; pred_j is the
 * argmax of row j's fp32 logits (lowest index on ties, reading R12);
 *   a    = max{ j <= w : pred_t == d_t for all t < j }   -> *accepted_len
 *   next = pred_a  (correction if a < w, bonus if a == w)  -> *next_token
 * O_i becomes x ++ d[0:a] ++ [next], kv_len = n + a, and KV pages wholly at
 * or beyond kv_len are freed.  A rejection (a < w) means the caller must
 * resync stages j < i to O_i (keep = n + a + 1).
 * opt_logits: NULL, or host/device float [w+1][vocab] receiving the rows'
 * logits.  Errors: w > max_window or token >= vocab -> PS_E_INVALID;
 * n + w > max_seq or no page -> PS_E_CAPACITY; empty O_i -> PS_E_CONTRACT. */
/* (Tensor parallel: opt_logits receives this rank's [w+1][vocab/tp_size]
 * vocabulary slice; a and next are the group's.) */
ps_status ps_verify(ps_stage* stage, const int32_t* window, int32_t w,
                    int32_t* accepted_len, int32_t* next_token, float* opt_logits);

/* Asynchronous verification pass (SURVEY §8(b) "an async variant writes
 * a/next/kv_len to device memory + pinned mirror and records a CUDA event").
 * ps_verify_async enqueues the same forward as ps_verify on the stage's stream
 * and returns without waiting: `window` may be host memory or DEVICE memory
 * (e.g. a drafter's output on a peer GPU); a device window is gathered into
 * the forward's rows by an on-stream copy, never read by the host.  The
 * result lands in the stage-owned device record *ticket->d_result and its
 * mapped pinned mirror *ticket->h_result (ps_verify_result, valid once
 * ticket->event -- a cudaEvent_t recorded after the forward -- has completed).
 * Until ps_verify_wait the stage is IN FLIGHT: every call that uses or changes
 * it (verify, draft, prefill, resync, rollback, synthetic, timing) returns
 * PS_E_INVALID; ps_verify_query, ps_stage_tokens and ps_stage_get_info are
 * allowed (O_i is unchanged until the commit).  ps_verify_wait blocks on the event,
 * then commits exactly as ps_verify does (O_i := x ++ d[0:a] ++ [next] with
 * d[0:a] = pred[0:a], kv_len = n + a, pages beyond kv_len freed) and returns
 * a and next.  A device window holding a token >= vocab is reported by the
 * kernel (rows = -1 in the record) and ps_verify_wait returns PS_E_INVALID
 * without changing O_i.  ps_verify_query sets *done to 1 if the in-flight
 * pass has completed (0 otherwise; 1 if nothing is in flight). */
typedef struct ps_verify_result {
  int32_t a, next;          /* accepted length, correction/bonus token          */
  int32_t rows;             /* rows of the forward (-1: invalid device window)  */
  int32_t kv_len;           /* n + a: KV positions valid after the commit       */
  int32_t pred[32];         /* greedy prediction of rows row0.. (pred[j], j<=w) */
} ps_verify_result;
typedef struct ps_verify_ticket {
  const ps_verify_result* d_result;   /* device address                         */
  const ps_verify_result* h_result;   /* mapped pinned host mirror               */
  void* event;                        /* cudaEvent_t, owned by the stage         */
} ps_verify_ticket;
ps_status ps_verify_async(ps_stage* stage, const int32_t* window, int32_t w, ps_verify_ticket* ticket);
ps_status ps_verify_wait(ps_stage* stage, int32_t* accepted_len, int32_t* next_token);
ps_status ps_verify_query(ps_stage* stage, int32_t* done);

/* Rollback: requires 1 <= keep_len <= len(O_i) else PS_E_CONTRACT.
 * O_i := O_i[0:keep_len], kv_len := min(kv_len, keep_len-1), pending :=
 * O_i[keep_len-1]; frees pages wholly beyond kv_len (O(#freed pages)).
 * keep_len == len(O_i) is a no-op. */
ps_status ps_kv_rollback(ps_stage* stage, int64_t keep_len);

/* Read O_i into out[0:min(cap,len)] (host); *len = len(O_i). */
ps_status ps_stage_tokens(const ps_stage* stage, int32_t* out, int64_t cap, int64_t* len);

typedef struct ps_stage_info {
  int64_t n_tokens, kv_len, pages_in_use, pages_total;
  int64_t launches_per_verify;  /* kernels one verify pass enqueues */
  int32_t rows_buckets[4];      /* padded row counts with captured graphs */
  /* device time of the forward kernels (CUDA events around the launches on
   * the stage stream): the last verify/draft forward, and the running sums
   * over all verify/draft forwards since creation (ps_stage_reset_timers). */
  double last_fwd_ms, sum_fwd_ms;
  int64_t n_fwd;
  int32_t max_window, max_seq;  /* the stage's creation options                */
  int32_t attn_sc;              /* 64-key chunks per attention work item (from max_seq) */
} ps_stage_info;
ps_status ps_stage_reset_timers(ps_stage* stage);
ps_status ps_stage_get_info(const ps_stage* stage, ps_stage_info* info);

/* Synthetic-alpha override (SURVEY §8(c)
 * c.1 #8).  S: device or host int32 target stream (the real M_K greedy stream
 * after the prompt), len_S entries; n_prompt: prompt length; level i and top K
 * (this stage is M_i of a K+1 model chain); alphas[j] = alpha_{j,j+1} for
 * j = i..K-1; seed: counter-generator seed.  While the stage's context is
 * on-path (generated tokens == S prefix) every predicted token is replaced by
 * the chained synthetic token; off-path predictions are the model's own.
 * The forward still runs in full.  len_S == 0 disables the override. */
ps_status ps_set_synthetic(ps_stage* stage, const int32_t* S, int32_t len_S, int32_t n_prompt,
                           int32_t level, int32_t top, const double* alphas, uint64_t seed);

/* Pipeline modes. */
enum { PS_MODE_AR = 0, PS_MODE_SYNC_SD = 1, PS_MODE_PIPESPEC = 2 };

/* One entry of a run's event log (for trace replay against the oracle's
 * brute-force verify).  Entries are written
 * in the order the committed buffers change (under the runtime's lock), so
 * replaying them from the prompt reproduces every O_i:
 *   PS_EV_DRAFT   stage 0 appended `next` to O_0[0:n]
 *   PS_EV_VERIFY  stage i verified window[0:w] on O_i[0:n]: O_i := O_i[0:n] ++
 *                 window[0:a] ++ [next]
 *   PS_EV_AR      the same with w = 0 (no draft available, lookahead 0)
 *   PS_EV_RESYNC  O_stage := O_origin[0:n] (rollback cascade, R2)
 *   PS_EV_STALE   a finished step of `stage` (its kind in `origin`) discarded
 *                 by an epoch change                                          */
enum { PS_EV_DRAFT = 0, PS_EV_VERIFY = 1, PS_EV_AR = 2, PS_EV_RESYNC = 3, PS_EV_STALE = 4 };
typedef struct ps_event {
  int64_t t_ns;                   /* since the start of decoding              */
  int32_t stage, kind, n, w, a, next, origin, pad;
  int32_t window[32];
} ps_event;

typedef struct ps_run_opts {
  int32_t mode;
  int32_t max_new_tokens;
  int32_t eos_id;                 /* -1 = none */
  const int32_t* gamma;           /* host [k]: window cap per stage (stage 0 unused);
                                     NULL = 8; SYNC_SD / PIPESPEC need 1..max_window */
  const int32_t* lookahead;       /* host [k]: 0 = verify whenever >= 1 draft */
  int32_t max_lead;               /* draft ring depth per stage pair (>= max gamma + 1) */
  /* Optional synthetic acceptance (reading R24): alpha
   * NULL = the models' own predictions; else host [k-1], alpha[i] =
   * alpha_{i,i+1}.  The run first decodes max_new_tokens of M_K
   * autoregressively (outside wall_ns) as the target stream S, then sets the
   * chained override with `seed` on every stage i < K (ps_set_synthetic). */
  const double* alpha;
  uint64_t seed;
  /* Optional virtual latencies: host [k] or NULL; stage i's every step
   * (draft / verify / AR) lasts at least virtual_ns[i] (the host pads it),
   * to emulate the paper's relative model speeds on any device. */
  const int64_t* virtual_ns;
  ps_event* event_log;            /* NULL or host [event_cap]                  */
  int32_t event_cap;
} ps_run_opts;

typedef struct ps_run_stats {
  int64_t tokens;                 /* generated tokens (== *out_len)            */
  int64_t wall_ns;                /* from first decode step to the last token  */
  int64_t steps[8], verify_steps[8], rollbacks[8], busy_ns[8];
  int64_t accept_hist[64];        /* tokens appended per stage-K verify step   */
  int64_t n_events;               /* events written (<= event_cap); events past
                                     the cap are counted in events_dropped     */
  int64_t events_dropped;
  int64_t fwd_ns[8], n_fwd[8];    /* device time (CUDA events) of the stages'
                                     forwards during the run, and their count */
} ps_run_stats;

/* Alg.1 end to end: prefill every stage with the prompt, then run the k
 * stages (k <= 8) in the given mode until max_new_tokens (or eos) are in O_K.
 * out: host int32[max_new_tokens] receiving the generated tokens (prompt
 * excluded); *out_len their count.  PS_MODE_PIPESPEC runs one host thread per
 * stage with non-blocking draft rings and rollback mailboxes. */
ps_status ps_pipeline_run(ps_stage* const* stages, int32_t k, const int32_t* prompt,
                          int32_t n_prompt, const ps_run_opts* opts, int32_t* out,
                          int32_t* out_len, ps_run_stats* stats);

/* Alg.1 with ONE PROCESS PER STAGE (the paper's layout: each model on its own
 * GPU(s)).  The stages share a "board" in POSIX shared
 * memory (same node) holding the committed buffers O_i, epochs and rollback
 * targets -- the only cross-stage traffic is these few tokens.
 * ps_board_create: one process creates board `name` (e.g. "/pipespec-run1")
 * for k stages and `capacity` >= n_prompt + max_new_tokens + 320 tokens
 * BEFORE any stage attaches (re-creating resets it); ps_board_unlink removes
 * it.  ps_pipeline_run_rank: process `rank` (stage M_rank, 0 = first drafter,
 * k-1 = target) prefills `stage` with the prompt, attaches, waits for all k
 * stages, runs its Alg.1 loop (PS_MODE_PIPESPEC only) and returns, on every
 * rank, the generated tokens of O_{k-1} in out[0:*out_len] and the run's
 * stats.  A stage that fails or a peer that never attaches (120 s) ends the
 * run on every rank with that status. */
ps_status ps_board_create(const char* name, int32_t k, int32_t capacity);
ps_status ps_board_unlink(const char* name);
ps_status ps_pipeline_run_rank(ps_stage* stage, int32_t rank, int32_t k, const char* board,
                               const int32_t* prompt, int32_t n_prompt, const ps_run_opts* opts,
                               int32_t* out, int32_t* out_len, ps_run_stats* stats);

/* ps_pipeline_run_rank for a stage M_rank that is TENSOR PARALLEL over the n
 * members group[0..n-1] (ranks of one group connected with
 * ps_tp_connect_local, e.g. on n GPUs driven by this process): every step of
 * the stage's loop (prefill, draft, verify, resync) runs on all members
 * concurrently, one host thread each; the members must agree bit for bit
 * (else PS_E_CUDA) and the leader's result drives the board.  n = 1 is
 * ps_pipeline_run_rank. */
ps_status ps_pipeline_run_rank_group(ps_stage* const* group, int32_t n, int32_t rank, int32_t k,
                                     const char* board, const int32_t* prompt, int32_t n_prompt,
                                     const ps_run_opts* opts, int32_t* out, int32_t* out_len,
                                     ps_run_stats* stats);

/* Device-side timing hook for benchmarks: number of kernels this library has
 * launched (graph launches count their kernels) since process start. */
int64_t ps_kernel_launch_count(void);



#ifdef __cplusplus
}
#endif
#endif /* PIPESPEC_H_ */
