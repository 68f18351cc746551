/*
 * pipespec_test.h — test hooks of the pipespec library (not part of the
 * user-facing ABI; used by tests/ to check single kernels in isolation).
 */
#ifndef PIPESPEC_TEST_H_
#define PIPESPEC_TEST_H_
#include <stdint.h>
#include "pipespec.h"
#ifdef __cplusplus
extern "C" {
#endif

/* out[r][n] = sum_k X[r][k] * W[n][k] for r < R, n < N (fp32), through the
 * production tcgen05 stream-K GEMM with a plain-store epilogue.
 * W: device bf16 [N, K]; X: device bf16 [32, K] (rows >= R ignored);
 * out: device float [R, N]; K % 64 == 0; 1 <= R <= 32.  Synchronises stream. */
ps_status ps_test_gemm(const void* W, const void* X, float* out, int32_t N, int32_t K, int32_t R, void* stream);

/* As ps_test_gemm, then `iters` timed launches: *avg_ms = CUDA-event time per
 * launch; cta_trace (host, may be NULL) receives per-CTA %globaltimer stamps
 * [iters][grid][4] = {entry, producer done, MMA done, exit} of every launch
 * (grid = min(#SMs, tiles * K/64)). */
ps_status ps_test_gemm_timed(const void* W, const void* X, float* out, int32_t N, int32_t K, int32_t R,
                             void* stream, int32_t iters, float* avg_ms, uint64_t* cta_trace);

/* Launch-overhead probe: an empty kernel with `smem` bytes of dynamic shared
 * memory, `iters` back-to-back launches; *avg_ms per launch. */
ps_status ps_test_launch_overhead(int32_t smem, int32_t threads, int32_t grid, int32_t iters, int32_t flags,
                                  float* avg_ms);
/* Test/profiling flags (process-wide; 0 = production behaviour):
 *   bit0  per-step path: launch GEMMs without programmatic dependent launch
 *   bit1  ps_test_gemm*: skip TMA loads        bit2  ps_test_gemm*: skip MMAs
 *   bit3  megakernel: record %globaltimer phase stamps (ps_test_read 9) and
 *         stream-K fixup stamps (ps_test_read 11); takes effect for stages
 *         created / tables built afterwards
 *   bit5  megakernel: 4-stage ring variant
 *   bit6  attention: per-item stage stamps (ps_test_read 10)
 *   bit8  megakernel: per-tile dataflow dependencies (experimental, slower)
 *   bit9  megakernel: cooperative launch even for a partial grid (max_ctas)
 *   bit10 attention: always combine inline (last-arriving CTA), no ACOMB phase
 *   bit11 attention: combine inline only when R*g <= 8 (ACOMB a pass-through) */
void ps_test_set_flags(int32_t flags);

/* Re-launch one kernel of the stage's most recent forward configuration
 * (same rows bucket, same device StepIn) `iters` times back to back on the
 * stage stream and return the average CUDA-event time per launch.
 * kind: 0 embed, 1 QKV GEMM, 2 attention, 3 O GEMM, 4 gate/up GEMM,
 * 5 down GEMM, 6 lm_head GEMM, 7 argmax/scan; layer selects the weights. */
ps_status ps_time_kernel(ps_stage* stage, int32_t kind, int32_t layer, int32_t iters, double* avg_ms);

/* Copy `bytes` of a stage scratch buffer to host dst (synchronises the stage
 * stream).  which: 0 x (fp32 [32,d]), 1 x∘g (bf16 [32,d]), 2 q (fp32 [32,H*hd]),
 * 3 attention out (bf16 [32,H*hd]), 4 SwiGLU out (bf16 [32,ffn]),
 * 5 sumsq slots (fp32 [32,ceil(d/128)]), 6 KV pool, 7 attention (m,l) partials,
 * 8 device page table (int32), 9 megakernel phase stamps, 10 attention stamps,
 * 11 stream-K fixup stamps, 12 tensor-parallel partials (fp32 [2][32][d]). */
ps_status ps_test_read(ps_stage* stage, int32_t which, void* dst, int64_t bytes);

/* Protocol test double of the async runtime (no GPU): k stages over a
 * closed-form host "model" -- stage k-1 emits next(c) = (c[-1]*7919 +
 * |c|*104729 + 13) mod vocab, stage i < k-1 agrees with stage i+1 with
 * probability alpha (hash of seed, i, |c|) -- stage i sleeping sleep_us*(1+3i) per step.
 * _pipeline runs the k stages as threads of this process (as
 * ps_pipeline_run PS_MODE_PIPESPEC), _run_rank as stage `rank` of a board in
 * shared memory (as ps_pipeline_run_rank). */
ps_status ps_test_fake_pipeline(int32_t k, const int32_t* prompt, int32_t n_prompt, const ps_run_opts* opts,
                                int32_t vocab, double alpha, uint64_t seed, int32_t sleep_us,
                                int32_t* out, int32_t* out_len, ps_run_stats* stats);
ps_status ps_test_fake_run_rank(int32_t rank, int32_t k, const char* board, const int32_t* prompt,
                                int32_t n_prompt, const ps_run_opts* opts, int32_t vocab, double alpha,
                                uint64_t seed, int32_t sleep_us, int32_t* out, int32_t* out_len,
                                ps_run_stats* stats);

#ifdef __cplusplus
}
#endif
#endif
