/*
 * pipespec_test.h — TEST library of the pipespec project (libpipespec_test.so,
 * built from csrc/ps_testlib.cu; never loaded by the product path).  It holds
 * the test double of the async runtime's protocol and hardware probes;
 * the product library libpipespec.so exports none of these.  Errors of this
 * library are read with ps_test_last_error.
 */
#ifndef PIPESPEC_TEST_H_
#define PIPESPEC_TEST_H_
#include <stdint.h>
#include "pipespec.h"
#ifdef __cplusplus
extern "C" {
#endif

const char* ps_test_last_error(void);

/* Launch-overhead probe: an empty kernel with `smem` bytes of dynamic shared
 * memory, `iters` back-to-back launches; *avg_ms per launch. */
ps_status ps_test_launch_overhead(int32_t smem, int32_t threads, int32_t grid, int32_t iters, float* avg_ms);

/* tcgen05 throughput probe (scripts/tc_probe.py): one CTA per SM, one thread
 * issues `iters` units of a mode (0: tcgen05.cp of a 16 KB tile to TMEM;
 * 1/2: 8 MMAs M128 N16 K16 with A in TMEM / smem; 3: copy + MMAs; 4-9: N and
 * accumulator-chain variants of the swap-AB orientation; 10/11: weights as
 * the B operand, N = 256 / 128), committing every `depth` units; writes the
 * slowest SM's ns per unit. */
ps_status ps_test_tc_probe(int32_t mode, int32_t iters, int32_t depth, double* ns_per_unit);
/* The same unit issued by the leader CTA of 2-CTA clusters as
 * tcgen05.mma.cta_group::2 with M = 256 (16 KB of weights per SM per unit). */
ps_status ps_test_tc_probe2(int32_t iters, int32_t depth, double* ns_per_unit);
/* mma.sync m16n8k16 bf16 issue interval: one CTA per SM of `warps` warps, each
 * issuing iters x 8 HMMAs in `chains` (1/2/4/8) independent accumulator chains;
 * ns (events) and cycles (clock64, CTA 0 warp 0) per HMMA per warp. */
ps_status ps_test_hmma_probe(int32_t warps, int32_t chains, int32_t iters, double* ns_per_hmma,
                             double* cycles_per_hmma);

/* Protocol test double of the async runtime (no GPU): k stages over a
 * closed-form host "model" -- stage k-1 emits next(c) = (c[-1]*7919 +
 * |c|*104729 + 13) mod vocab, stage i < k-1 agrees with stage i+1 with
 * probability alpha (hash of seed, i, |c|) -- stage i sleeping sleep_us*(1+3i)
 * per step.  _pipeline runs the k stages as threads of this process over the
 * same board code as ps_pipeline_run PS_MODE_PIPESPEC (event log included),
 * _run_rank as stage `rank` of a board in shared memory (as
 * ps_pipeline_run_rank; create it with ps_test_board_create). */
ps_status ps_test_fake_pipeline(int32_t k, const int32_t* prompt, int32_t n_prompt, const ps_run_opts* opts,
                                int32_t vocab, double alpha, uint64_t seed, int32_t sleep_us,
                                int32_t* out, int32_t* out_len, ps_run_stats* stats);
ps_status ps_test_fake_run_rank(int32_t rank, int32_t k, const char* board, const int32_t* prompt,
                                int32_t n_prompt, const ps_run_opts* opts, int32_t vocab, double alpha,
                                uint64_t seed, int32_t sleep_us, int32_t* out, int32_t* out_len,
                                ps_run_stats* stats);
ps_status ps_test_board_create(const char* name, int32_t k, int32_t capacity);
ps_status ps_test_board_unlink(const char* name);

/* Trace build only (libpipespec_trace.so, PS_TRACE=1; scripts/timeline.py):
 * copy `bytes` of a stage buffer to host dst.  which: 0 x, 1 x∘g, 2 q,
 * 3 attention out, 4 SwiGLU out, 5 sumsq slots, 6 KV pool, 7 attention (m,l)
 * partials, 8 page table, 9 megakernel phase stamps [G][n_ph][8],
 * 10 attention stamps, 11 stream-K fixup stamps, 12 tensor-parallel partials. */
ps_status ps_trace_read(ps_stage* stage, int32_t which, void* dst, int64_t bytes);

#ifdef __cplusplus
}
#endif
#endif
