// ps_kernels.cuh — the device functions of the verify pass (sm_100a), run as
// the phases of the persistent megakernel (ps_mega.cuh):
//
//   embed_row           a1+a2+a3: window rows -> x (fp32 residual), x∘g (split-bf16
//                        GEMM operand) and per-128-column sum-of-squares slots
//   GEMM phases         a4/a7/a8/a9/a10: stream-K skinny GEMM on tcgen05 (the
//                        mainloop lives in ps_mega.cuh), fused epilogues:
//                          EPI_QKV    RMSNorm row scale + RoPE + paged KV append (a3,a5)
//                          EPI_RESID  residual add + next RMSNorm operand + sumsq (a7,a9)
//                          EPI_SWIGLU RMSNorm row scale + SiLU(gate)*up           (a8)
//                          EPI_LMHEAD final-norm scale + fp32 logits (on request)
//                                     + per-row greedy key by atomicMax       (a10)
//                          EPI_STORE  plain fp32 store (unit tests)
//   attn_run            a6: split-KV decode attention over the paged KV cache,
//                        fixed 64-key chunks at absolute positions, causal inside the
//                        window, GQA; deterministic last-CTA combine
//   argmax_run          a11 (+a13 data): vocab argmax from the partials, synthetic
//                        override (benchmarks), draft compare, first-mismatch scan
//
// RMSNorm is applied as a deferred row scale: the producer of x writes the bf16
// operand x∘g and per-slot sums of x^2; the consumer GEMM multiplies its output
// row r by rstd_r = 1/sqrt(mean(x_r^2)+eps)  ((x∘g)·W^T scaled by rstd is the
// RMSNorm'd product, PAPER-independent algebra).
#pragma once
#include <type_traits>

#include "ps_device.cuh"

namespace ps {

constexpr int kMaxRows = 32;       // max rows of a forward with the lm_head (verify / draft: w <= 31)
constexpr int kRowsCap = 64;       // max rows of any forward (prefill chunks: the 64-row bucket)
constexpr int kAttnChunk = 64;     // keys per split-KV chunk (absolute positions)

// Split-bf16 activations (reading R28).  Every bf16 operand the
// path derives from an fp32 activation is stored as a PAIR hi = bf16(v),
// lo = bf16(v - hi) (~16 significant bits): the GEMM operands x∘g, attention
// output and SwiGLU output (buffers of 2*kRowsCap rows: hi rows [0, 64), lo
// rows [64, 128); the tensor cores take both, W·hi + W·lo accumulated in fp32),
// the query and softmax probabilities inside attention, and the KV cache.
// With plain bf16 activations a 32-layer LLaMA-3.1-8B forward drifts ~4% of
// max|logit| from exact arithmetic (scripts/precision_probe.py), twice the
// north star's bound; split operands keep it at fp32-like error.
PS_DEV void split_bf16(float v, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16(v);
  lo = __float2bfloat16(v - __bfloat162float(hi));
}
PS_DEV uint32_t pack2(__nv_bfloat16 a, __nv_bfloat16 b) {
  return (uint32_t)__bfloat16_as_ushort(a) | ((uint32_t)__bfloat16_as_ushort(b) << 16);
}
// KV cache page layout [page][layer][plane][kv_head][page_size][hd] bf16,
// planes K_hi, K_lo, V_hi, V_lo.
constexpr int kKvPlanes = 4;

struct StepIn {                    // written by the host before every forward
  int32_t R;                       // rows in this forward, 1..kRowsCap (<= kMaxRows with the lm_head)
  int32_t pos0;                    // absolute position of row 0
  int32_t w;                       // drafts in the window (rows 1..w), verify only
  int32_t flags;                   // kFlagLogits | kFlagSynth | kFlagChainIn | kFlagChainOut
  int32_t syn_p0;                  // generated index predicted by row row0 (= n - n_prompt)
  int32_t syn_onpath;              // 1 iff the committed context is on the target stream
  int32_t row0;                    // first prediction row (rows before it are KV catch-up)
  int32_t gen;                     // forwards so far on this stage (megakernel counter target)
  int32_t gen_head;                // forwards with lm_head so far (targets of the head phases)
  int32_t chain_idx;               // chained draft forwards (ps_draft): this forward's slot in the chain array
  int32_t pad2[2];
  int32_t tokens[kRowsCap];        // row tokens: [pending, d_0, ..., d_{w-1}] (or a prefill chunk)
};
constexpr int kFlagLogits = 1;
constexpr int kFlagSynth = 2;
// Chained draft forwards (ps_draft of n > 1 tokens, launched back to back with
// no host round trip): a forward with kFlagChainOut stores its token in
// chain[chain_idx] (bit 31: the context is still on the synthetic target
// stream after it); one with kFlagChainIn takes its row-0 token and that
// on-path bit from chain[chain_idx - 1] instead of the host's StepIn.
constexpr int kFlagChainIn = 4;
constexpr int kFlagChainOut = 8;
constexpr int kMaxChain = 256;     // longest chain of draft forwards (one ps_draft call)

struct StepOut {                   // written by argmax_run (== ps_verify_result)
  int32_t a, next, R, kv_len;      // R = -1: a row token was out of range (nothing committed)
  int32_t pred[kMaxRows];
};

struct SynthParams {               // synthetic-alpha override (device resident)
  const int32_t* S;
  int32_t len_S, level, top, vocab;
  uint64_t seed;
  uint64_t thr[8];                 // thr[j] = floor(alpha_{j,j+1} * 2^53)
};

enum { EPI_STORE = 0, EPI_QKV = 1, EPI_RESID = 2, EPI_SWIGLU = 3, EPI_LMHEAD = 4 };

struct GemmParams {
  int mode;
  int N;                           // output features (SWIGLU: d_ffn)
  int n_tiles, kb_total;           // 128-feature tiles, 64-wide K blocks
  int t1, t2;                      // QKV: tiles [0,t1) q, [t1,t2) k, [t2,n) v
  int nq, nk;                      // QKV: rows of Wq, Wk (== Wv)
  int maxseg;                      // stream-K segments per tile (workspace stride)
  int grid;                        // CTAs the stream-K partition spans (<= persistent grid)
  const StepIn* step;
  // deferred RMSNorm scale (nullptr: none)
  const float* ss_in; int ss_n, ss_ld; float inv_d, eps;
  // EPI_RESID
  float* x; int ld_x;
  __nv_bfloat16* xg; int ld_xg; const __nv_bfloat16* gain;
  float* ss_out; int ss_out_ld;
  // EPI_SWIGLU
  __nv_bfloat16* h; int ld_h;
  // EPI_QKV
  float* q; int ld_q;
  __nv_bfloat16* kv; const int32_t* page_table; int page_size, layer, hkv, hd;
  long long page_stride;           // elements per KV page (all layers)
  const float2* rope_cs;           // [max_seq][hd/2] (cos, sin)
  // EPI_LMHEAD
  float* logits; int ld_logits;
  unsigned long long* amax; int amax_ld;
  int vocab_off;                   // tensor parallel: first vocabulary id of this rank's slice
  int amax_par;                    // 1: amax has two [kMaxRows] slots selected by gen_head parity
  // EPI_STORE
  float* out; int ld_out;
  // stream-K fixup (per 16-row chunk of the 64-row bucket: ws + chunk * ws_chunk floats,
  // counters + chunk * cnt_chunk)
  float* ws; unsigned* counters;
  long long ws_chunk; int cnt_chunk;
  int ll;                          // 1: flag-in-data partials (below); 0: release counter + reducer spin
  int ll_tag;                      // distinct per GEMM of a forward (< 1024); flag = gen << 10 ^ ll_tag
  unsigned long long* dbg;         // optional per-CTA %globaltimer trace [grid][4]
  int test_mode;                   // test hooks: bit0 skip TMA, bit1 skip MMA
};

// ------------------------------------------------------------------ stream-K partition
// CTA c of G owns units [b_c, b_{c+1}), b_c = floor(c*U/G); units are
// (tile, k-block) pairs in tile-major order.
PS_DEV long long sk_begin(long long U, int G, int c) { return U * c / G; }
PS_DEV int sk_owner(long long U, int G, long long u) { return (int)(((u + 1) * G - 1) / U); }

// Accumulator of one unit segment: the MMA's N = 2 RP columns hold W·x_hi
// (columns [0, RP)) and W·x_lo (columns [RP, 2 RP)) of the split operand; the
// row result is their fp32 sum (fixed order: hi + lo).
template <int RP>
PS_DEV void load_acc(uint32_t taddr, float* v) {
  float lo[RP];
  tmem_ld16(taddr, v);
  if constexpr (RP == 32) tmem_ld16(taddr + 16, v + 16);
  tmem_ld16(taddr + RP, lo);
  if constexpr (RP == 32) tmem_ld16(taddr + RP + 16, lo + 16);
#pragma unroll
  for (int r = 0; r < RP; ++r) v[r] += lo[r];
}

// Per-kernel (or per-phase) epilogue preparation: rstd_r from the producer's
// sum-of-squares slots (128/RP threads per row load their slots in one batch;
// partials combined in fixed order) and, for QKV, each row's KV slot offset.
template <int RP>
PS_DEV void epi_prepare(const GemmParams& p, int e, int R, int pos0, float* scratch, float* rstd, long long* kvrow) {
  // rstd_r from the producer's sum-of-squares slots in a FIXED order whatever
  // the rows bucket (row-bucket invariance): part q = 0..7 of row r sums the
  // slots j = q, q + 8, ... in increasing j; the 8 parts are then added in
  // order.  128 threads cover 16 rows x 8 parts per pass.
  {
    constexpr int MAXS = 8;                  // slots per part (ss_n <= 64, d <= 8192)
    const int part = e & 7;
#pragma unroll
    for (int r0 = 0; r0 < RP; r0 += 16) {
      const int row = r0 + (e >> 3);
      float sv[MAXS];
#pragma unroll
      for (int k = 0; k < MAXS; ++k) {
        const int j = part + 8 * k;
        sv[k] = (p.ss_in != nullptr && j < p.ss_n) ? p.ss_in[row * p.ss_ld + j] : 0.f;
      }
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < MAXS; ++k) s += sv[k];
      scratch[row * 8 + part] = s;
    }
  }
  named_bar(1, 128);
  if (e < RP) {
    float r_ = 1.0f;
    if (p.ss_in != nullptr) {
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) s += scratch[e * 8 + k];
      r_ = rsqrtf(s * p.inv_d + p.eps);
    }
    rstd[e] = r_;
    if (p.mode == EPI_QKV) {   // element offset of row e's KV slot (page + slot), head-independent
      long long off = 0;
      if (e < R) {
        const int pos = pos0 + e;
        off = (long long)p.page_table[pos / p.page_size] * p.page_stride + (long long)(pos % p.page_size) * p.hd;
      }
      kvrow[e] = off;
    }
  }
  named_bar(1, 128);
}

// Fixed-order sum over the nseg stream-K partials of one tile for the first
// 4*J rows: ((0 + p_0) + p_1) + ...; NIF segments' loads are in flight at once.
template <int RP, int J>
PS_DEV void sk_reduce(const float4* wsp, float* v, int e, int seg, int nseg) {
  constexpr int V4 = RP / 4;
  constexpr int JJ = J < V4 ? J : V4;
  constexpr int NIF = 16 / JJ;
  float acc[4 * JJ];
#pragma unroll
  for (int r = 0; r < 4 * JJ; ++r) acc[r] = 0.f;
  for (int q0 = 0; q0 < nseg; q0 += NIF) {
    float4 w4[NIF][JJ];
#pragma unroll
    for (int h = 0; h < NIF; ++h) {
      const int q = q0 + h;
#pragma unroll
      for (int j = 0; j < JJ; ++j) {
        if (q == seg) w4[h][j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        else if (q < nseg) w4[h][j] = __ldcg(&wsp[((size_t)q * 128 + e) * V4 + j]);
        else w4[h][j] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int h = 0; h < NIF; ++h) {
      if (q0 + h < nseg) {
#pragma unroll
        for (int j = 0; j < JJ; ++j) {
          acc[4 * j] += w4[h][j].x;
          acc[4 * j + 1] += w4[h][j].y;
          acc[4 * j + 2] += w4[h][j].z;
          acc[4 * j + 3] += w4[h][j].w;
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4 * JJ; ++r) v[r] = acc[r];
}

// The same fixed-order sum, with the other segments' partials staged into
// shared memory by cp.async first: every live float4 of every segment is in
// flight at once (the register version keeps 16 in flight, i.e. several round
// trips once R > 8 rows), and no registers are held for them.  Each thread
// reads back only its own copies, so no barrier is needed.  Bit-identical to
// sk_reduce: ((0 + p_0) + p_1) + ... with this CTA's own partial at `seg`.
template <int RP>
PS_DEV void sk_reduce_smem(const float4* wsp, float* v, int e, int seg, int nseg, int R4, float4* stage,
                           int cap_f4) {
  constexpr int V4 = RP / 4;
  float acc[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) acc[r] = 0.f;
  const int per_seg = 128 * R4;
  const int batch = cap_f4 / per_seg > 1 ? cap_f4 / per_seg : 1;
  for (int q0 = 0; q0 < nseg; q0 += batch) {
    const int q1 = nseg < q0 + batch ? nseg : q0 + batch;
    for (int q = q0; q < q1; ++q) {
      if (q == seg) continue;
#pragma unroll
      for (int j = 0; j < V4; ++j)
        if (j < R4)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(stage + ((q - q0) * 128 + e) * R4 + j)),
                       "l"(wsp + ((size_t)q * 128 + e) * V4 + j) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    for (int q = q0; q < q1; ++q) {
#pragma unroll
      for (int j = 0; j < V4; ++j) {
        if (j >= R4) continue;
        float4 w;
        if (q == seg) w = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        else w = stage[((q - q0) * 128 + e) * R4 + j];
        acc[4 * j] += w.x;
        acc[4 * j + 1] += w.y;
        acc[4 * j + 2] += w.z;
        acc[4 * j + 3] += w.w;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < V4; ++j)
    if (j < R4) {
      v[4 * j] = acc[4 * j];
      v[4 * j + 1] = acc[4 * j + 1];
      v[4 * j + 2] = acc[4 * j + 2];
      v[4 * j + 3] = acc[4 * j + 3];
    }
}

// Flag-in-data stream-K partials ("LL" protocol): every fp32 partial travels
// with a 32-bit flag in one 64-bit word (single-copy atomic), flag = (forward
// generation << 10) ^ GEMM tag, unique per use of a workspace slot.  The
// reducer polls the data itself: no store -> release -> acquire chain, no
// counter, no barrier; a partial is usable the moment it lands in L2.
PS_DEV void st_ll2(unsigned long long* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
PS_DEV void ld_ll2(const unsigned long long* p, unsigned long long& a, unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
PS_DEV unsigned long long ll_pack(float v, uint32_t flag) {
  return ((unsigned long long)flag << 32) | (unsigned long long)__float_as_uint(v);
}
PS_DEV bool ll_ok(unsigned long long w, uint32_t flag) { return (uint32_t)(w >> 32) == flag; }
PS_DEV float ll_val(unsigned long long w) { return __uint_as_float((uint32_t)w); }

// Fixed-order sum over the nseg LL partials of one tile, for row pairs
// [j0, j0 + JJ): ((0 + p_0) + p_1) + ... (the same order as sk_reduce); NIF
// segments' loads are issued before any is checked, stragglers re-polled.
template <int RP, int JJ, int NIF>
PS_DEV void sk_reduce_ll_group(const unsigned long long* wsp, float* v, int j0, int R2, int e, int seg, int nseg,
                               uint32_t flag) {
  float acc[2 * JJ];
#pragma unroll
  for (int r = 0; r < 2 * JJ; ++r) acc[r] = 0.f;
  for (int q0 = 0; q0 < nseg; q0 += NIF) {
    unsigned long long w[NIF][JJ][2];
#pragma unroll
    for (int h = 0; h < NIF; ++h) {
      const int q = q0 + h;
      if (q < nseg && q != seg) {
#pragma unroll
        for (int j = 0; j < JJ; ++j)
          if (j0 + j < R2) ld_ll2(wsp + ((size_t)q * 128 + e) * RP + 2 * (j0 + j), w[h][j][0], w[h][j][1]);
      }
    }
#pragma unroll
    for (int h = 0; h < NIF; ++h) {
      const int q = q0 + h;
      if (q >= nseg) continue;
      if (q == seg) {
#pragma unroll
        for (int r = 0; r < 2 * JJ; ++r) acc[r] += v[2 * j0 + r];
        continue;
      }
#pragma unroll
      for (int j = 0; j < JJ; ++j) {
        if (j0 + j >= R2) continue;              // row pairs past R: never published, never used
        unsigned ns = 32, polls = 0;
        unsigned long long t0 = 0;
        while (!ll_ok(w[h][j][0], flag) || !ll_ok(w[h][j][1], flag)) {
          __nanosleep(ns);
          ns = ns < 128 ? ns * 2 : 128;
          spin_check(polls, t0);
          ld_ll2(wsp + ((size_t)q * 128 + e) * RP + 2 * (j0 + j), w[h][j][0], w[h][j][1]);
        }
        acc[2 * j] += ll_val(w[h][j][0]);
        acc[2 * j + 1] += ll_val(w[h][j][1]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 2 * JJ; ++r) v[2 * j0 + r] = acc[r];
}

template <int RP>
PS_DEV void sk_reduce_ll(const unsigned long long* wsp, float* v, int R2, int e, int seg, int nseg, uint32_t flag) {
  if (R2 <= 1) sk_reduce_ll_group<RP, 1, 8>(wsp, v, 0, R2, e, seg, nseg, flag);
  else if (R2 <= 2) sk_reduce_ll_group<RP, 2, 4>(wsp, v, 0, R2, e, seg, nseg, flag);
  else {
#pragma unroll
    for (int j0 = 0; j0 < RP / 2; j0 += 4)
      if (j0 < R2) sk_reduce_ll_group<RP, 4, 2>(wsp, v, j0, R2, e, seg, nseg, flag);
  }
}

// One accumulator segment of tile t (units [seg_begin, seg_end) of this CTA c
// out of G): stream-K fixup (deterministic fixed segment order) then the
// fused epilogue for the tile if this CTA completes it.  128 epilogue threads.
// kLL: compile the flag-in-data fixup (p.ll selects it at run time); the
// 2-CTA/SM standalone GEMM keeps the register-lean release/counter fixup.
template <int RP, bool kLL = false>
PS_DEV bool epi_segment(const GemmParams& p, int t, long long seg_begin, long long seg_end, long long U, int G, int c,
                        int kbt, float* v, int e, int lane, int quarter, int R, int pos0, float* scratch,
                        unsigned long long* red, const float* rstd, const long long* kvrow, volatile int* flag,
                        float4* stage = nullptr, int stage_f4 = 0, int r0 = 0) {
  // r0: first row of this 16-row chunk (64-row bucket; 0 otherwise): rows r of
  // the chunk are rows r0 + r of the forward (rstd / kvrow / pos0 are passed
  // already offset); each chunk has its own partials and counters
  float* const wsb = p.ws + (size_t)(r0 / 16) * p.ws_chunk;
  unsigned* const cnt = p.counters + (r0 / 16) * p.cnt_chunk;
  bool finalized = false;
  // Epilogue operands that do not depend on this tile's result (residual x and
  // its gain; RoPE cos/sin) are loaded BEFORE the stream-K wait, so their
  // round trip overlaps the partials' arrival instead of following it.
  // (Rows bucket 16 only: at 32 rows the extra live registers spill.)
  constexpr bool kPre = RP <= 16;
  const long long tile_u00 = (long long)t * kbt;
  const bool will_fin = kPre && ((seg_begin == tile_u00 && seg_end == tile_u00 + kbt) || sk_owner(U, G, tile_u00) == c);
  float pre_x[RP];
  float pre_g = 0.f;
  float2 pre_cs[RP];
  if (will_fin && p.mode == EPI_RESID) {
    const int f = t * 128 + e;
    const bool ok = f < p.N;
    pre_g = ok ? __bfloat162float(p.gain[f]) : 0.f;
#pragma unroll
    for (int r = 0; r < RP; ++r) pre_x[r] = (r < R && ok) ? p.x[(size_t)(r0 + r) * p.ld_x + f] : 0.f;
  }
  if (will_fin && p.mode == EPI_QKV && t < p.t2) {
    const int f = t < p.t1 ? t * 128 + e : (t - p.t1) * 128 + e;
    const int j = (f % p.hd) & ((p.hd >> 1) - 1);
#pragma unroll
    for (int r = 0; r < RP; ++r)
      pre_cs[r] = r < R ? p.rope_cs[(size_t)(pos0 + r) * (p.hd >> 1) + j] : make_float2(1.f, 0.f);
  }
  do {
    // ---- stream-K fixup: deterministic, fixed segment order ----
    // Partials are laid out [tile][seg][lane e][RP] so every thread moves
    // RP contiguous floats with 16-byte accesses; the reducing CTA issues all
    // of a segment's loads before using them (latency, not bandwidth, bound).
    const long long tile_u0 = (long long)t * kbt;
    // LL only for R <= 4 (at most 2 row pairs per thread: the reducer keeps 8
    // segments' loads in flight); wider windows keep the release path, whose
    // float4 partials batch more segments per round trip (measured: 1B R=1
    // -2.6%, 8B R=5 +3.5% with LL)
    if (kLL && p.ll && R <= 4 && !(seg_begin == tile_u0 && seg_end == tile_u0 + kbt)) {
      const int first = sk_owner(U, G, tile_u0);
      const int nseg = sk_owner(U, G, tile_u0 + kbt - 1) - first + 1;
      const int seg = c - first;
      const uint32_t flag = ((uint32_t)p.step->gen << 10) ^ (uint32_t)p.ll_tag;
      unsigned long long* wsp = reinterpret_cast<unsigned long long*>(wsb) + (size_t)(t * p.maxseg) * RP * 128;
      const int R2 = (R + 1) >> 1;               // live row pairs
      if (seg != 0) {                            // publish: data + flag, nothing else
#pragma unroll
        for (int j = 0; j < RP / 2; ++j)
          if (j < R2) st_ll2(wsp + ((size_t)seg * 128 + e) * RP + 2 * j, ll_pack(v[2 * j], flag), ll_pack(v[2 * j + 1], flag));
        if (e == 0) PS_TRACE_STAMP(p.dbg, c * 4 + 0);
        break;
      }
      if (e == 0) { PS_TRACE_STAMP(p.dbg, c * 4 + 0); PS_TRACE_STAMP(p.dbg, c * 4 + 1); }
      sk_reduce_ll<RP>(wsp, v, R2, e, seg, nseg, flag);
      if (e == 0) PS_TRACE_STAMP(p.dbg, c * 4 + 2);
    } else if (!(seg_begin == tile_u0 && seg_end == tile_u0 + kbt)) {
      const int first = sk_owner(U, G, tile_u0);
      const int nseg = sk_owner(U, G, tile_u0 + kbt - 1) - first + 1;
      const int seg = c - first;
      float4* wsp = reinterpret_cast<float4*>(wsb + (size_t)(t * p.maxseg) * RP * 128);
      constexpr int V4 = RP / 4;
      const int R4 = (R + 3) >> 2;               // float4s per thread that hold live rows
      if (seg != 0) {
#pragma unroll
        for (int j = 0; j < V4; ++j)
          if (j < R4)
            __stcg(&wsp[((size_t)seg * 128 + e) * V4 + j], make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
      }
      // Static reducer: segment 0's CTA (its range ENDS in this tile, so it
      // reaches this tile last anyway) waits for the other nseg-1 segments;
      // they publish with a fire-and-forget release add (no round trip) after
      // a barrier that orders all 128 threads' partial stores before it.
      if (seg != 0) {
        named_bar(1, 128);
        if (e == 0) PS_TRACE_STAMP(p.dbg, c * 4 + 0);
        if (e == 0) red_release_add_gpu(&cnt[t], 1u);
        break;
      }
      if (e == 0) PS_TRACE_STAMP(p.dbg, c * 4 + 0);
      if (e == 0) {
        spin_until_gpu(&cnt[t], (unsigned)(nseg - 1));
        cnt[t] = 0u;                           // ready for the next forward
      }
      named_bar(1, 128);
      if (e == 0) PS_TRACE_STAMP(p.dbg, c * 4 + 1);
      // reduce: only the live rows, with up to 16 float4 loads in flight
      if (R4 <= 1) sk_reduce<RP, 1>(wsp, v, e, seg, nseg);
      else if (R4 <= 2) sk_reduce<RP, 2>(wsp, v, e, seg, nseg);
      else if (R4 <= 4) sk_reduce<RP, 4>(wsp, v, e, seg, nseg);
      // > 16 rows: staged through shared memory (measured: R=17 8B pass -2.7%;
      // R=9 +0.6%, so the 16-in-flight register version stays up to 16 rows)
      else if (stage != nullptr) sk_reduce_smem<RP>(wsp, v, e, seg, nseg, R4, stage, stage_f4);
      else sk_reduce<RP, (RP / 4 < 8 ? RP / 4 : 8)>(wsp, v, e, seg, nseg);
      if (e == 0) PS_TRACE_STAMP(p.dbg, c * 4 + 2);
    }

    // ---- fused epilogues (global loads batched ahead of use) ----
    if (p.mode == EPI_STORE) {
      const int f = t * 128 + e;
      if (f < p.N) {
#pragma unroll
        for (int r = 0; r < RP; ++r)
          if (r < R) p.out[(size_t)(r0 + r) * p.ld_out + f] = v[r];
      }
    } else if (p.mode == EPI_RESID) {
      const int f = t * 128 + e;
      const bool ok = f < p.N;
      if constexpr (!kPre) {
        pre_g = ok ? __bfloat162float(p.gain[f]) : 0.f;
#pragma unroll
        for (int r = 0; r < RP; ++r) pre_x[r] = (r < R && ok) ? p.x[(size_t)(r0 + r) * p.ld_x + f] : 0.f;
      }
      const float g = pre_g;
      const float* xo = pre_x;
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        if (r >= R) break;
        float sq = 0.f;
        if (ok) {
          const float xn = xo[r] + v[r];
          p.x[(size_t)(r0 + r) * p.ld_x + f] = xn;
          split_bf16(xn * g, p.xg[(size_t)(r0 + r) * p.ld_xg + f], p.xg[(size_t)(r0 + r + kRowsCap) * p.ld_xg + f]);
          sq = xn * xn;
        }
        sq = warp_sum(sq);
        if (lane == 0) scratch[quarter * RP + r] = sq;
      }
      named_bar(1, 128);
      if (e < R)
        p.ss_out[(size_t)(r0 + e) * p.ss_out_ld + t] =
            ((scratch[0 * RP + e] + scratch[1 * RP + e]) + scratch[2 * RP + e]) + scratch[3 * RP + e];
      named_bar(1, 128);
    } else if (p.mode == EPI_SWIGLU) {
#pragma unroll
      for (int r = 0; r < RP; ++r) scratch[e * (RP + 1) + r] = v[r] * rstd[r];
      named_bar(1, 128);
      if (e < 64) {
        const int f = t * 64 + e;
        if (f < p.N) {
#pragma unroll
          for (int r = 0; r < RP; ++r) {
            if (r < R) {
              const float gt = scratch[e * (RP + 1) + r];
              const float up = scratch[(e + 64) * (RP + 1) + r];
              split_bf16(gt / (1.0f + __expf(-gt)) * up, p.h[(size_t)(r0 + r) * p.ld_h + f],
                         p.h[(size_t)(r0 + r + kRowsCap) * p.ld_h + f]);
            }
          }
        }
      }
      named_bar(1, 128);
    } else if (p.mode == EPI_QKV) {
      int kind, f, nrows;
      if (t < p.t1) { kind = 0; f = t * 128 + e; nrows = p.nq; }
      else if (t < p.t2) { kind = 1; f = (t - p.t1) * 128 + e; nrows = p.nk; }
      else { kind = 2; f = (t - p.t2) * 128 + e; nrows = p.nk; }
#pragma unroll
      for (int r = 0; r < RP; ++r) v[r] *= rstd[r];
      const int hd = p.hd, half = hd >> 1;
      const int i = f % hd;
      if (kind < 2) {   // rotate-half RoPE at absolute positions pos0 + r
        if constexpr (!kPre) {
          const int j = i & (half - 1);
#pragma unroll
          for (int r = 0; r < RP; ++r) pre_cs[r] = r < R ? p.rope_cs[(size_t)(pos0 + r) * half + j] : make_float2(1.f, 0.f);
        }
        const float2* cs = pre_cs;
#pragma unroll
        for (int r = 0; r < RP; ++r) scratch[e * (RP + 1) + r] = v[r];
        named_bar(1, 128);
        const int pe = e ^ half;
#pragma unroll
        for (int r = 0; r < RP; ++r) {
          const float pv = scratch[pe * (RP + 1) + r];
          v[r] = (i < half) ? (v[r] * cs[r].x - pv * cs[r].y) : (v[r] * cs[r].x + pv * cs[r].y);
        }
        named_bar(1, 128);
      }
      if (f < nrows) {
        if (kind == 0) {
#pragma unroll
          for (int r = 0; r < RP; ++r)
            if (r < R) p.q[(size_t)(r0 + r) * p.ld_q + f] = v[r];
        } else {
          const int kh = f / hd;
          const size_t plane = (size_t)p.hkv * p.page_size * hd;   // elements per (layer, plane)
          const size_t head_off = ((size_t)(p.layer * kKvPlanes + 2 * (kind - 1)) * p.hkv + kh) * p.page_size * hd + i;
#pragma unroll
          for (int r = 0; r < RP; ++r)
            if (r < R) split_bf16(v[r], p.kv[(size_t)kvrow[r] + head_off], p.kv[(size_t)kvrow[r] + head_off + plane]);
        }
      }
    } else {  // EPI_LMHEAD: logits (on request) + per-row greedy key, atomicMax (order-free, exact)
      const int f = t * 128 + e;
      const bool ok = f < p.N;
      const bool want = p.logits != nullptr && (p.step->flags & kFlagLogits);
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        if (r >= R) break;                       // live rows only (a warp max per row)
        const float z = v[r] * rstd[r];
        if (want && ok) p.logits[(size_t)r * p.ld_logits + f] = z;
        unsigned long long k = ok ? argmax_key(z, (uint32_t)(f + p.vocab_off)) : 0ull;
        k = warp_max_u64(k);
        if (lane == 0) red[quarter * RP + r] = k;
      }
      named_bar(1, 128);
      if (e < R) {
        unsigned long long k = red[e];
        for (int q = 1; q < 4; ++q) k = red[q * RP + e] > k ? red[q * RP + e] : k;
        unsigned long long* am = p.amax_par ? p.amax + (p.step->gen_head & 1) * kMaxRows : p.amax;
        atomicMax(&am[e], k);
      }
      named_bar(1, 128);
    }
    finalized = true;
    if (e == 0) PS_TRACE_STAMP(p.dbg, c * 4 + 3);
  } while (0);
  return finalized;   // this CTA completed tile t (its outputs are written)
}

// ------------------------------------------------------------------ embed (a1-a3)
struct EmbedParams {
  const StepIn* step;
  const __nv_bfloat16* embed; int d; int vocab;
  const __nv_bfloat16* gain;
  float* x; int ld_x;
  __nv_bfloat16* xg; int ld_xg;
  float* ss; int ss_ld;
};

// Row r of the window: x = E[tok] (fp32), x∘g (bf16 operand), per-128-col sum of squares.
PS_DEV void embed_row(const EmbedParams& p, int r, int tid /* 0..127 */) {
  // thread t owns columns [32t, 32t+32) (d <= 4096 per pass); 4 threads per
  // 128-column sum-of-squares slot.  All loads are issued before any use.
  // (a device-resident window is not validated by the host: an out-of-range
  // id reads row 0 here and the argmax phase reports it, rows = -1)
  const int tok0 = p.step->tokens[r];
  const int tok = (tok0 >= 0 && tok0 < p.vocab) ? tok0 : 0;
  const __nv_bfloat16* src = p.embed + (size_t)tok * p.d;
  for (int c0 = 0; c0 < p.d; c0 += 128 * 32) {
    const int col = c0 + tid * 32;
    const bool ok = col < p.d;
    uint4 xr[4], gr[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      xr[k] = ok ? reinterpret_cast<const uint4*>(src + col)[k] : make_uint4(0, 0, 0, 0);
      gr[k] = ok ? reinterpret_cast<const uint4*>(p.gain + col)[k] : make_uint4(0, 0, 0, 0);
    }
    float sq = 0.f;
    if (ok) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const __nv_bfloat162* xb = reinterpret_cast<const __nv_bfloat162*>(&xr[k]);
        const __nv_bfloat162* gb = reinterpret_cast<const __nv_bfloat162*>(&gr[k]);
        float xf[8];
        uint32_t oh[4], ol[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 xv = __bfloat1622float2(xb[q]);
          const float2 gv = __bfloat1622float2(gb[q]);
          xf[2 * q] = xv.x;
          xf[2 * q + 1] = xv.y;
          __nv_bfloat16 h0, l0, h1, l1;
          split_bf16(xv.x * gv.x, h0, l0);
          split_bf16(xv.y * gv.y, h1, l1);
          oh[q] = pack2(h0, h1);
          ol[q] = pack2(l0, l1);
          sq += xv.x * xv.x + xv.y * xv.y;
        }
        float4* xd = reinterpret_cast<float4*>(p.x + (size_t)r * p.ld_x + col + 8 * k);
        xd[0] = make_float4(xf[0], xf[1], xf[2], xf[3]);
        xd[1] = make_float4(xf[4], xf[5], xf[6], xf[7]);
        *reinterpret_cast<uint4*>(p.xg + (size_t)r * p.ld_xg + col + 8 * k) = make_uint4(oh[0], oh[1], oh[2], oh[3]);
        *reinterpret_cast<uint4*>(p.xg + (size_t)(r + kRowsCap) * p.ld_xg + col + 8 * k) =
            make_uint4(ol[0], ol[1], ol[2], ol[3]);
      }
    }
    sq += __shfl_xor_sync(0xffffffffu, sq, 1);
    sq += __shfl_xor_sync(0xffffffffu, sq, 2);
    if (ok && (tid & 3) == 0) p.ss[(size_t)r * p.ss_ld + col / 128] = sq;
  }
}

// ------------------------------------------------------------------ tensor-parallel reduce (a14)
// Row-parallel O / down projections leave each rank a partial [R, d] (fp32, in
// its exchange buffer).  Every rank sums the T partials in rank order (so all
// ranks hold bit-identical x), adds the residual, and writes the next RMSNorm
// operand x∘g and the per-128-column sums of squares -- the EPI_RESID epilogue
// of the single-GPU path with the all-reduce folded in.
struct TpParams {
  const float* part[8];            // rank q's partial [kRowsCap][d] (peer memory for q != rank)
  int n;                           // tp_size
  float* x; int ld_x;
  __nv_bfloat16* xg; int ld_xg; const __nv_bfloat16* gain;
  float* ss_out; int ss_out_ld;
  int d;
};

// One unit = (row r, 128-column tile t), one warp: 4 columns per lane.
PS_DEV void tp_reduce_unit(const TpParams& p, int r, int t, int lane) {
  const int f = t * 128 + lane * 4;
  const size_t off = (size_t)r * p.d + f;
  const float4 xo = *reinterpret_cast<const float4*>(p.x + (size_t)r * p.ld_x + f);
  float4 s = __ldcg(reinterpret_cast<const float4*>(p.part[0] + off));
  for (int q = 1; q < p.n; ++q) {    // rank order: ((p_0 + p_1) + p_2) + ...
    const float4 v = __ldcg(reinterpret_cast<const float4*>(p.part[q] + off));
    s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
  }
  const float4 xn = make_float4(xo.x + s.x, xo.y + s.y, xo.z + s.z, xo.w + s.w);
  *reinterpret_cast<float4*>(p.x + (size_t)r * p.ld_x + f) = xn;
  const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(p.gain + f);
  const float2 ga = __bfloat1622float2(g2[0]), gb = __bfloat1622float2(g2[1]);
  __nv_bfloat16 h[4], l[4];
  split_bf16(xn.x * ga.x, h[0], l[0]);
  split_bf16(xn.y * ga.y, h[1], l[1]);
  split_bf16(xn.z * gb.x, h[2], l[2]);
  split_bf16(xn.w * gb.y, h[3], l[3]);
  *reinterpret_cast<uint2*>(p.xg + (size_t)r * p.ld_xg + f) = make_uint2(pack2(h[0], h[1]), pack2(h[2], h[3]));
  *reinterpret_cast<uint2*>(p.xg + (size_t)(r + kRowsCap) * p.ld_xg + f) = make_uint2(pack2(l[0], l[1]), pack2(l[2], l[3]));
  float sq = xn.x * xn.x + xn.y * xn.y + xn.z * xn.z + xn.w * xn.w;
  sq = warp_sum(sq);
  if (lane == 0) p.ss_out[(size_t)r * p.ss_out_ld + t] = sq;
}

// ------------------------------------------------------------------ attention (a6)
// Split-KV decode attention, GQA-grouped.  Work item = (KV head kh, row block
// rb of up to 128 query rows, chunk c of 64 keys at absolute positions
// [64c, 64c+64)).  Query row m of a block is (window row r = m / g, query head
// kh*g + m % g), so one K/V chunk read serves all g heads that share it.
// S = Q K^T and O = P V run on the tensor cores (mma.sync m16n8k16 bf16 ->
// fp32; one warp per 16 rows), softmax in fp32 in the exp2 domain.  Chunk
// partials (m, l, O) go to a workspace; the last CTA of each (kh, rb)
// combines them in chunk order (deterministic; a row's result does not depend
// on R because chunks sit at absolute positions and fully masked chunks
// contribute exact zeros).
struct AttnParams {
  const StepIn* step;
  const float* q; int ld_q;
  const int32_t* page_table; int page_size, page_shift;   // page_size = 1 << page_shift
  const CUtensorMap* kvmap;        // the KV pool as {hd, rows, plane}, box {64, 16, 4}, 128B swizzle
  long long rows_per_page;         // page_stride / hd
  int layer, hkv, H, hd;
  float scale_log2;                // log2(e) / sqrt(hd)
  int max_chunks, rows_cap;        // item partials per (head, row); query rows per head (kRowsCap * g)
  int sc;                          // 64-key chunks per work item (a per-stage constant)
  float* ws_o;                     // [hkv][max_chunks][rows_cap][hd]
  float* ws_ml;                    // [hkv][max_chunks][rows_cap][2]
  __nv_bfloat16* out; int ld_out;
  unsigned long long* dbg;         // optional per-CTA stamps [cta][8] (PS_TRACE builds)
};

// ---------------------------------------------------------------- decode attention (a6)
// Work items: (KV head kh, row block rb, item j = sc consecutive 64-key chunks
// at absolute positions [64 sc j, 64 sc (j + 1))).  sc is a per-stage constant
// (ps_stage: from max_seq), so a row's arithmetic does not depend on R or on
// the context length (row-bucket invariance: a verify row equals the AR step
// at that position bit for bit).  CTA c of G owns the contiguous item range
// [c n / G, (c + 1) n / G) and streams the items' 16-key stages back to back
// through a 4-deep TMA ring (3 stages in flight while one is used), so the
// schedule never changes an item's math.
//
// Keys on the MMA's M side: per 16-key stage S^T = K Q^T (A = K, 16 keys x 16
// dims by ldmatrix from the ring; B = Q^T, 16 dims x 8 query rows per n-tile,
// in registers) and O^T = V^T P^T (A = V^T by ldmatrix.trans; B = P^T, the S^T
// accumulator transposed in registers by movmatrix).  A row block is NR = 1..3
// n-tiles of 8 rows (query row m of a block = window row m / g, head kh g +
// m % g): a decode step (R = 1, g = 4: 4 rows) costs one 8-row n-tile, and up
// to 24 rows (R <= 6 at g = 4, the bench's verify window) take ONE pass over
// the keys.  The 4 warps split the head dimension (warp w owns dims [w hd/4,
// (w+1) hd/4)); S^T is summed from the 4 warps' partial dot products (smem
// exchange, fixed order w = 0..3, identical in every warp); every warp runs the
// same online softmax and accumulates O^T for its own dims.  Split-bf16
// operands on mma.sync m16n8k16: (k_hi + k_lo)(q_hi + q_lo) ~ k_hi q_hi +
// k_hi q_lo + k_lo q_hi (the lo*lo term ~2^-16 relative), likewise V P.
// Every per-row operation (the MMA's per-element dot products, the fixed-order
// warp sums, the xor-4/8/16 shuffle trees over a row's 8 key lanes) is the
// same whichever n-tile column holds the row, so rows are bit-identical for
// any R.
constexpr int kAttnRB = 8;                  // query rows per n-tile (row blocks: NR n-tiles)
constexpr int kAttnMaxNR = 3;
constexpr int kAttnStep = 16;               // keys per ring stage
constexpr int kAttnStages = 4;              // ring depth
template <int HD> __host__ __device__ constexpr int attn_stage_bytes() { return kKvPlanes * kAttnStep * HD * 2; }
// smem: the ring (kAttnStages x [hd/64][plane][16 keys][128 B], 128B-swizzled
// by TMA) + its full barriers; the S exchange lives in the GEMM ring's
// activation slots (idle during an attention phase, see ps_mega.cuh)
constexpr int attn_smem_bytes(int /*nw*/) { return kAttnStages * attn_stage_bytes<128>() + 64; }
constexpr int kAttnWarps = 4;               // consumer warps = item partials per item
static_assert(kAttnStages == kAttnWarps, "warp w consumes ring slot w (stages s = w mod 4 of an item)");
// Q^T fragments of an item, [k step][n-tile][hi|lo][lane] uint2, double-buffered
// by item parity (written by all 4 warps, one barrier per item)
constexpr int kAttnQBufBytes = (128 / 16) * kAttnMaxNR * 2 * 32 * 8;
constexpr int kAttnXAreaBytes = 2 * kAttnQBufBytes;
// n-tiles per row block.  Any choice gives the same per-row arithmetic (see
// above), so it is picked per forward for speed, from a sweep of the 8B with
// the count forced to 1 / 2 / 3 (`gpurun_out/s4q_nr.log`, 1K-16K keys, R = 3
// .. 17): the fewest n-tiles processed (row blocks x n-tiles each), ties to 2
// (3 n-tiles per pass run with more register pressure); a 3-n-tile window
// (R = 5-6 at g = 4) at up to 1.5K keys as three 1-n-tile passes (more,
// lighter items: the short attention phase is latency-bound; the bench's
// verify pass, 600 keys: 3.855 vs 3.89 ms).
__host__ __device__ constexpr int attn_nr(int rows, int n_keys) {
  const int tiles = (rows + 7) / 8;
  if (tiles <= 1) return 1;
#ifdef PS_ATTN_NR                           // A/B builds: n-tiles forced
  return PS_ATTN_NR < tiles ? PS_ATTN_NR : tiles;
#endif
  if (tiles == 2) return 2;
  if (tiles == 3) return n_keys <= 1536 ? 1 : 3;
  return ((tiles + 2) / 3) * 3 < ((tiles + 1) / 2) * 2 ? 3 : 2;
}

PS_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
PS_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
PS_DEV void mma16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// 8x8 b16 matrix transpose across the warp (lane l: row l / 4, columns 2 (l % 4) .. +1)
PS_DEV uint32_t movm_t(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
  return d;
}
// Split a pair of fp32 values into hi / lo packed bf16x2 registers.
PS_DEV void split_pack(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  __nv_bfloat16 h0, l0, h1, l1;
  split_bf16(x0, h0, l0);
  split_bf16(x1, h1, l1);
  hi = pack2(h0, h1);
  lo = pack2(l0, l1);
}
// Byte offset of (plane pl, key r, dim d; d % 8 == 0) in a ring stage laid out
// [hd/64][plane][16 keys][128 B] with the TMA 128B swizzle (16-byte chunk c of
// row r at c ^ (r & 7)): ldmatrix rows of 8 keys hit 8 distinct bank groups.
PS_DEV uint32_t attn_sw(int pl, int r, int d) {
  return (uint32_t)((d >> 6) * (kKvPlanes * kAttnStep * 128) + pl * (kAttnStep * 128) + r * 128 +
                    ((((d & 63) >> 3) ^ (r & 7)) << 4));
}

struct AttnGeom {
  int rows, nr, rb_rows, n_rb, n_keys, nsc, n_items;
  PS_DEV AttnGeom(const AttnParams& p) {
    const int R = p.step->R;
    rows = R * (p.H / p.hkv);
    n_keys = p.step->pos0 + R;
    nr = attn_nr(rows, n_keys);
    rb_rows = kAttnRB * nr;
    n_rb = (rows + rb_rows - 1) / rb_rows;
    const int nchunks = (n_keys + kAttnChunk - 1) / kAttnChunk;
    nsc = (nchunks + p.sc - 1) / p.sc;
    n_items = p.hkv * n_rb * nsc;
  }
  PS_DEV int first(int c, int G) const { return (int)((long long)c * n_items / G); }
  // item -> KV head, row block, item index j, key range [kbeg, kend), stages
  PS_DEV void item(const AttnParams& p, int it, int& kh, int& rb, int& j, int& kbeg, int& kend, int& ns) const {
    // row blocks fastest: the row blocks of one key range run back to back
    // (mostly on one CTA), so the second read of those K/V stages hits L2
    rb = it % n_rb;
    j = (it / n_rb) % nsc;
    kh = it / (nsc * n_rb);
    kbeg = j * p.sc * kAttnChunk;
    kend = min(n_keys, (j + 1) * p.sc * kAttnChunk);
    // stages, padded to a multiple of kAttnWarps (only the context's last item
    // pads: its extra stages are fully masked, exact no-ops)
    ns = ((kend - kbeg + kAttnStep - 1) / kAttnStep + kAttnWarps - 1) / kAttnWarps * kAttnWarps;
  }
};

// Ring producer state (one thread of the X-loader warp): the stream position
// of the next stage to issue and the KV row of its first key (plane 0).
struct AttnProducer {
  int item, s, ns, kbeg, kh;
  long long row;                       // pool row of key kbeg + 16 s, plane 0 (valid if more)
  bool more;
};
PS_DEV long long attn_row(const AttnParams& p, int kh, int k0) {
  const long long page = p.page_table[k0 >> p.page_shift];
  return page * p.rows_per_page + ((long long)(p.layer * kKvPlanes * p.hkv + kh) << p.page_shift) +
         (k0 & (p.page_size - 1));
}
PS_DEV void attn_producer_init(const AttnParams& p, const AttnGeom& gm, int it0, int it_end, AttnProducer& u) {
  u.more = it0 < it_end;
  if (!u.more) return;
  int rb, j, kend;
  u.item = it0;
  u.s = 0;
  gm.item(p, it0, u.kh, rb, j, u.kbeg, kend, u.ns);
  u.row = attn_row(p, u.kh, u.kbeg);
}
// advance to the next stage of the stream, then look up its row
PS_DEV void attn_producer_seek(const AttnParams& p, const AttnGeom& gm, int it_end, AttnProducer& u) {
  if (++u.s >= u.ns) {
    if (++u.item >= it_end) {
      u.more = false;
      return;
    }
    int rb, j, kend;
    gm.item(p, u.item, u.kh, rb, j, u.kbeg, kend, u.ns);
    u.s = 0;
  }
  // (a padded stage past the context loads the last key's page: any finite rows)
  u.row = attn_row(p, u.kh, min(u.kbeg + u.s * kAttnStep, gm.n_keys - 1));
}
// TMA of ring stage `seq` (buffer seq % 4): 16 keys x all four planes, one box
// per 64 dims.  Keys past the context are loaded too (finite: the pool is
// zeroed at stage creation) and masked.
template <int HD>
PS_DEV void attn_issue(const AttnParams& p, uint32_t ring_u32, uint32_t full_u32, uint32_t seq, long long row) {
  const int buf = seq % kAttnStages;
  const uint32_t bar = full_u32 + buf * 8;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(attn_stage_bytes<HD>())
               : "memory");
#pragma unroll
  for (int h = 0; h < HD / 64; ++h)
    tma_load_3d(ring_u32 + buf * attn_stage_bytes<HD>() + h * (kKvPlanes * kAttnStep * 128), p.kvmap, bar, h * 64,
                (int)row, 0, kEvictFirst);
}

// (noinline: ptxas allocates a called function's registers beside the
// caller's live ones, so the megakernel keeps little live across the call)
//
// Key split: warp w takes the stages s = w, w + 4, ... of every item (ring slot
// w: items are whole multiples of 4 stages and the CTA's stream starts at slot
// 0), over the whole head dimension, with its own online softmax state, and
// writes its own item partial (index 4 j + w).  Which keys a warp sees depends
// only on their absolute positions, so rows stay bit-identical for any R.  No
// per-stage exchange or barrier: one barrier per item publishes the item's
// Q^T fragments (each warp converts a quarter of the k steps).  S^T is
// accumulated in two chains (even / odd k steps) added at the end.
// NR = attn_nr(R g): n-tiles of 8 query rows per item.
template <int HD, int NR>
__device__ __noinline__ void attn_run(const AttnParams& p, uint8_t* ring, uint64_t* full, uint64_t* empty, uint8_t* xbuf,
                                      int tid, int cta, int ncta, uint32_t& seq) {
  constexpr int KS = HD / 16;         // 16-dim k steps of K Q^T
  constexpr int MT = HD / 16;         // 16-dim m tiles of V^T P^T
  constexpr uint32_t SB = attn_stage_bytes<HD>();
  constexpr uint32_t PL = kAttnStep * 128;   // plane stride inside a 64-dim block
  constexpr int QB = kAttnQBufBytes / 8;     // one Q buffer (uint2s)
  const AttnGeom gm(p);
  const int it0 = gm.first(cta, ncta), it_end = gm.first(cta + 1, ncta);
  if (it0 >= it_end) return;
  const int g = p.H / p.hkv, pos0 = p.step->pos0;
  const float* const qp = p.q;
  const int ld_q = p.ld_q;
  const float qscale = p.scale_log2;
  const int warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
  const uint32_t sb = smem_u32(ring) + warp * SB;       // this warp's ring slot
  // per-lane ldmatrix rows: K as the A operand (key rows), V^T as the A operand (transposed)
  const int kr = (lane & 7) + ((lane >> 3) & 1) * 8, kd = (lane >> 4) * 8;
  const int vr = (lane & 7) + (lane >> 4) * 8, vd = ((lane >> 3) & 1) * 8;
  uint2* const qs = reinterpret_cast<uint2*>(xbuf) + lane;
#if PS_TRACE
  if (tid == 0) PS_TRACE_STAMP(p.dbg, cta * 8 + 0);
  unsigned long long tr_wait = 0, tr_qk = 0, tr_pv = 0, tr_t = globaltimer();
#define PS_ATTN_LAP(acc)                         \
  do {                                           \
    const unsigned long long t_ = globaltimer(); \
    acc += t_ - tr_t;                            \
    tr_t = t_;                                   \
  } while (0)
#else
#define PS_ATTN_LAP(acc) \
  do {                   \
  } while (0)
#endif
  for (int it = it0; it < it_end; ++it) {
    int kh, rb, j, kbeg, kend, ns;
    gm.item(p, it, kh, rb, j, kbeg, kend, ns);
    const int m0 = rb * gm.rb_rows;
    const int mrows = min(gm.rb_rows, gm.rows - m0);
    uint2* const qb = qs + (it & 1) * QB;
    // ---- Q^T fragments of this item: this warp's k steps kk = warp mod 4
#pragma unroll
    for (int n = 0; n < NR; ++n) {
      // B fragment column n-index gq = query row 8 n + gq of the block
      const int m = n * 8 + gq;
      const int mg = m0 + m, r = mg / g, h = kh * g + mg % g;
      const int qo = m < mrows ? r * ld_q + h * HD : -1;
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        if ((kk & 3) != warp) continue;
        uint32_t bh[2], bl[2];
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          const int d = kk * 16 + tq * 2 + hf * 8;
          const float2 qv = qo >= 0 ? *reinterpret_cast<const float2*>(qp + qo + d) : make_float2(0.f, 0.f);
          split_pack(qv.x * qscale, qv.y * qscale, bh[hf], bl[hf]);
        }
        qb[((kk * NR + n) * 2 + 0) * 32] = make_uint2(bh[0], bh[1]);
        qb[((kk * NR + n) * 2 + 1) * 32] = make_uint2(bl[0], bl[1]);
      }
    }
    named_bar(2, 128);
    float mrow[NR][2], lrow[NR][2];
    float oacc[MT][NR][4];
#pragma unroll
    for (int n = 0; n < NR; ++n) {
      mrow[n][0] = mrow[n][1] = -INFINITY;
      lrow[n][0] = lrow[n][1] = 0.f;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) oacc[mt][n][0] = oacc[mt][n][1] = oacc[mt][n][2] = oacc[mt][n][3] = 0.f;
    }
    // causal limit of S^T column (row 8 n + 2 tq + e of the block): the row's position, within the item
    auto qpos_of = [&](int n, int e) { return min(kend - 1, pos0 + (m0 + n * 8 + tq * 2 + e) / g); };
    for (int st = warp; st < ns; st += kAttnWarps) {
      const uint32_t u = seq + st;           // ring sequence number (u % 4 == warp)
      mbar_wait(&full[warp], (u / kAttnStages) & 1);
      PS_ATTN_LAP(tr_wait);
      // ---- S^T = K Q^T over all dims: chains a (even k steps) and b (odd)
      float a[NR][4], b[NR][4];
#pragma unroll
      for (int n = 0; n < NR; ++n) a[n][0] = a[n][1] = a[n][2] = a[n][3] = b[n][0] = b[n][1] = b[n][2] = b[n][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        uint32_t kh4[4], kl4[4];
        const uint32_t ko = attn_sw(0, kr, kk * 16 + kd);
        ldsm_x4(sb + ko, kh4[0], kh4[1], kh4[2], kh4[3]);        // K_hi
        ldsm_x4(sb + PL + ko, kl4[0], kl4[1], kl4[2], kl4[3]);   // K_lo
#pragma unroll
        for (int n = 0; n < NR; ++n) {
          const uint2 qh2 = qb[((kk * NR + n) * 2 + 0) * 32], ql2 = qb[((kk * NR + n) * 2 + 1) * 32];
          float* acc = (kk & 1) ? b[n] : a[n];
          mma16816(acc, kh4, qh2.x, qh2.y);
          mma16816(acc, kh4, ql2.x, ql2.y);
          mma16816(acc, kl4, qh2.x, qh2.y);
        }
      }
      PS_ATTN_LAP(tr_qk);
      // ---- mask, online softmax
      const int k0 = kbeg + st * kAttnStep;
      float scale[NR][2];
      uint32_t pbh[NR][2], pbl[NR][2];     // P^T as B fragments (keys 0-7 / 8-15 of the stage), hi / lo
#pragma unroll
      for (int n = 0; n < NR; ++n) {
        float pv[4];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          // this thread's S^T entries of row 8 n + 2 tq + e: keys gq (c_e) and gq + 8 (c_{2+e})
          float sa = a[n][e] + b[n][e], sb8 = a[n][2 + e] + b[n][2 + e];
          const int qpos = qpos_of(n, e);
          if (k0 + gq > qpos) sa = -INFINITY;
          if (k0 + gq + 8 > qpos) sb8 = -INFINITY;
          float mx = fmaxf(sa, sb8);
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
          const float mn = fmaxf(mrow[n][e], mx);
          scale[n][e] = (mrow[n][e] == -INFINITY) ? 0.f : ex2_approx(mrow[n][e] - mn);
          mrow[n][e] = mn;
          const float pa = (mn == -INFINITY) ? 0.f : ex2_approx(sa - mn);
          const float pb = (mn == -INFINITY) ? 0.f : ex2_approx(sb8 - mn);
          // this lane's share of the row sum (its two keys); the lanes' shares
          // are added once per item (the max must be row-uniform, the sum not)
          lrow[n][e] = lrow[n][e] * scale[n][e] + (pa + pb);
          pv[e] = pa;
          pv[2 + e] = pb;
        }
        uint32_t h01, l01, h23, l23;
        split_pack(pv[0], pv[1], h01, l01);      // key gq, rows 2 tq, 2 tq + 1
        split_pack(pv[2], pv[3], h23, l23);      // key gq + 8
        pbh[n][0] = movm_t(h01);                 // -> row gq, keys 2 tq, 2 tq + 1 (the B layout)
        pbh[n][1] = movm_t(h23);
        pbl[n][0] = movm_t(l01);
        pbl[n][1] = movm_t(l23);
      }
      // ---- O^T = O^T * scale + V^T P^T over all dims
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        uint32_t vh[4], vl[4];
        const uint32_t vo = attn_sw(2, vr, mt * 16 + vd);
        ldsm_x4_t(sb + vo, vh[0], vh[1], vh[2], vh[3]);          // V_hi
        ldsm_x4_t(sb + PL + vo, vl[0], vl[1], vl[2], vl[3]);     // V_lo
#pragma unroll
        for (int n = 0; n < NR; ++n) {
          oacc[mt][n][0] *= scale[n][0]; oacc[mt][n][1] *= scale[n][1];
          oacc[mt][n][2] *= scale[n][0]; oacc[mt][n][3] *= scale[n][1];
          mma16816(oacc[mt][n], vh, pbh[n][0], pbh[n][1]);
          mma16816(oacc[mt][n], vl, pbh[n][0], pbh[n][1]);
          mma16816(oacc[mt][n], vh, pbl[n][0], pbl[n][1]);
        }
      }
      // this warp is done with the slot (K/V fragments are in registers)
      __syncwarp();
      if (lane == 0) mbar_arrive_n(&empty[warp], kAttnWarps);   // (the barrier counts 4 consumers)
      PS_ATTN_LAP(tr_pv);
    }
    seq += ns;
    // ---- this warp's item partial -> workspace [kh][4 j + warp][row][HD] (all dims)
    const size_t base = ((size_t)kh * p.max_chunks + (size_t)j * kAttnWarps + warp) * p.rows_cap + (size_t)m0;
#pragma unroll
    for (int n = 0; n < NR; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        float ls = lrow[n][e];                // row sum over the 8 key lanes (fixed tree)
        ls += __shfl_xor_sync(0xffffffffu, ls, 4);
        ls += __shfl_xor_sync(0xffffffffu, ls, 8);
        ls += __shfl_xor_sync(0xffffffffu, ls, 16);
        lrow[n][e] = ls;
      }
#pragma unroll
    for (int n = 0; n < NR; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = n * 8 + tq * 2 + e;
        if (m >= mrows) continue;           // a later row block's row (or none)
        float* op = p.ws_o + (base + m) * HD + gq;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          __stcg(op + mt * 16, oacc[mt][n][e]);
          __stcg(op + mt * 16 + 8, oacc[mt][n][2 + e]);
        }
        if (gq == 0) __stcg(reinterpret_cast<float2*>(p.ws_ml + (base + m) * 2), make_float2(mrow[n][e], lrow[n][e]));
      }
  }
#if PS_TRACE
  if (tid == 0) PS_TRACE_STAMP(p.dbg, cta * 8 + 4);
  if (tid == 0 && p.dbg) {
    p.dbg[cta * 8 + 5] = tr_wait;
    p.dbg[cta * 8 + 6] = tr_qk;
    p.dbg[cta * 8 + 7] = tr_pv;
  }
#endif
#undef PS_ATTN_LAP
}

// Combine of the item partials (next phase; kAttnWarps per item, partial
// 4 j + w from warp w of item j): one CTA per output row (kh, m),
// its 4 warps take the partials c = w, w + 4, ... (a split independent of the
// partial count, so the extra all-masked partials of a longer window add exact
// zeros: row-bucket invariance).  Per row M = max_c m_c, L = sum_c 2^(m_c - M)
// l_c, O = sum_c 2^(m_c - M) O_c / L; each warp sums its partials in order
// (8 O loads in flight), the 4 warp sums are added in warp order.
template <int HD>
PS_DEV void attn_combine(const AttnParams& p, float* xs, int tid, int cta, int ncta) {
  const StepIn* st = p.step;
  const int R = st->R, pos0 = st->pos0;
  const int g = p.H / p.hkv;
  const int rows = R * g;
  const int np = kAttnWarps * (((pos0 + R + kAttnChunk - 1) / kAttnChunk + p.sc - 1) / p.sc);   // item partials
  const int warp = tid >> 5, lane = tid & 31;
  constexpr int DPL = HD / 32;
  using VecT = typename std::conditional<DPL == 4, float4, float2>::type;
  constexpr int kIF = 8;                  // O loads in flight per warp
  const size_t cstride = (size_t)p.rows_cap;   // rows between partial c and c + 1 of a row
  for (int it = cta; it < p.hkv * rows; it += ncta) {
    const int kh = it / rows, mg = it % rows;
    const size_t rbase = (size_t)kh * p.max_chunks * cstride + mg;   // partial c of this row: rbase + c * cstride
    // this warp's first 32 partials' (m, l) go out before the M pass (they
    // do not depend on M: one round trip for both)
    float2 ml0 = make_float2(-INFINITY, 0.f);
    if (warp + 4 * lane < np) ml0 = __ldcg(reinterpret_cast<const float2*>(p.ws_ml + (rbase + (warp + 4 * lane) * cstride) * 2));
    float M = -INFINITY;
    for (int c = lane; c < np; c += 32) M = fmaxf(M, __ldcg(p.ws_ml + (rbase + c * cstride) * 2));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float acc[DPL];
#pragma unroll
    for (int t = 0; t < DPL; ++t) acc[t] = 0.f;
    float Lp = 0.f;
    // this warp's partials c = warp + 4 i; 32 of them per round (lane i holds c's scale)
    for (int i0 = 0; warp + 4 * i0 < np; i0 += 32) {
      const int cl = warp + 4 * (i0 + lane);
      float sc = 0.f;
      if (cl < np) {
        const float2 ml = i0 == 0 ? ml0 : __ldcg(reinterpret_cast<const float2*>(p.ws_ml + (rbase + cl * cstride) * 2));
        sc = (ml.x == -INFINITY) ? 0.f : exp2f(ml.x - M);
        Lp += sc * ml.y;
      }
      const int nh = min(32, (np - warp + 3) / 4 - i0);
      for (int q0 = 0; q0 < nh; q0 += kIF) {
        VecT ov[kIF];
#pragma unroll
        for (int q = 0; q < kIF; ++q)
          if (q0 + q < nh)
            ov[q] = __ldcg(reinterpret_cast<const VecT*>(p.ws_o + (rbase + (size_t)(warp + 4 * (i0 + q0 + q)) * cstride) * HD +
                                                         lane * DPL));
#pragma unroll
        for (int q = 0; q < kIF; ++q) {
          const float sq = __shfl_sync(0xffffffffu, sc, (q0 + q) & 31);
          if (q0 + q < nh) {
            if constexpr (DPL == 4) {
              acc[0] += sq * ov[q].x; acc[1] += sq * ov[q].y; acc[2] += sq * ov[q].z; acc[3] += sq * ov[q].w;
            } else {
              acc[0] += sq * ov[q].x; acc[1] += sq * ov[q].y;
            }
          }
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) Lp += __shfl_xor_sync(0xffffffffu, Lp, o);
    // ---- the 4 warp sums, in warp order
#pragma unroll
    for (int t = 0; t < DPL; ++t) xs[(warp * DPL + t) * 32 + lane] = acc[t];
    if (lane == 0) xs[4 * DPL * 32 + warp] = Lp;
    named_bar(1, 128);
    if (warp == 0) {
      float o[DPL];
#pragma unroll
      for (int t = 0; t < DPL; ++t) {
        o[t] = xs[(0 * DPL + t) * 32 + lane];
#pragma unroll
        for (int w = 1; w < 4; ++w) o[t] += xs[(w * DPL + t) * 32 + lane];
      }
      float L = xs[4 * DPL * 32 + 0];
#pragma unroll
      for (int w = 1; w < 4; ++w) L += xs[4 * DPL * 32 + w];
      const float invL = 1.0f / L;
      const int r = mg / g, h = kh * g + mg % g;
      __nv_bfloat16* dst = p.out + (size_t)r * p.ld_out + h * HD + lane * DPL;
#pragma unroll
      for (int t = 0; t < DPL; ++t) split_bf16(o[t] * invL, dst[t], dst[t + (size_t)kRowsCap * p.ld_out]);
    }
    named_bar(1, 128);
  }
}

// ------------------------------------------------------------------ argmax + compare + scan (a11)
struct ArgmaxParams {
  const StepIn* step;
  unsigned long long* amax; int n_tiles, amax_ld;   // amax[r]: per-row greedy key (atomicMax)
  StepOut* out;            // device
  StepOut* mirror;         // mapped pinned host memory (zero-copy), may be null
  const SynthParams* syn;  // may be null
  int vocab;               // full vocabulary (row-token range check)
  // tensor parallel (tp_n > 1): every rank's per-row keys, two parity slots
  // [2][kMaxRows] each (slot = gen_head & 1); amax is this rank's own block
  int tp_n;
  const unsigned long long* tp_keys[8];
};

PS_DEV int synth_token(const SynthParams* sp, int p) {
  // chained token of stage `level` at on-path generated index p (R24)
  int t = sp->S[p];
  for (int j = sp->top - 1; j >= sp->level; --j) {
    const uint64_t base = splitmix64(sp->seed ^ ((uint64_t)1 << 56) ^ ((uint64_t)j << 48));
    const uint64_t hu = splitmix64(base ^ (uint64_t)p);
    if (!((hu >> 11) < sp->thr[j])) {
      const uint64_t bd = splitmix64(sp->seed ^ ((uint64_t)2 << 56) ^ ((uint64_t)j << 48));
      const uint64_t hd = splitmix64(bd ^ (uint64_t)p);
      const uint64_t V = (uint64_t)sp->vocab;
      t = (int)(((uint64_t)t + 1 + hd % (V - 1)) % V);
    }
  }
  return t;
}

// Vocab argmax from the per-tile partials, synthetic override, compare + scan.
// NT threads (multiple of 32); s_pred: smem int[kMaxRows]; bar: named barrier id.
template <int NT>
PS_DEV void argmax_run(const ArgmaxParams& p, int tid, int* s_pred, int bar) {
  const StepIn* st = p.step;
  const int R = st->R;
  if (p.tp_n > 1) {
    // vocab-parallel lm_head: max over the ranks' keys (exact, order-free); the
    // other parity slot (previous head forward, read by every peer before this
    // forward's lm_head could complete on it) is reset for the next forward
    const int par = st->gen_head & 1;
    for (int row = tid; row < kMaxRows; row += NT) {
      if (row < R) {
        unsigned long long k = 0ull;
        for (int q = 0; q < p.tp_n; ++q) {
          const unsigned long long kq = __ldcg(p.tp_keys[q] + par * kMaxRows + row);
          k = kq > k ? kq : k;
        }
        s_pred[row] = (int)argmax_key_idx(k);
      }
      p.amax[(par ^ 1) * kMaxRows + row] = 0ull;
    }
  } else {
    for (int row = tid; row < R; row += NT) {
      s_pred[row] = (int)argmax_key_idx(__ldcg(&p.amax[row]));
      p.amax[row] = 0ull;                // reset the atomicMax slot for the next forward
    }
  }
  named_bar(bar, NT);
  if (tid < 32) {
    // one warp: lane j holds prediction row r0 + j (w <= 31 < 32 lanes)
    const int lane = tid;
    const int w = st->w;
    const int r0 = st->row0;             // prediction rows r0 .. r0 + w
    const bool live = lane <= w;
    const int d = lane < w ? st->tokens[r0 + 1 + lane] : -1;   // draft d_lane
    int pred = live ? s_pred[r0 + lane] : -1;
    if ((st->flags & kFlagSynth) && p.syn != nullptr && p.syn->len_S > 0 && st->syn_onpath) {
      // prediction row j's context is x ++ d[0:j]: on-path while d_t == S[p0+t]
      // for all t < j, i.e. for j <= the first draft that leaves S
      const int pj = st->syn_p0 + lane;
      const unsigned off = __ballot_sync(0xffffffffu, lane < w && (pj >= p.syn->len_S || d != p.syn->S[pj]));
      const int first_off = off ? __ffs(off) - 1 : 32;
      if (live && lane <= first_off && pj < p.syn->len_S) pred = synth_token(p.syn, pj);
    }
    // a = longest prefix with pred_j == d_j: first mismatching lane (ballot + ffs)
    const unsigned miss = __ballot_sync(0xffffffffu, lane < w && pred != d);
    const int a = miss ? __ffs(miss) - 1 : w;
    const int next = __shfl_sync(0xffffffffu, pred, a);
    // every row token must be a vocabulary id (device windows are not host-checked)
    const bool bad_tok = lane < R && (st->tokens[lane] < 0 || st->tokens[lane] >= p.vocab);
    const bool bad = __any_sync(0xffffffffu, bad_tok);
    p.out->pred[lane] = live ? pred : -1;
    if (p.mirror != nullptr) reinterpret_cast<volatile int*>(p.mirror)[4 + lane] = live ? pred : -1;
    if (lane == 0) {
      // KV now valid for positions < n + a, n - 1 = pos0 + row0 (the pending row)
      const int kv_len = st->pos0 + r0 + 1 + a;
      p.out->a = a;
      p.out->next = next;
      p.out->R = bad ? -1 : R;
      p.out->kv_len = kv_len;
      if (p.mirror != nullptr) {
        volatile int* m = reinterpret_cast<volatile int*>(p.mirror);
        m[0] = a;
        m[1] = next;
        m[3] = kv_len;
        __threadfence_system();
        m[2] = bad ? -1 : R;             // written last: the host polls it
        __threadfence_system();
      }
    }
  }
}

}  // namespace ps
