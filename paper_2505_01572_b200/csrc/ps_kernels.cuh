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
  int32_t flags;                   // kFlagLogits | kFlagSynth
  int32_t syn_p0;                  // generated index predicted by row row0 (= n - n_prompt)
  int32_t syn_onpath;              // 1 iff the committed context is on the target stream
  int32_t row0;                    // first prediction row (rows before it are KV catch-up)
  int32_t gen;                     // forwards so far on this stage (megakernel counter target)
  int32_t gen_head;                // forwards with lm_head so far (targets of the head phases)
  int32_t pad2[3];
  int32_t tokens[kRowsCap];        // row tokens: [pending, d_0, ..., d_{w-1}] (or a prefill chunk)
};
constexpr int kFlagLogits = 1;
constexpr int kFlagSynth = 2;

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
  const __nv_bfloat16* kv; const int32_t* page_table; int page_size; long long page_stride;
  int layer, hkv, H, hd;
  float scale_log2;                // log2(e) / sqrt(hd)
  int max_chunks, max_rb;
  float* ws_o;                     // [hkv][max_rb][max_chunks][rows per block][hd]
  float* ws_ml;                    // [hkv][max_rb][max_chunks][rows per block][2]
  unsigned* counters;              // [hkv][max_rb]
  __nv_bfloat16* out; int ld_out;
  unsigned long long* dbg;         // optional per-CTA stage stamps [cta][8] (first item)
};

constexpr int kAttnPad = 8;        // smem row padding (bf16 elements): conflict-free ldmatrix
// smem: K_hi, K_lo, V_hi, V_lo chunks [64][HD+8] bf16 + combine scratch (the
// query fragments live in registers, built from the fp32 q directly)
constexpr int attn_smem_bytes(int /*nw*/) { return kKvPlanes * kAttnChunk * (128 + kAttnPad) * 2 + 64 * 4 * 3 + 64; }
constexpr int kAttnSmem = attn_smem_bytes(8);

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
PS_DEV uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// Split a pair of fp32 values into hi / lo packed bf16x2 registers.
PS_DEV void split_pack(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  __nv_bfloat16 h0, l0, h1, l1;
  split_bf16(x0, h0, l0);
  split_bf16(x1, h1, l1);
  hi = pack2(h0, h1);
  lo = pack2(l0, l1);
}

// Issue (cp.async, one commit group) the K/V chunk (all four planes) of this
// CTA's first work item if it lies wholly in the context (positions < pos0:
// not rewritten by the coming QKV phase).  Returns the prefetched item id, or -1.
template <int HD, int NW>
PS_DEV int attn_prefetch_kv(const AttnParams& p, uint8_t* attn_smem, int tid, int cta) {
  constexpr int kRB = NW * 16, NT = NW * 32, LD = HD + kAttnPad, VPR = HD / 8;
  const StepIn* st = p.step;
  const int R = st->R, pos0 = st->pos0;
  const int rows = R * (p.H / p.hkv);
  const int n_rb = (rows + kRB - 1) / kRB;
  const int nchunks = (pos0 + R + kAttnChunk - 1) / kAttnChunk;
  if (cta >= p.hkv * n_rb * nchunks) return -1;
  const int c = cta % nchunks, kh = cta / (nchunks * n_rb);
  const int k0 = c * kAttnChunk;
  if (k0 + kAttnChunk > pos0) return -1;
  __nv_bfloat16* sKV = reinterpret_cast<__nv_bfloat16*>(attn_smem);
  const long long page = p.page_table[k0 / p.page_size];
  const int slot0 = k0 % p.page_size;
  for (int i = tid; i < kKvPlanes * kAttnChunk * VPR; i += NT) {
    const int pl = i / (kAttnChunk * VPR), row = (i / VPR) % kAttnChunk, cv = i % VPR;
    const __nv_bfloat16* src = p.kv + (size_t)page * p.page_stride +
                               ((size_t)((p.layer * kKvPlanes + pl) * p.hkv + kh) * p.page_size + slot0 + row) * HD + cv * 8;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sKV + (pl * kAttnChunk + row) * LD + cv * 8)),
                 "l"(src) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  return cta;
}

// S = Q K^T and O = P V with split-bf16 operands on mma.sync m16n8k16:
// (q_hi + q_lo)(k_hi + k_lo)^T ~ q_hi k_hi + q_lo k_hi + q_hi k_lo (the
// dropped lo*lo term is ~2^-16 relative), likewise P V.
template <int HD, int NW, bool kInlineCombine = true>
PS_DEV void attn_run(const AttnParams& p, uint8_t* attn_smem, int tid, int cta, int ncta, int bar,
                     int pref_item = -1) {
  constexpr int kRB = NW * 16;                          // query rows per block
  constexpr int NT = NW * 32;
  constexpr int LD = HD + kAttnPad;                     // smem row stride (elements)
  __nv_bfloat16* sKh = reinterpret_cast<__nv_bfloat16*>(attn_smem);
  __nv_bfloat16* sKl = sKh + kAttnChunk * LD;
  __nv_bfloat16* sVh = sKl + kAttnChunk * LD;
  __nv_bfloat16* sVl = sVh + kAttnChunk * LD;
  float* sM = reinterpret_cast<float*>(sVl + kAttnChunk * LD);   // combine scratch [64]
  int& s_last = *reinterpret_cast<int*>(sM + 3 * 64);
  const StepIn* st = p.step;
  const int R = st->R, pos0 = st->pos0;
  const int g = p.H / p.hkv;
  const int rows = R * g;
  const int n_rb = (rows + kRB - 1) / kRB;
  const int n_keys = pos0 + R;
  const int nchunks = (n_keys + kAttnChunk - 1) / kAttnChunk;
  const int warp = tid >> 5, lane = tid & 31;
  const int n_items = p.hkv * n_rb * nchunks;
  for (int item = cta; item < n_items; item += ncta) {
    const int c = item % nchunks;
    const int rb = (item / nchunks) % n_rb;
    const int kh = item / (nchunks * n_rb);
    const int m0 = rb * kRB;
    const int mrows = min(kRB, rows - m0);
    const int k0 = c * kAttnChunk;
    const int nk = min(kAttnChunk, n_keys - k0);
    const bool stamp = tid == 0 && item == cta;
    if (stamp) PS_TRACE_STAMP(p.dbg, cta * 8 + 0);
    const int nwarps_used = (mrows + 15) / 16;
    // ---- K/V chunk, four planes: cp.async (16 B, zero-fill past nk) -- every
    // copy in flight at once (skipped when prefetched during the QKV phase)
    const long long page = p.page_table[k0 / p.page_size];
    const int slot0 = k0 % p.page_size;
    constexpr int VPR = HD / 8;                          // 16-byte vectors per row
    for (int i = (item == pref_item) ? kKvPlanes * kAttnChunk * VPR : tid; i < kKvPlanes * kAttnChunk * VPR; i += NT) {
      const int pl = i / (kAttnChunk * VPR), row = (i / VPR) % kAttnChunk, cv = i % VPR;
      const int ok = row < nk ? 16 : 0;
      const __nv_bfloat16* src = p.kv + (size_t)page * p.page_stride +
                                 ((size_t)((p.layer * kKvPlanes + pl) * p.hkv + kh) * p.page_size + slot0 +
                                  (row < nk ? row : 0)) * HD + cv * 8;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(sKh + (pl * kAttnChunk + row) * LD + cv * 8)),
                   "l"(src), "r"(ok) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // ---- this warp's query fragments (A operand of m16n8k16, rows lane/4 and
    // lane/4 + 8, dims 2(lane%4) + {0,1} and + 8 of each 16-wide k step),
    // loaded straight from the fp32 q, pre-scaled, split into hi / lo
    uint32_t qh[HD / 16][4], ql[HD / 16][4];
    {
      int qoff[2];
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int m = warp * 16 + (lane >> 2) + hr * 8;
        const int mg = m0 + m, r = mg / g, h = kh * g + mg % g;
        qoff[hr] = m < mrows ? r * p.ld_q + h * HD : -1;
      }
      float2 qv[HD / 16][4];
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int o = qoff[j & 1];
          const int d = kk * 16 + (lane & 3) * 2 + (j >> 1) * 8;
          qv[kk][j] = (o >= 0 && warp < nwarps_used) ? *reinterpret_cast<const float2*>(p.q + o + d)
                                                     : make_float2(0.f, 0.f);
        }
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          split_pack(qv[kk][j].x * p.scale_log2, qv[kk][j].y * p.scale_log2, qh[kk][j], ql[kk][j]);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    named_bar(bar, NT);
    if (stamp) PS_TRACE_STAMP(p.dbg, cta * 8 + 1);
    if (warp < nwarps_used) {
      // ---- S = Q K^T for this warp's 16 rows x 64 keys
      float sacc[8][4];
#pragma unroll
      for (int j = 0; j < 8; ++j) sacc[j][0] = sacc[j][1] = sacc[j][2] = sacc[j][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
        for (int jp = 0; jp < 4; ++jp) {   // pairs of 8-key n-tiles
          const int krow = jp * 16 + (lane & 7) + ((lane >> 4) << 3);
          const int kcol = kk * 16 + ((lane >> 3) & 1) * 8;
          uint32_t b0, b1, b2, b3, c0, c1, c2, c3;
          ldsm_x4(smem_u32(sKh + krow * LD + kcol), b0, b1, b2, b3);
          ldsm_x4(smem_u32(sKl + krow * LD + kcol), c0, c1, c2, c3);
          mma16816(sacc[2 * jp], qh[kk], b0, b1);
          mma16816(sacc[2 * jp + 1], qh[kk], b2, b3);
          mma16816(sacc[2 * jp], ql[kk], b0, b1);
          mma16816(sacc[2 * jp + 1], ql[kk], b2, b3);
          mma16816(sacc[2 * jp], qh[kk], c0, c1);
          mma16816(sacc[2 * jp + 1], qh[kk], c2, c3);
        }
      }
      // ---- causal / length mask and chunk-local softmax (rows lane/4 and lane/4+8)
      float mrow[2] = {-INFINITY, -INFINITY};
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int m = warp * 16 + (lane >> 2) + hr * 8;
        const int qpos = pos0 + (m0 + m) / g;
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
          for (int e2 = 0; e2 < 2; ++e2) {
            const int key = j * 8 + (lane & 3) * 2 + e2;
            float& sv = sacc[j][hr * 2 + e2];
            if (key >= nk || k0 + key > qpos) sv = -INFINITY;
            mrow[hr] = fmaxf(mrow[hr], sv);
          }
        mrow[hr] = fmaxf(mrow[hr], __shfl_xor_sync(0xffffffffu, mrow[hr], 1));
        mrow[hr] = fmaxf(mrow[hr], __shfl_xor_sync(0xffffffffu, mrow[hr], 2));
      }
      float lrow[2] = {0.f, 0.f};
      uint32_t pah[4][4], pal[4][4];      // P as A fragments (hi / lo), 4 k-blocks of 16 keys
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float pv[4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int hr = q4 >> 1;
          pv[q4] = (mrow[hr] == -INFINITY) ? 0.f : exp2f(sacc[j][q4] - mrow[hr]);
          lrow[hr] += pv[q4];
        }
        const int kb = j >> 1, half2 = j & 1;
        split_pack(pv[0], pv[1], pah[kb][half2 * 2 + 0], pal[kb][half2 * 2 + 0]);
        split_pack(pv[2], pv[3], pah[kb][half2 * 2 + 1], pal[kb][half2 * 2 + 1]);
      }
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        lrow[hr] += __shfl_xor_sync(0xffffffffu, lrow[hr], 1);
        lrow[hr] += __shfl_xor_sync(0xffffffffu, lrow[hr], 2);
      }
      if (stamp) PS_TRACE_STAMP(p.dbg, cta * 8 + 2);
      // ---- O = P V  (16 rows x HD)
      float oacc[HD / 8][4];
#pragma unroll
      for (int n = 0; n < HD / 8; ++n) oacc[n][0] = oacc[n][1] = oacc[n][2] = oacc[n][3] = 0.f;
#pragma unroll
      for (int kb = 0; kb < 4; ++kb) {
#pragma unroll
        for (int np = 0; np < HD / 16; ++np) {
          const int vrow = kb * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
          const int vcol = np * 16 + (lane >> 4) * 8;
          uint32_t b0, b1, b2, b3, c0, c1, c2, c3;
          ldsm_x4_t(smem_u32(sVh + vrow * LD + vcol), b0, b1, b2, b3);
          ldsm_x4_t(smem_u32(sVl + vrow * LD + vcol), c0, c1, c2, c3);
          mma16816(oacc[2 * np], pah[kb], b0, b1);
          mma16816(oacc[2 * np + 1], pah[kb], b2, b3);
          mma16816(oacc[2 * np], pal[kb], b0, b1);
          mma16816(oacc[2 * np + 1], pal[kb], b2, b3);
          mma16816(oacc[2 * np], pah[kb], c0, c1);
          mma16816(oacc[2 * np + 1], pah[kb], c2, c3);
        }
      }
      if (stamp) PS_TRACE_STAMP(p.dbg, cta * 8 + 3);
      // ---- chunk partials -> workspace
      const size_t base = ((size_t)((kh * p.max_rb + rb) * p.max_chunks + c) * kRB);
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int m = warp * 16 + (lane >> 2) + hr * 8;
        float* op = p.ws_o + (base + m) * HD;
#pragma unroll
        for (int n = 0; n < HD / 8; ++n)
          __stcg(reinterpret_cast<float2*>(op + n * 8 + (lane & 3) * 2),
                 make_float2(oacc[n][hr * 2], oacc[n][hr * 2 + 1]));
        if ((lane & 3) == 0) __stcg(reinterpret_cast<float2*>(p.ws_ml + (base + m) * 2), make_float2(mrow[hr], lrow[hr]));
      }
    }
    if constexpr (!kInlineCombine) {    // partials only; attn_combine runs after a grid barrier
      named_bar(bar, NT);
      if (stamp) PS_TRACE_STAMP(p.dbg, cta * 8 + 4);
      continue;
    }
    fence_acq_rel_gpu();
    named_bar(bar, NT);
    if (tid == 0) s_last = atomicAdd(&p.counters[kh * p.max_rb + rb], 1u) == (unsigned)(nchunks - 1);
    named_bar(bar, NT);
    if (s_last) {
      fence_acq_rel_gpu();
      // combine: per row M = max_c m_c, L = sum_c 2^(m_c-M) l_c, O = sum_c 2^(m_c-M) O_c / L
      const size_t rbase = (size_t)(kh * p.max_rb + rb) * p.max_chunks;
      for (int m = warp; m < mrows; m += NW) {
        float M = -INFINITY;
        for (int cc = lane; cc < nchunks; cc += 32)
          M = fmaxf(M, __ldcg(p.ws_ml + ((rbase + cc) * kRB + m) * 2));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        float Lp = 0.f;
        for (int cc = lane; cc < nchunks; cc += 32) {
          const float2 ml = __ldcg(reinterpret_cast<const float2*>(p.ws_ml + ((rbase + cc) * kRB + m) * 2));
          Lp += (ml.x == -INFINITY) ? 0.f : exp2f(ml.x - M) * ml.y;
        }
        // fixed-order sum over chunks: lanes hold chunk-strided partials, reduce by tree
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) Lp += __shfl_xor_sync(0xffffffffu, Lp, o);
        const float invL = 1.0f / Lp;
        constexpr int DPL = HD / 32;   // dims per lane
        float acc[DPL];
#pragma unroll
        for (int t = 0; t < DPL; ++t) acc[t] = 0.f;
#pragma unroll 8
        for (int cc = 0; cc < nchunks; ++cc) {
          const float mc = __ldcg(p.ws_ml + ((rbase + cc) * kRB + m) * 2);
          const float sc = (mc == -INFINITY) ? 0.f : exp2f(mc - M);
          const float* op = p.ws_o + ((rbase + cc) * kRB + m) * HD + lane * DPL;
          if constexpr (DPL == 4) {
            const float4 o4 = __ldcg(reinterpret_cast<const float4*>(op));
            acc[0] += sc * o4.x; acc[1] += sc * o4.y; acc[2] += sc * o4.z; acc[3] += sc * o4.w;
          } else {
            const float2 o2 = __ldcg(reinterpret_cast<const float2*>(op));
            acc[0] += sc * o2.x; acc[1] += sc * o2.y;
          }
        }
        const int mg = m0 + m, r = mg / g, h = kh * g + mg % g;
        __nv_bfloat16* dst = p.out + (size_t)r * p.ld_out + h * HD + lane * DPL;
#pragma unroll
        for (int t = 0; t < DPL; ++t) split_bf16(acc[t] * invL, dst[t], dst[t + (size_t)kRowsCap * p.ld_out]);
      }
      if (tid == 0) p.counters[kh * p.max_rb + rb] = 0u;
    }
    named_bar(bar, NT);
  }
}

// Combine of the chunk partials written by attn_run<.., false>: one warp per
// output row (kh, m); lanes hold HD/32 dims.  Per row M = max_c m_c, L = sum_c
// 2^(m_c - M) l_c, O = sum_c 2^(m_c - M) O_c / L in chunk order.  Lane c loads
// chunk c's (m, l) once (its scale reaches the other lanes by shuffles) and
// the O loads of 4 chunks are issued before any is used.
template <int HD, int kRB>
PS_DEV void attn_combine(const AttnParams& p, int gwarp, int nwarps_total) {
  const StepIn* st = p.step;
  const int R = st->R, pos0 = st->pos0;
  const int g = p.H / p.hkv;
  const int rows = R * g;
  const int nchunks = (pos0 + R + kAttnChunk - 1) / kAttnChunk;
  const int lane = threadIdx.x & 31;
  constexpr int DPL = HD / 32;
  using VecT = typename std::conditional<DPL == 4, float4, float2>::type;
  for (int item = gwarp; item < p.hkv * rows; item += nwarps_total) {
    const int kh = item / rows, mg = item % rows;
    const int rb = mg / kRB, m = mg % kRB;
    const size_t rbase = (size_t)(kh * p.max_rb + rb) * p.max_chunks;
    float acc[DPL];
#pragma unroll
    for (int t = 0; t < DPL; ++t) acc[t] = 0.f;
    float M = -INFINITY;
    for (int c0 = 0; c0 < nchunks; c0 += 32)
      if (c0 + lane < nchunks) M = fmaxf(M, __ldcg(p.ws_ml + ((rbase + c0 + lane) * kRB + m) * 2));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float Lp = 0.f;
    for (int c0 = 0; c0 < nchunks; c0 += 32) {
      float sc = 0.f;                    // 2^(m_c - M) of chunk c0 + lane
      if (c0 + lane < nchunks) {
        const float2 ml = __ldcg(reinterpret_cast<const float2*>(p.ws_ml + ((rbase + c0 + lane) * kRB + m) * 2));
        sc = (ml.x == -INFINITY) ? 0.f : exp2f(ml.x - M);
        Lp += sc * ml.y;
      }
      const int nh = min(32, nchunks - c0);
      for (int q0 = 0; q0 < nh; q0 += 4) {
        VecT ov[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q0 + q < nh)
            ov[q] = __ldcg(reinterpret_cast<const VecT*>(p.ws_o + ((rbase + c0 + q0 + q) * kRB + m) * HD + lane * DPL));
#pragma unroll
        for (int q = 0; q < 4; ++q) {
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
    // fixed-order sum over chunks: lanes hold chunk-strided partials, reduce by tree
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) Lp += __shfl_xor_sync(0xffffffffu, Lp, o);
    const float invL = 1.0f / Lp;
    const int r = mg / g, h = kh * g + mg % g;
    __nv_bfloat16* dst = p.out + (size_t)r * p.ld_out + h * HD + lane * DPL;
#pragma unroll
    for (int t = 0; t < DPL; ++t) split_bf16(acc[t] * invL, dst[t], dst[t + (size_t)kRowsCap * p.ld_out]);
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
