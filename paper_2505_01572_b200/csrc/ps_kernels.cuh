// ps_kernels.cuh — the verify-pass kernels (sm_100a).
//
//   embed_kernel        a1+a2+a3: window rows -> x (fp32 residual), x∘g (bf16 GEMM
//                        operand) and per-128-column sum-of-squares slots
//   gemm_kernel         a4/a7/a8/a9/a10: persistent stream-K skinny GEMM on tcgen05
//                        (swap-AB: weights are the M=128 side, the R<=32 rows the
//                        N side), TMA-staged weights with a STAGES-deep mbarrier
//                        ring, TMEM accumulators double-buffered, fused epilogues:
//                          EPI_QKV    RMSNorm row scale + RoPE + paged KV append (a3,a5)
//                          EPI_RESID  residual add + next RMSNorm operand + sumsq (a7,a9)
//                          EPI_SWIGLU RMSNorm row scale + SiLU(gate)*up           (a8)
//                          EPI_LMHEAD final-norm scale + fp32 logits + per-tile
//                                     (max,idx) argmax partials                   (a10)
//                          EPI_STORE  plain fp32 store (unit tests)
//   attn_kernel         a6: split-KV decode attention over the paged KV cache,
//                        fixed 64-key chunks at absolute positions, causal inside the
//                        window, GQA; deterministic last-CTA combine
//   argmax_scan_kernel  a11 (+a13 data): vocab argmax from the partials, synthetic
//                        override (benchmarks), draft compare, first-mismatch scan
//
// RMSNorm is applied as a deferred row scale: the producer of x writes the bf16
// operand x∘g and per-slot sums of x^2; the consumer GEMM multiplies its output
// row r by rstd_r = 1/sqrt(mean(x_r^2)+eps)  ((x∘g)·W^T scaled by rstd is the
// RMSNorm'd product, PAPER-independent algebra).
#pragma once
#include "ps_device.cuh"

namespace ps {

constexpr int kMaxRows = 32;       // max rows per forward (w <= 31)
constexpr int kAttnChunk = 64;     // keys per split-KV chunk (absolute positions)

struct StepIn {                    // written by the host before every forward
  int32_t R;                       // rows in this forward, 1..kMaxRows
  int32_t pos0;                    // absolute position of row 0
  int32_t w;                       // drafts in the window (rows 1..w), verify only
  int32_t flags;                   // kFlagLogits | kFlagSynth
  int32_t syn_p0;                  // generated index predicted by row row0 (= n - n_prompt)
  int32_t syn_onpath;              // 1 iff the committed context is on the target stream
  int32_t row0;                    // first prediction row (rows before it are KV catch-up)
  int32_t pad;
  int32_t tokens[kMaxRows];        // row tokens: [pending, d_0, ..., d_{w-1}]
};
constexpr int kFlagLogits = 1;
constexpr int kFlagSynth = 2;

struct StepOut {                   // written by argmax_scan_kernel
  int32_t a, next, R, pad;
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
  // EPI_STORE
  float* out; int ld_out;
  // stream-K fixup
  float* ws; unsigned* counters;
};

// ------------------------------------------------------------------ stream-K partition
// CTA c of G owns units [b_c, b_{c+1}), b_c = floor(c*U/G); units are
// (tile, k-block) pairs in tile-major order.
PS_DEV long long sk_begin(long long U, int G, int c) { return U * c / G; }
PS_DEV int sk_owner(long long U, int G, long long u) { return (int)(((u + 1) * G - 1) / U); }

template <int RP, int STAGES, bool GU>
struct GemmSmem {
  static constexpr int kABytes = 128 * 64 * 2;      // 16 KB weight tile (128 rows x 64 K)
  static constexpr int kXBytes = RP * 64 * 2;       // activation tile (RP rows x 64 K)
  static constexpr int kScratch = 128 * (RP + 1) * 4;
  static constexpr int kOffX = STAGES * kABytes;
  static constexpr int kOffScratch = kOffX + STAGES * kXBytes;
  static constexpr int kOffRed = kOffScratch + kScratch;            // u64 [4][RP]
  static constexpr int kOffRstd = kOffRed + 4 * RP * 8;             // float [RP]
  static constexpr int kOffBar = (kOffRstd + RP * 4 + 7) / 8 * 8;   // full, empty, tfull[2], tempty[2]
  static constexpr int kOffMisc = kOffBar + (2 * STAGES + 4) * 8;   // tmem base, flag
  static constexpr int kBytes = kOffMisc + 16 + 1024;               // + alignment slack
};

template <int RP>
PS_DEV void load_acc(uint32_t taddr, float* v) {
  tmem_ld16(taddr, v);
  if constexpr (RP == 32) tmem_ld16(taddr + 16, v + 16);
}

template <int RP, int STAGES, bool GU>
__global__ void __launch_bounds__(256, 1)
gemm_kernel(const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mA1,
            const __grid_constant__ CUtensorMap mA2, const __grid_constant__ CUtensorMap mX,
            const __grid_constant__ GemmParams p) {
  using L = GemmSmem<RP, STAGES, GU>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sX = smem + L::kOffX;
  float* scratch = (float*)(smem + L::kOffScratch);
  unsigned long long* red = (unsigned long long*)(smem + L::kOffRed);
  float* rstd = (float*)(smem + L::kOffRstd);
  uint64_t* full = (uint64_t*)(smem + L::kOffBar);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(smem + L::kOffMisc);
  volatile int* flag = (volatile int*)(smem + L::kOffMisc + 4);

  constexpr int kTmemCols = RP == 16 ? 32 : 64;
  constexpr uint32_t kIdesc = idesc_bf16_f32<128, RP>();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long U = (long long)p.n_tiles * p.kb_total;
  const int G = gridDim.x, c = blockIdx.x;
  const long long u_begin = sk_begin(U, G, c), u_end = sk_begin(U, G, c + 1);
  const int kbt = p.kb_total;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&mA0);
    if (GU || p.mode == EPI_QKV) tma_prefetch_desc(&mA1);
    if (p.mode == EPI_QKV) tma_prefetch_desc(&mA2);
    tma_prefetch_desc(&mX);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 128); }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch_dependents();

  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0) {
      auto load_A = [&](long long u, int s) {
        const int t = (int)(u / kbt), kb = (int)(u % kbt);
        uint8_t* dst = sA + s * L::kABytes;
        if constexpr (GU) {
          tma_load_2d(dst, &mA0, &full[s], kb * 64, t * 64, kEvictFirst);
          tma_load_2d(dst + 64 * 128, &mA1, &full[s], kb * 64, t * 64, kEvictFirst);
        } else if (p.mode == EPI_QKV) {
          if (t < p.t1) tma_load_2d(dst, &mA0, &full[s], kb * 64, t * 128, kEvictFirst);
          else if (t < p.t2) tma_load_2d(dst, &mA1, &full[s], kb * 64, (t - p.t1) * 128, kEvictFirst);
          else tma_load_2d(dst, &mA2, &full[s], kb * 64, (t - p.t2) * 128, kEvictFirst);
        } else {
          tma_load_2d(dst, &mA0, &full[s], kb * 64, t * 128, kEvictFirst);
        }
      };
      auto load_X = [&](long long u, int s) {
        const int kb = (int)(u % kbt);
        tma_load_2d(sX + s * L::kXBytes, &mX, &full[s], kb * 64, 0, kEvictLast);
      };
      const long long n_units = u_end - u_begin;
      const int pre = (int)(n_units < STAGES ? n_units : STAGES);
      // Weights do not depend on the previous kernel: stream them before the
      // grid dependency resolves (PDL), then fetch the activation tiles.
      for (int i = 0; i < pre; ++i) {
        mbar_arrive_expect_tx(&full[i], L::kABytes + L::kXBytes);
        load_A(u_begin + i, i);
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i) load_X(u_begin + i, i);
      int stage = 0;
      uint32_t phase = 1;   // ring wrapped once by the prologue (if pre == STAGES)
      for (long long u = u_begin + pre; u < u_end; ++u) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], L::kABytes + L::kXBytes);
        load_A(u, stage);
        load_X(u, stage);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      long long u = u_begin;
      while (u < u_end) {
        const int t = (int)(u / kbt);
        const long long seg_begin = u;
        const long long seg_end = min(u_end, (long long)(t + 1) * kbt);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem + acc * RP;
        for (; u < seg_end; ++u) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * L::kABytes);
          const uint32_t x0 = smem_u32(sX + stage * L::kXBytes);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_bf16(dcol, smem_desc_sw128(a0 + 32 * k), smem_desc_sw128(x0 + 32 * k), kIdesc,
                     (u != seg_begin || k > 0) ? 1u : 0u);
          mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue (128 threads, TMEM lane = e) =================
    const int e = threadIdx.x - 128;
    const int quarter = warp - 4;
    pdl_wait();
    const StepIn* st = p.step;
    const int R = st->R;
    const int pos0 = st->pos0;
    if (e < RP) {
      float r_ = 1.0f;
      if (p.ss_in != nullptr) {
        float s = 0.f;
        for (int j = 0; j < p.ss_n; ++j) s += p.ss_in[e * p.ss_ld + j];
        r_ = rsqrtf(s * p.inv_d + p.eps);
      }
      rstd[e] = r_;
    }
    named_bar(1, 128);
    int acc = 0;
    uint32_t acc_phase = 0;
    long long u = u_begin;
    while (u < u_end) {
      const int t = (int)(u / kbt);
      const long long seg_begin = u;
      const long long seg_end = min(u_end, (long long)(t + 1) * kbt);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      float v[RP];
      load_acc<RP>(tmem + ((uint32_t)(quarter * 32) << 16) + acc * RP, v);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      u = seg_end;

      // ---- stream-K fixup: deterministic, fixed segment order ----
      const long long tile_u0 = (long long)t * kbt;
      if (!(seg_begin == tile_u0 && seg_end == tile_u0 + kbt)) {
        const int first = sk_owner(U, G, tile_u0);
        const int nseg = sk_owner(U, G, tile_u0 + kbt - 1) - first + 1;
        const int seg = c - first;
        float* wsp = p.ws + (size_t)(t * p.maxseg) * RP * 128;
#pragma unroll
        for (int r = 0; r < RP; ++r) __stcg(&wsp[((size_t)seg * RP + r) * 128 + e], v[r]);
        __threadfence();
        named_bar(1, 128);
        if (e == 0) *flag = (atomicAdd(&p.counters[t], 1u) == (unsigned)(nseg - 1)) ? 1 : 0;
        named_bar(1, 128);
        const int last = *flag;
        named_bar(1, 128);
        if (!last) continue;
        __threadfence();
#pragma unroll
        for (int r = 0; r < RP; ++r) {
          float s = 0.f;
          for (int q = 0; q < nseg; ++q) s += (q == seg) ? v[r] : __ldcg(&wsp[((size_t)q * RP + r) * 128 + e]);
          v[r] = s;
        }
        if (e == 0) p.counters[t] = 0u;
      }

      // ---- fused epilogues ----
      if (p.mode == EPI_STORE) {
        const int f = t * 128 + e;
        if (f < p.N)
          for (int r = 0; r < R; ++r) p.out[(size_t)r * p.ld_out + f] = v[r];
      } else if (p.mode == EPI_RESID) {
        const int f = t * 128 + e;
        const bool ok = f < p.N;
        const float g = ok ? __bfloat162float(p.gain[f]) : 0.f;
#pragma unroll
        for (int r = 0; r < RP; ++r) {
          float sq = 0.f;
          if (r < R && ok) {
            const float xn = p.x[(size_t)r * p.ld_x + f] + v[r];
            p.x[(size_t)r * p.ld_x + f] = xn;
            p.xg[(size_t)r * p.ld_xg + f] = __float2bfloat16(xn * g);
            sq = xn * xn;
          }
          sq = warp_sum(sq);
          if (lane == 0) scratch[quarter * RP + r] = sq;
        }
        named_bar(1, 128);
        if (e < R)
          p.ss_out[(size_t)e * p.ss_out_ld + t] =
              ((scratch[0 * RP + e] + scratch[1 * RP + e]) + scratch[2 * RP + e]) + scratch[3 * RP + e];
        named_bar(1, 128);
      } else if (p.mode == EPI_SWIGLU) {
#pragma unroll
        for (int r = 0; r < RP; ++r) scratch[e * (RP + 1) + r] = v[r] * rstd[r];
        named_bar(1, 128);
        if (e < 64) {
          const int f = t * 64 + e;
          if (f < p.N)
            for (int r = 0; r < R; ++r) {
              const float gt = scratch[e * (RP + 1) + r];
              const float up = scratch[(e + 64) * (RP + 1) + r];
              p.h[(size_t)r * p.ld_h + f] = __float2bfloat16(gt / (1.0f + __expf(-gt)) * up);
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
#pragma unroll
          for (int r = 0; r < RP; ++r) scratch[e * (RP + 1) + r] = v[r];
          named_bar(1, 128);
          const int pe = e ^ half;
          const int j = i & (half - 1);
          for (int r = 0; r < R; ++r) {
            const float2 cs = p.rope_cs[(size_t)(pos0 + r) * half + j];
            const float pv = scratch[pe * (RP + 1) + r];
            v[r] = (i < half) ? (v[r] * cs.x - pv * cs.y) : (v[r] * cs.x + pv * cs.y);
          }
          named_bar(1, 128);
        }
        if (f < nrows) {
          if (kind == 0) {
            for (int r = 0; r < R; ++r) p.q[(size_t)r * p.ld_q + f] = v[r];
          } else {
            const int kh = f / hd;
            for (int r = 0; r < R; ++r) {
              const int pos = pos0 + r;
              const long long page = p.page_table[pos / p.page_size];
              const int slot = pos % p.page_size;
              const size_t off = (size_t)page * p.page_stride +
                                 ((size_t)((p.layer * 2 + (kind - 1)) * p.hkv + kh) * p.page_size + slot) * hd + i;
              p.kv[off] = __float2bfloat16(v[r]);
            }
          }
        }
      } else {  // EPI_LMHEAD
        const int f = t * 128 + e;
        const bool ok = f < p.N;
#pragma unroll
        for (int r = 0; r < RP; ++r) {
          const float z = v[r] * rstd[r];
          if (ok && r < R && p.logits != nullptr) p.logits[(size_t)r * p.ld_logits + f] = z;
          unsigned long long k = ok ? argmax_key(z, (uint32_t)f) : 0ull;
          k = warp_max_u64(k);
          if (lane == 0) red[quarter * RP + r] = k;
        }
        named_bar(1, 128);
        if (e < R) {
          unsigned long long k = red[e];
          for (int q = 1; q < 4; ++q) k = red[q * RP + e] > k ? red[q * RP + e] : k;
          p.amax[(size_t)e * p.amax_ld + t] = k;
        }
        named_bar(1, 128);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<kTmemCols>(tmem);
}

// ------------------------------------------------------------------ embed (a1-a3)
struct EmbedParams {
  const StepIn* step;
  const __nv_bfloat16* embed; int d;
  const __nv_bfloat16* gain;
  float* x; int ld_x;
  __nv_bfloat16* xg; int ld_xg;
  float* ss; int ss_ld;
};

__global__ void __launch_bounds__(128) embed_kernel(const __grid_constant__ EmbedParams p) {
  pdl_wait();
  pdl_launch_dependents();
  const int r = blockIdx.x;
  if (r >= p.step->R) return;
  const int tok = p.step->tokens[r];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nslots = (p.d + 127) / 128;
  const __nv_bfloat16* src = p.embed + (size_t)tok * p.d;
  for (int j = warp; j < nslots; j += 4) {
    float sq = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int col = j * 128 + lane * 4 + k;
      if (col < p.d) {
        const float xv = __bfloat162float(src[col]);
        p.x[(size_t)r * p.ld_x + col] = xv;
        p.xg[(size_t)r * p.ld_xg + col] = __float2bfloat16(xv * __bfloat162float(p.gain[col]));
        sq += xv * xv;
      }
    }
    sq = warp_sum(sq);
    if (lane == 0) p.ss[(size_t)r * p.ss_ld + j] = sq;
  }
}

// ------------------------------------------------------------------ attention (a6)
struct AttnParams {
  const StepIn* step;
  const float* q; int ld_q;
  const __nv_bfloat16* kv; const int32_t* page_table; int page_size; long long page_stride;
  int layer, hkv, H, hd;
  float scale;
  int max_chunks;
  float* ws_o;     // [H][max_chunks][kMaxRows][hd]
  float* ws_ml;    // [H][max_chunks][kMaxRows][2]
  unsigned* counters;
  __nv_bfloat16* out; int ld_out;
};

// One work item = (query head h, chunk c of kAttnChunk keys at absolute
// positions [c*64, c*64+64)).  Scores, softmax and P·V in fp32 on CUDA cores.
constexpr int kAttnSmem = 2 * kAttnChunk * 128 * 2 + kMaxRows * 128 * 4 + kMaxRows * (kAttnChunk + 1) * 4 + 16;

__global__ void __launch_bounds__(128) attn_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ __align__(16) uint8_t attn_smem[];
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(attn_smem);
  __nv_bfloat16* sV = sK + kAttnChunk * 128;
  float* sQ = reinterpret_cast<float*>(sV + kAttnChunk * 128);
  float* sP = sQ + kMaxRows * 128;
  int& s_last = *reinterpret_cast<int*>(sP + kMaxRows * (kAttnChunk + 1));
  pdl_wait();
  pdl_launch_dependents();
  const int R = p.step->R, pos0 = p.step->pos0;
  const int n_keys = pos0 + R;
  const int nchunks = (n_keys + kAttnChunk - 1) / kAttnChunk;
  const int hd = p.hd, g = p.H / p.hkv;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int item = blockIdx.x; item < p.H * nchunks; item += gridDim.x) {
    const int h = item / nchunks, c = item % nchunks, kh = h / g;
    const int k0 = c * kAttnChunk;
    const int nk = min(kAttnChunk, n_keys - k0);
    // K/V chunk: one page holds page_size >= 64 consecutive positions.
    const int page = p.page_table[k0 / p.page_size];
    const int slot0 = k0 % p.page_size;
    const __nv_bfloat16* Kp = p.kv + (size_t)page * p.page_stride +
                              ((size_t)((p.layer * 2 + 0) * p.hkv + kh) * p.page_size + slot0) * hd;
    const __nv_bfloat16* Vp = p.kv + (size_t)page * p.page_stride +
                              ((size_t)((p.layer * 2 + 1) * p.hkv + kh) * p.page_size + slot0) * hd;
    const int nvec = nk * hd / 8;
    for (int i = tid; i < nvec; i += 128) {
      reinterpret_cast<uint4*>(sK)[i] = reinterpret_cast<const uint4*>(Kp)[i];
      reinterpret_cast<uint4*>(sV)[i] = reinterpret_cast<const uint4*>(Vp)[i];
    }
    for (int i = tid; i < R * hd; i += 128) sQ[i] = p.q[(size_t)(i / hd) * p.ld_q + h * hd + (i % hd)];
    __syncthreads();
    for (int i = tid; i < R * kAttnChunk; i += 128) {
      const int r = i / kAttnChunk, j = i % kAttnChunk;
      float s = -INFINITY;
      if (j < nk && k0 + j <= pos0 + r) {   // causal: key position <= query position
        s = 0.f;
        const float* qr = sQ + r * hd;
        const __nv_bfloat16* kj = sK + j * hd;
        for (int d = 0; d < hd; d += 2) {
          const float2 kf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(kj + d));
          s = fmaf(qr[d], kf.x, s);
          s = fmaf(qr[d + 1], kf.y, s);
        }
        s *= p.scale;
      }
      sP[r * (kAttnChunk + 1) + j] = s;
    }
    __syncthreads();
    float* mlp = p.ws_ml + ((size_t)(h * p.max_chunks + c) * kMaxRows) * 2;
    for (int r = warp; r < R; r += 4) {
      float* row = sP + r * (kAttnChunk + 1);
      const float a0 = row[lane], a1 = row[lane + 32];
      float m = fmaxf(a0, a1);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      float e0 = 0.f, e1 = 0.f;
      if (m != -INFINITY) { e0 = __expf(a0 - m); e1 = __expf(a1 - m); }
      row[lane] = e0;
      row[lane + 32] = e1;
      const float l = warp_sum(e0 + e1);
      if (lane == 0) { mlp[r * 2 + 0] = m; mlp[r * 2 + 1] = l; }
    }
    __syncthreads();
    if (tid < hd) {
      float* op = p.ws_o + ((size_t)(h * p.max_chunks + c) * kMaxRows) * hd;
      for (int r = 0; r < R; ++r) {
        const float* pr = sP + r * (kAttnChunk + 1);
        float acc = 0.f;
        for (int j = 0; j < nk; ++j) acc = fmaf(pr[j], __bfloat162float(sV[j * hd + tid]), acc);
        __stcg(&op[(size_t)r * hd + tid], acc);
      }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&p.counters[h], 1u) == (unsigned)(nchunks - 1);
    __syncthreads();
    if (s_last) {
      __threadfence();
      if (tid < hd) {
        for (int r = 0; r < R; ++r) {
          float M = -INFINITY;
          for (int cc = 0; cc < nchunks; ++cc)
            M = fmaxf(M, __ldcg(&p.ws_ml[((size_t)(h * p.max_chunks + cc) * kMaxRows + r) * 2]));
          float O = 0.f, Lsum = 0.f;
          for (int cc = 0; cc < nchunks; ++cc) {
            const size_t base = (size_t)(h * p.max_chunks + cc) * kMaxRows + r;
            const float mc = __ldcg(&p.ws_ml[base * 2]);
            const float sc = (mc == -INFINITY) ? 0.f : __expf(mc - M);
            Lsum += sc * __ldcg(&p.ws_ml[base * 2 + 1]);
            O += sc * __ldcg(&p.ws_o[base * hd + tid]);
          }
          p.out[(size_t)r * p.ld_out + h * hd + tid] = __float2bfloat16(O / Lsum);
        }
      }
      if (tid == 0) p.counters[h] = 0u;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ argmax + compare + scan (a11)
struct ArgmaxParams {
  const StepIn* step;
  const unsigned long long* amax; int n_tiles, amax_ld;
  StepOut* out;            // device
  StepOut* mirror;         // mapped pinned host memory (zero-copy), may be null
  const SynthParams* syn;  // may be null
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

__global__ void __launch_bounds__(1024) argmax_scan_kernel(const __grid_constant__ ArgmaxParams p) {
  __shared__ int s_pred[kMaxRows];
  pdl_wait();
  pdl_launch_dependents();
  const StepIn* st = p.step;
  const int R = st->R;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < R) {
    unsigned long long k = 0;
    for (int t = lane; t < p.n_tiles; t += 32) {
      const unsigned long long v = p.amax[(size_t)warp * p.amax_ld + t];
      k = v > k ? v : k;
    }
    k = warp_max_u64(k);
    if (lane == 0) s_pred[warp] = (int)argmax_key_idx(k);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int w = st->w;
    const int r0 = st->row0;             // prediction rows r0 .. r0 + w
    if ((st->flags & kFlagSynth) && p.syn != nullptr && p.syn->len_S > 0 && st->syn_onpath) {
      // prediction row j's context is x ++ d[0:j]; on-path while the drafts follow S
      bool on = true;
      for (int j = 0; j <= w && on; ++j) {
        const int pj = st->syn_p0 + j;
        if (pj >= p.syn->len_S) break;
        s_pred[r0 + j] = synth_token(p.syn, pj);
        if (j < w) on = (st->tokens[r0 + 1 + j] == p.syn->S[pj]);
      }
    }
    int a = 0;
    while (a < w && s_pred[r0 + a] == st->tokens[r0 + 1 + a]) ++a;
    StepOut o;
    o.a = a;
    o.next = s_pred[r0 + a];
    o.R = R;
    o.pad = 0;
    for (int j = 0; j < kMaxRows; ++j) o.pred[j] = j <= w ? s_pred[r0 + j] : -1;
    *p.out = o;
    if (p.mirror != nullptr) {
      volatile int* m = reinterpret_cast<volatile int*>(p.mirror);
      for (int j = 0; j < kMaxRows; ++j) m[4 + j] = o.pred[j];
      m[0] = o.a;
      m[1] = o.next;
      m[2] = o.R;
      __threadfence_system();
    }
  }
}

}  // namespace ps
