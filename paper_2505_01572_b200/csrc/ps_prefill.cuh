// ps_prefill.cuh — NEXT-3 prefill ("The prefill phase processes the
// initial input prompt"; the prompt through the GEMMs at
// N = 64-256+ rows, the tensor-core-bound regime, plus a prefill attention).
//
// A decode forward has R <= 32 rows and streams every weight once per pass
// (HBM-bound, the megakernel of ps_mega.cuh).  A prompt chunk has up to
// kPfRows = 512 tokens, so each weight tile is reused 512 times: the GEMMs are
// bound by the tensor pipe, and the work runs as ordinary grid-wide kernels,
// one per step of the layer:
//
//   pf_norm_kernel     (embed +) RMSNorm: xs = split(x * rstd * g)
//   pf_gemm_kernel     persistent tcgen05 GEMM, TOKENS as the M = 128 side,
//                      128 or 256 weight rows as N, K in 64-wide TMA blocks;
//                      the split-bf16 operand (DESIGN R28) as two MMAs into
//                      ONE accumulator (x_hi W^T + x_lo W^T); two TMEM
//                      accumulators, so a tile's epilogue overlaps the next
//                      tile's mainloop; fused epilogues:
//                        PF_QKV    RoPE + paged split-bf16 KV append + fp32 q
//                        PF_RESID  residual add into x (O and down)
//                        PF_SWIGLU SiLU(gate) * up (gate and up rows stacked in
//                                  one N operand: one accumulator holds both)
//   pf_attn_kernel     causal GQA attention of the chunk's queries over the
//                      paged KV (prompt prefix + this chunk), mma.sync with
//                      split operands, online softmax in the exp2 domain
//
// The arithmetic is the oracle's forward (oracle/llama.py): x_{l+1/2} = x_l +
// Attn(RMSNorm(x_l)) Wo^T, x_{l+1} = x_{l+1/2} + (SiLU(h Wg^T) * (h Wu^T)) Wd^T,
// h = RMSNorm(x_{l+1/2}); only the order of the fp32 sums differs from the
// decode megakernel, so prompt KV written here is within rounding, not
// bit-identical, to KV written by decode forwards (ps_set_prefill_path
// selects the megakernel's 64-row bucket where bit-identity is wanted).
#pragma once
#include "ps_kernels.cuh"

namespace ps {

constexpr int kPfRows = 512;                     // tokens per prefill chunk (4 M tiles of 128)
constexpr int kPfThreads = 192;                  // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
constexpr int kPfTile = 128 * 64 * 2;            // one 128-row x 64-col bf16 TMA box (16 KB)

enum { PF_QKV = 0, PF_RESID = 1, PF_SWIGLU = 2 };

// Tile = 128 tokens x BN output features (BN = 128 or 256; SwiGLU: BN / 2 gate
// rows + BN / 2 up rows of the same features, stacked into one N = BN operand,
// BN = 128, 224 or 256).  Per stage: x_hi, x_lo (128 tokens x 64) and the
// BN-row weight block.
template <int BN> __host__ __device__ constexpr int pf_stages() { return BN > 128 ? 3 : 4; }
template <int BN> __host__ __device__ constexpr uint32_t pf_tmem_cols() { return BN > 128 ? 512 : 256; }
template <int BN> __host__ __device__ constexpr int pf_stage_bytes() { return 2 * kPfTile + BN * 128; }
template <int BN> __host__ __device__ constexpr int pf_smem_bytes() {
  return pf_stages<BN>() * pf_stage_bytes<BN>() + 1024 + 256;
}

struct PfGemmParams {
  CUtensorMap mX;                  // split-bf16 operand [2 kPfRows][K] (hi rows, then lo rows), box {64, 128}
  CUtensorMap mW0, mW1, mW2;       // weights [out][K], box {64, 128}: QKV q/k/v; SwiGLU gate/up; else mW0
  CUtensorMap mG64, mU64;          // SwiGLU with 128-wide tiles: gate / up, box {64, 64}
  CUtensorMap mG112, mU112;        // SwiGLU with 224-wide tiles: gate / up, box {64, 112}
  int K;                           // reduction length (multiple of 64)
  int N;                           // output features (QKV: all three; SwiGLU: d_ffn)
  int n_tiles, m_tiles;            // output tiles: BN-feature blocks x 128-token blocks
  int t1, t2;                      // QKV: BN-feature tiles [0, t1) q, [t1, t2) k, [t2, ..) v
  int nq, nk;                      // QKV: rows of Wq, of Wk (= Wv)
  int T;                           // valid tokens of the chunk
  int pos0;                        // absolute position of token 0
  // PF_QKV
  float* q; int ld_q;
  __nv_bfloat16* kv; const int32_t* page_table; int page_size, page_shift, layer, hkv, hd;
  long long page_stride;           // elements per KV page (all layers)
  const float2* rope_cs;           // [max_seq][hd/2] (cos, sin)
  // PF_RESID
  float* x; int ld_x;
  // PF_SWIGLU (split: hi rows [0, kPfRows), lo rows [kPfRows, 2 kPfRows))
  __nv_bfloat16* h; int ld_h;
};

PS_DEV void store_split8(__nv_bfloat16* hi, __nv_bfloat16* lo, const float* v) {
  uint32_t h4[4], l4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat16 a, b, c, d;
    split_bf16(v[2 * i], a, b);
    split_bf16(v[2 * i + 1], c, d);
    h4[i] = pack2(a, c);
    l4[i] = pack2(b, d);
  }
  *reinterpret_cast<uint4*>(hi) = make_uint4(h4[0], h4[1], h4[2], h4[3]);
  *reinterpret_cast<uint4*>(lo) = make_uint4(l4[0], l4[1], l4[2], l4[3]);
}

// Persistent: CTA b of G takes tiles b, b + G, ... (tile i = (token block
// i % m_tiles, feature block i / m_tiles): the token blocks sharing a weight
// block run side by side and re-read it from L2).  Warp 0 streams every
// tile's k-blocks through one ring; warp 1 issues the MMAs into two TMEM
// accumulators alternately, so the epilogue of tile j (warps 2-5) overlaps the
// mainloop of tile j + 1.
template <int MODE, int BN>
__global__ void __launch_bounds__(kPfThreads, 1) pf_gemm_kernel(const __grid_constant__ PfGemmParams p) {
  static_assert(BN == 128 || BN == 256 || (BN == 224 && MODE == PF_SWIGLU), "tile width");
  constexpr int kStages = pf_stages<BN>();
  constexpr int kSB = pf_stage_bytes<BN>();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kSB);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = p.K / 64;
  const int n_all = p.n_tiles * p.m_tiles;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 128); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<pf_tmem_cols<BN>()>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  // which weight matrix / local block a feature tile reads
  auto tile_kind = [&](int nt, int& kind, int& lt) {
    kind = 0;
    lt = nt;
    if (MODE == PF_QKV) {
      if (nt >= p.t2) { kind = 2; lt = nt - p.t2; }
      else if (nt >= p.t1) { kind = 1; lt = nt - p.t1; }
    }
  };
  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&p.mX);
      uint32_t it = 0;
      for (int i = blockIdx.x; i < n_all; i += gridDim.x) {
        const int m0 = (i % p.m_tiles) * 128, nt = i / p.m_tiles;
        int kind, lt;
        tile_kind(nt, kind, lt);
        const CUtensorMap* w0 = kind == 0 ? &p.mW0 : kind == 1 ? &p.mW1 : &p.mW2;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % kStages;
          mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
          uint8_t* st = smem + s * kSB;
          mbar_arrive_expect_tx(&full[s], kSB);
          tma_load_2d(st, &p.mX, &full[s], kb * 64, m0, kEvictLast);
          tma_load_2d(st + kPfTile, &p.mX, &full[s], kb * 64, kPfRows + m0, kEvictLast);
          if (MODE == PF_SWIGLU && BN == 256) {         // 128 gate rows, then 128 up rows
            tma_load_2d(st + 2 * kPfTile, &p.mW0, &full[s], kb * 64, lt * 128, kEvictNormal);
            tma_load_2d(st + 3 * kPfTile, &p.mW1, &full[s], kb * 64, lt * 128, kEvictNormal);
          } else if (MODE == PF_SWIGLU && BN == 224) {  // 112 gate rows, then 112 up rows
            tma_load_2d(st + 2 * kPfTile, &p.mG112, &full[s], kb * 64, lt * 112, kEvictNormal);
            tma_load_2d(st + 2 * kPfTile + 112 * 128, &p.mU112, &full[s], kb * 64, lt * 112, kEvictNormal);
          } else if (MODE == PF_SWIGLU) {               // 64 gate rows, then 64 up rows
            tma_load_2d(st + 2 * kPfTile, &p.mG64, &full[s], kb * 64, lt * 64, kEvictNormal);
            tma_load_2d(st + 2 * kPfTile + kPfTile / 2, &p.mU64, &full[s], kb * 64, lt * 64, kEvictNormal);
          } else {
#pragma unroll
            for (int h = 0; h < BN / 128; ++h)
              tma_load_2d(st + (2 + h) * kPfTile, w0, &full[s], kb * 64, lt * BN + h * 128, kEvictNormal);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t kI = idesc_bf16_f32<128, BN>();
      uint32_t it = 0, j = 0;
      for (int i = blockIdx.x; i < n_all; i += gridDim.x, ++j) {
        const int a = j & 1;
        mbar_wait(&tempty[a], ((j >> 1) & 1) ^ 1);      // the epilogue has drained this accumulator
        tc_fence_after();
        const uint32_t d = tmem + a * BN;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % kStages;
          mbar_wait(&full[s], (it / kStages) & 1);
          tc_fence_after();
          const uint32_t xh = smem_u32(smem + s * kSB), xl = xh + kPfTile, w = xh + 2 * kPfTile;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            // D[token][feature] += x_hi W^T, then += x_lo W^T (fixed order)
            mma_bf16(d, smem_desc_sw128(xh + 32 * k), smem_desc_sw128(w + 32 * k), kI, (kb > 0 || k > 0) ? 1u : 0u);
            mma_bf16(d, smem_desc_sw128(xl + 32 * k), smem_desc_sw128(w + 32 * k), kI, 1u);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[a]);
      }
    }
  } else {
    // ---- epilogue: warp w reads TMEM lanes [32 (w % 4), +32) = tokens m0 + that range
    const int quarter = warp & 3;
    uint32_t j = 0;
    for (int i = blockIdx.x; i < n_all; i += gridDim.x, ++j) {
      const int a = j & 1;
      const int m0 = (i % p.m_tiles) * 128, nt = i / p.m_tiles;
      int kind, lt;
      tile_kind(nt, kind, lt);
      const int tok = m0 + quarter * 32 + lane;
      const bool ok = tok < p.T;
      const uint32_t tq = tmem + ((uint32_t)(quarter * 32) << 16) + a * BN;
      mbar_wait(&tfull[a], (j >> 1) & 1);
      tc_fence_after();
      if (MODE == PF_RESID) {
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
          tmem_ld32(tq + c0, v);
          const int f0 = nt * BN + c0;
          if (ok && f0 < p.N) {
            float4* xr = reinterpret_cast<float4*>(p.x + (size_t)tok * p.ld_x + f0);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              float4 o = xr[q];
              o.x += v[4 * q]; o.y += v[4 * q + 1]; o.z += v[4 * q + 2]; o.w += v[4 * q + 3];
              xr[q] = o;
            }
          }
        }
      } else if (MODE == PF_SWIGLU) {
        constexpr int HB = BN / 2;                   // gate columns [0, HB), up columns [HB, BN)
        constexpr int CW = HB % 32 == 0 ? 32 : 16;   // columns per TMEM load
#pragma unroll 1
        for (int c0 = 0; c0 < HB; c0 += CW) {
          float g[CW], u[CW];
          if constexpr (CW == 32) {
            tmem_ld32(tq + c0, g);
            tmem_ld32(tq + HB + c0, u);
          } else {
            tmem_ld16(tq + c0, g);
            tmem_ld16(tq + HB + c0, u);
          }
          const int f0 = lt * HB + c0;
          if (ok && f0 < p.N) {
#pragma unroll
            for (int q = 0; q < CW; ++q) g[q] = g[q] / (1.0f + __expf(-g[q])) * u[q];
#pragma unroll
            for (int q = 0; q < CW / 8; ++q)
              store_split8(p.h + (size_t)tok * p.ld_h + f0 + 8 * q, p.h + (size_t)(kPfRows + tok) * p.ld_h + f0 + 8 * q,
                           g + 8 * q);
          }
        }
      } else {
        // QKV: the tile's BN features of kind q / k / v = BN / hd whole heads;
        // rotate-half RoPE pairs dims (j, j + hd/2) of a head: columns c and c + hd/2
        const int hd = p.hd, half = hd >> 1;
        const int nrows = kind == 0 ? p.nq : p.nk;
        const int pos = p.pos0 + tok;
#pragma unroll 1
        for (int h0 = 0; h0 < BN; h0 += hd) {
#pragma unroll 1
          for (int c = 0; c < half; c += 32) {
            float x0[32], x1[32];
            tmem_ld32(tq + h0 + c, x0);
            tmem_ld32(tq + h0 + half + c, x1);
            const int fa = lt * BN + h0 + c;          // feature of x0[0] within q / k / v
            // (no early exit: every lane of the warp must reach the next tcgen05.ld)
            if (ok && fa < nrows && kind < 2) {
              const float4* cs = reinterpret_cast<const float4*>(p.rope_cs + (size_t)pos * half + c);
#pragma unroll
              for (int q = 0; q < 16; ++q) {
                const float4 t = cs[q];            // (cos, sin) of dims c + 2q, c + 2q + 1
                const float a0 = x0[2 * q], b0 = x1[2 * q], a1 = x0[2 * q + 1], b1 = x1[2 * q + 1];
                x0[2 * q] = a0 * t.x - b0 * t.y;
                x1[2 * q] = b0 * t.x + a0 * t.y;
                x0[2 * q + 1] = a1 * t.z - b1 * t.w;
                x1[2 * q + 1] = b1 * t.z + a1 * t.w;
              }
            }
            if (!ok || fa >= nrows) {
            } else if (kind == 0) {
              float4* qa = reinterpret_cast<float4*>(p.q + (size_t)tok * p.ld_q + fa);
              float4* qb = reinterpret_cast<float4*>(p.q + (size_t)tok * p.ld_q + fa + half);
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                qa[q] = make_float4(x0[4 * q], x0[4 * q + 1], x0[4 * q + 2], x0[4 * q + 3]);
                qb[q] = make_float4(x1[4 * q], x1[4 * q + 1], x1[4 * q + 2], x1[4 * q + 3]);
              }
            } else {
              const int kh = fa / hd;
              const size_t plane = (size_t)p.hkv * p.page_size * hd;   // elements per (layer, plane)
              const size_t base = (size_t)p.page_table[pos >> p.page_shift] * p.page_stride +
                                  ((size_t)(p.layer * kKvPlanes + 2 * (kind - 1)) * p.hkv + kh) * p.page_size * hd +
                                  (size_t)(pos & (p.page_size - 1)) * hd + c;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                store_split8(p.kv + base + 8 * q, p.kv + base + plane + 8 * q, x0 + 8 * q);
                store_split8(p.kv + base + half + 8 * q, p.kv + base + plane + half + 8 * q, x1 + 8 * q);
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[a]);                       // this accumulator may be overwritten
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<pf_tmem_cols<BN>()>(tmem);
}

// ------------------------------------------------------------------ RMSNorm (+ embed)
// Row r: x = E[tok_r] (when tok != nullptr), then xs = split(x * rstd * g),
// rstd = 1 / sqrt(mean(x^2) + eps); sum of squares in a fixed block order.
constexpr int kPfNormThreads = 256;
__global__ void __launch_bounds__(kPfNormThreads) pf_norm_kernel(const int32_t* tok, const __nv_bfloat16* embed, int vocab,
                                                                 float* x, int d, const __nv_bfloat16* gain, float eps,
                                                                 __nv_bfloat16* xs) {
  __shared__ float red[kPfNormThreads / 32];
  const int r = blockIdx.x, t = threadIdx.x;
  float* xr = x + (size_t)r * d;
  if (tok != nullptr) {
    int id = tok[r];
    id = (id >= 0 && id < vocab) ? id : 0;
    const __nv_bfloat16* e = embed + (size_t)id * d;
    for (int c = t * 8; c < d; c += kPfNormThreads * 8) {
      const uint4 u = *reinterpret_cast<const uint4*>(e + c);
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
      float v[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(b[i]);
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
      }
      reinterpret_cast<float4*>(xr + c)[0] = make_float4(v[0], v[1], v[2], v[3]);
      reinterpret_cast<float4*>(xr + c)[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
    __syncthreads();
  }
  float sq = 0.f;
  for (int c = t * 8; c < d; c += kPfNormThreads * 8) {
    const float4 a = reinterpret_cast<const float4*>(xr + c)[0], b = reinterpret_cast<const float4*>(xr + c)[1];
    sq += a.x * a.x + a.y * a.y + a.z * a.z + a.w * a.w + b.x * b.x + b.y * b.y + b.z * b.z + b.w * b.w;
  }
  sq = warp_sum(sq);
  if ((t & 31) == 0) red[t >> 5] = sq;
  __syncthreads();
  float s = 0.f;
#pragma unroll
  for (int w = 0; w < kPfNormThreads / 32; ++w) s += red[w];
  const float rstd = rsqrtf(s / d + eps);
  for (int c = t * 8; c < d; c += kPfNormThreads * 8) {
    const float4 a = reinterpret_cast<const float4*>(xr + c)[0], b = reinterpret_cast<const float4*>(xr + c)[1];
    const uint4 gu = *reinterpret_cast<const uint4*>(gain + c);
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gu);
    const float xv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    float v[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 g = __bfloat1622float2(g2[i]);
      v[2 * i] = xv[2 * i] * rstd * g.x;
      v[2 * i + 1] = xv[2 * i + 1] * rstd * g.y;
    }
    store_split8(xs + (size_t)r * d + c, xs + (size_t)(kPfRows + r) * d + c, v);
  }
}

// ------------------------------------------------------------------ causal attention
// CTA = (query block qb, KV head kh): 64 query rows, row m = (token qb QB + m / g,
// head kh g + m % g), QB = 64 / g, so one K/V tile read serves the g heads that
// share it; warp w owns rows [16 w, 16 w + 16) (one m16 group, all hd dims).
// Keys [0, pos of the block's last token] in 32-key tiles (4 planes K_hi, K_lo,
// V_hi, V_lo) through a cp.async double buffer; S = Q K^T and O = P V on
// mma.sync m16n8k16 with split operands (q_hi k_hi + q_lo k_hi + q_hi k_lo, the
// lo*lo term ~2^-16 relative, dropped; likewise P V), causal mask, online
// softmax in the exp2 domain.  Output: split-bf16 att [2 kPfRows][H hd].
constexpr int kPfAttnKeys = 32;
struct PfAttnParams {
  const float* q; int ld_q;        // fp32 [kPfRows][H hd] (RoPE applied)
  const __nv_bfloat16* kv; const int32_t* page_table; int page_size, page_shift, layer, hkv, H;
  long long page_stride;
  float scale_log2;                // log2(e) / sqrt(hd)
  int T, pos0;
  __nv_bfloat16* out; int ld_out;  // split: hi rows [0, kPfRows), lo rows [kPfRows, 2 kPfRows)
};
template <int HD> __host__ __device__ constexpr int pf_attn_row_bytes() { return HD * 2 + 16; }   // padded rows
template <int HD> __host__ __device__ constexpr int pf_attn_smem_bytes() {
  return 2 * kKvPlanes * kPfAttnKeys * pf_attn_row_bytes<HD>();
}

template <int HD>
__global__ void __launch_bounds__(128) pf_attn_kernel(const __grid_constant__ PfAttnParams p) {
  constexpr int KS = HD / 16, NT = HD / 8, RB = pf_attn_row_bytes<HD>();
  constexpr int PLANE = kPfAttnKeys * RB, BUF = kKvPlanes * PLANE;
  extern __shared__ __align__(16) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int kh = blockIdx.y, g = p.H / p.hkv, QB = 64 / g;
  const int t_first = blockIdx.x * QB;                       // first token of this block
  const int t_last = min(p.T, t_first + QB) - 1;
  const int kend = p.pos0 + t_last + 1;                      // keys [0, kend)
  const int nkt = (kend + kPfAttnKeys - 1) / kPfAttnKeys;
  const size_t plane_el = (size_t)p.hkv * p.page_size * HD;
  auto load_tile = [&](int j, int buf) {   // keys [32 j, 32 j + 32): one page (page_size >= 64)
    const int k0 = j * kPfAttnKeys;
    const size_t base = (size_t)p.page_table[k0 >> p.page_shift] * p.page_stride +
                        ((size_t)p.layer * kKvPlanes * p.hkv + kh) * p.page_size * HD +
                        (size_t)(k0 & (p.page_size - 1)) * HD;
    constexpr int CPR = HD / 8;                               // 16-byte chunks per key row
    for (int i = tid; i < kKvPlanes * kPfAttnKeys * CPR; i += 128) {
      const int pl = i / (kPfAttnKeys * CPR), r = (i / CPR) % kPfAttnKeys, c = i % CPR;
      const __nv_bfloat16* src = p.kv + base + pl * plane_el + (size_t)r * HD + c * 8;
      const uint32_t dst = smem_u32(sm + buf * BUF + pl * PLANE + r * RB + c * 16);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  load_tile(0, 0);
  // query fragments (A operand, rows lane/4 and lane/4 + 8 of this warp's 16)
  uint32_t qh[KS][4], ql[KS][4];
  int qpos[2];
  {
    int qoff[2];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int m = warp * 16 + (lane >> 2) + hr * 8;
      const int t = t_first + m / g, h = kh * g + m % g;
      qoff[hr] = t <= t_last ? t * p.ld_q + h * HD : -1;
      qpos[hr] = p.pos0 + min(t, t_last);
    }
#pragma unroll
    for (int kk = 0; kk < KS; ++kk)
#pragma unroll
      for (int jq = 0; jq < 4; ++jq) {
        const int o = qoff[jq & 1];
        const int d = kk * 16 + (lane & 3) * 2 + (jq >> 1) * 8;
        const float2 qv = o >= 0 ? *reinterpret_cast<const float2*>(p.q + o + d) : make_float2(0.f, 0.f);
        split_pack(qv.x * p.scale_log2, qv.y * p.scale_log2, qh[kk][jq], ql[kk][jq]);
      }
  }
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  float oacc[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) oacc[n][0] = oacc[n][1] = oacc[n][2] = oacc[n][3] = 0.f;
  // per-lane ldmatrix offsets: K non-transposed (keys x dims), V transposed
  const uint32_t koff = ((lane & 7) + ((lane >> 4) << 3)) * RB + ((lane >> 3) & 1) * 16;
  const uint32_t voff = ((lane & 7) + ((lane >> 3) & 1) * 8) * RB + (lane >> 4) * 16;
  for (int j = 0; j < nkt; ++j) {
    if (j + 1 < nkt) {
      load_tile(j + 1, (j + 1) & 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const uint32_t sb = smem_u32(sm + (j & 1) * BUF);
    // ---- S = Q K^T over 32 keys (4 n-tiles of 8)
    float s[4][4];
#pragma unroll
    for (int n = 0; n < 4; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int kp = 0; kp < 2; ++kp) {                          // key pairs of n-tiles (16 keys)
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        uint32_t b0, b1, b2, b3, c0, c1, c2, c3;
        const uint32_t a = sb + kp * 16 * RB + koff + kk * 32;
        ldsm_x4(a, b0, b1, b2, b3);                           // K_hi
        ldsm_x4(a + PLANE, c0, c1, c2, c3);                   // K_lo
        mma16816(s[2 * kp], qh[kk], b0, b1);
        mma16816(s[2 * kp + 1], qh[kk], b2, b3);
        mma16816(s[2 * kp], ql[kk], b0, b1);
        mma16816(s[2 * kp + 1], ql[kk], b2, b3);
        mma16816(s[2 * kp], qh[kk], c0, c1);
        mma16816(s[2 * kp + 1], qh[kk], c2, c3);
      }
    }
    // ---- causal mask, online softmax
    const int k0 = j * kPfAttnKeys;
    float scale[2];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      float mx = -INFINITY;
#pragma unroll
      for (int n = 0; n < 4; ++n)
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2) {
          const int key = k0 + n * 8 + (lane & 3) * 2 + e2;
          float& sv = s[n][hr * 2 + e2];
          if (key > qpos[hr]) sv = -INFINITY;
          mx = fmaxf(mx, sv);
        }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float mn = fmaxf(mrow[hr], mx);
      scale[hr] = (mrow[hr] == -INFINITY) ? 0.f : exp2f(mrow[hr] - mn);
      mrow[hr] = mn;
    }
    float lsum[2] = {0.f, 0.f};
    uint32_t pah[2][4], pal[2][4];                            // P (16 rows x 32 keys) as two k16 A fragments
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      float pv[4];
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const int hr = q4 >> 1;
        pv[q4] = (mrow[hr] == -INFINITY) ? 0.f : exp2f(s[n][q4] - mrow[hr]);
        lsum[hr] += pv[q4];
      }
      split_pack(pv[0], pv[1], pah[n >> 1][(n & 1) * 2 + 0], pal[n >> 1][(n & 1) * 2 + 0]);
      split_pack(pv[2], pv[3], pah[n >> 1][(n & 1) * 2 + 1], pal[n >> 1][(n & 1) * 2 + 1]);
    }
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      lsum[hr] += __shfl_xor_sync(0xffffffffu, lsum[hr], 1);
      lsum[hr] += __shfl_xor_sync(0xffffffffu, lsum[hr], 2);
      lrow[hr] = lrow[hr] * scale[hr] + lsum[hr];
    }
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      oacc[n][0] *= scale[0]; oacc[n][1] *= scale[0];
      oacc[n][2] *= scale[1]; oacc[n][3] *= scale[1];
    }
    // ---- O += P V (two 16-key steps, NT/2 pairs of 8-dim n-tiles)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
      for (int np = 0; np < NT / 2; ++np) {
        uint32_t v0, v1, v2, v3, w0, w1, w2, w3;
        const uint32_t a = sb + 2 * PLANE + ks * 16 * RB + voff + np * 32;
        ldsm_x4_t(a, v0, v1, v2, v3);                         // V_hi
        ldsm_x4_t(a + PLANE, w0, w1, w2, w3);                 // V_lo
        mma16816(oacc[2 * np], pah[ks], v0, v1);
        mma16816(oacc[2 * np + 1], pah[ks], v2, v3);
        mma16816(oacc[2 * np], pal[ks], v0, v1);
        mma16816(oacc[2 * np + 1], pal[ks], v2, v3);
        mma16816(oacc[2 * np], pah[ks], w0, w1);
        mma16816(oacc[2 * np + 1], pah[ks], w2, w3);
      }
    }
    __syncthreads();                                          // buffer j & 1 is refilled next iteration
  }
  // ---- O / l -> split-bf16 output rows
#pragma unroll
  for (int hr = 0; hr < 2; ++hr) {
    const int m = warp * 16 + (lane >> 2) + hr * 8;
    const int t = t_first + m / g, h = kh * g + m % g;
    if (t > t_last) continue;
    const float inv = 1.0f / lrow[hr];
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int d = n * 8 + (lane & 3) * 2;
      __nv_bfloat16 h0, l0, h1, l1;
      split_bf16(oacc[n][hr * 2] * inv, h0, l0);
      split_bf16(oacc[n][hr * 2 + 1] * inv, h1, l1);
      *reinterpret_cast<uint32_t*>(p.out + (size_t)t * p.ld_out + h * HD + d) = pack2(h0, h1);
      *reinterpret_cast<uint32_t*>(p.out + (size_t)(kPfRows + t) * p.ld_out + h * HD + d) = pack2(l0, l1);
    }
  }
}

}  // namespace ps
