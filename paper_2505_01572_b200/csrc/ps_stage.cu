// ps_stage.cu — host side of the verify hot path: stage state (token buffer O_i,
// paged-KV page table and free list), TMA descriptors over the borrowed
// weights, the megakernel's phase tables (one persistent launch per forward)
// and the C ABI of include/pipespec.h.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/pipespec.h"
#include "ps_host.cuh"
#include "ps_prefill.cuh"

// ============================================================================ errors
static thread_local std::string g_err;
std::atomic<long long> g_launches{0};

ps_status fail(ps_status code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

// ============================================================================ stage
struct LayerMaps {
  CUtensorMap q, k, v, o, g, u, d;
};

struct ps_stage {
  ps_model_shape sh{};
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int max_seq = 0, max_window = 0, page_size = 0;
  // weights (borrowed)
  const __nv_bfloat16* embed = nullptr;
  const __nv_bfloat16* lm_head = nullptr;
  const __nv_bfloat16* final_norm = nullptr;
  std::vector<const __nv_bfloat16*> lw;   // [L][9]
  std::vector<LayerMaps> maps;
  CUtensorMap map_lm;
  CUtensorMap map_kv;      // the KV pool as [rows][hd] bf16 rows (attention TMA, box 16 rows)
  CUtensorMap map_xg[3], map_att[3], map_h[3];   // per rows bucket (16, 32, 64)
  // KV pool (borrowed) + paging
  __nv_bfloat16* kv = nullptr;
  long long page_elems = 0;
  int pages_total = 0;
  std::vector<int> page_of;     // logical page -> physical (-1 unmapped)
  std::vector<int> free_pages;  // stack
  int n_mapped = 0;             // logical pages [0, n_mapped) are mapped
  int32_t* d_page_table = nullptr;
  int32_t* h_page_table = nullptr;   // pinned mirror
  // scratch (owned)
  StepIn* d_in = nullptr;
  StepIn* h_in = nullptr;            // pinned staging ring [kInSlots]; host writes slot `in_slot`
  cudaEvent_t in_ev[8] = {};         // recorded after each slot's H2D copy
  int in_slot = 0;
  int last_bucket = 0;
  cudaEvent_t fwd_ev[2] = {nullptr, nullptr};   // around the last head forward's kernels
  double last_fwd_ms = 0, sum_fwd_ms = 0;
  long long n_fwd = 0;
  // megakernel: phase tables per (bucket, with_head), device tensor maps, counters
  MegaPhase* mega_ph[6] = {};          // per (rows bucket, with lm_head)
  CUtensorMap* mega_maps[6] = {};
  int mega_n[6] = {};
  unsigned* mega_done = nullptr;
  unsigned long long* mega_dbg = nullptr;   // PS_TRACE builds only: timeline stamps
  unsigned long long* epi_dbg = nullptr;
  unsigned long long* attn_dbg = nullptr;
  unsigned gen = 0, gen_head = 0;
  int n_ctas = 0;                    // megakernel grid (persistent CTAs, <= #SMs)
  // tensor parallelism (a14): this rank's exchange buffer = [phase counters |
  // partial [2][kRowsCap][d] fp32 | argmax keys [2][kMaxRows] u64]; peers[q] is
  // rank q's buffer as mapped in this process (peer memory for q != tp_rank)
  int tp_rank = 0, tp_size = 1;
  int vocab_full = 0, vocab_off = 0;
  uint8_t* xch = nullptr;
  size_t off_part = 0, off_keys = 0, xch_bytes = 0;
  uint8_t* peers[8] = {};
  bool peer_ipc[8] = {};
  bool tp_connected = false;
  size_t ws_bytes = 0;
  long long ws_chunk = 0;            // floats per 16-row chunk region of the stream-K workspace
  int cnt_chunk = 0;
  // asynchronous verify (ps_verify_async / ps_verify_wait)
  bool inflight = false;
  long long if_n = 0;                // len(O_i) when the pass was enqueued
  int if_w = 0;
  cudaEvent_t done_ev = nullptr;     // recorded after the in-flight pass
  StepOut* d_out = nullptr;
  StepOut* h_out = nullptr;          // mapped pinned mirror
  StepOut* h_out_dev = nullptr;      // its device alias
  float *x = nullptr, *q = nullptr, *ss = nullptr, *logits = nullptr, *ws = nullptr;
  __nv_bfloat16 *xg = nullptr, *att = nullptr, *h = nullptr;
  unsigned long long* amax = nullptr;
  unsigned *counters = nullptr, *attn_counters = nullptr;
  float *attn_o = nullptr, *attn_ml = nullptr;
  float2* rope_cs = nullptr;
  SynthParams* d_syn = nullptr;
  SynthParams h_syn{};
  int32_t* d_S = nullptr;
  int n_prompt = 0;
  int ss_ld = 0, xg_ld = 0, max_chunks = 0, max_rb = 0, attn_grid = 0, attn_sc = 1;
  GemmShape gs_qkv, gs_o, gs_gu, gs_d, gs_lm;
  int lm_tiles = 0;
  // token buffer O_i
  std::vector<int32_t> tokens;
  long long kv_len = 0;
  int onpath = 0;                    // generated tokens matching the synthetic target S
  std::vector<int32_t> S_host;
  // NEXT-3 prefill kernels (ps_prefill.cuh; single-GPU stages): chunk buffers
  // of kPfRows tokens and the per-layer GEMM parameter templates
  int prefill_path = PS_PREFILL_AUTO;
  bool pf_ready = false;
  float *pf_x = nullptr, *pf_q = nullptr;
  __nv_bfloat16 *pf_xs = nullptr, *pf_att = nullptr, *pf_h = nullptr;
  int32_t* pf_tok = nullptr;            // device tokens of the chunk
  int32_t* h_pf_tok = nullptr;          // pinned staging
  cudaEvent_t pf_tok_ev = nullptr;      // the staging buffer's previous copy ran
  std::vector<PfGemmParams> pf_gemm;    // [L][4]: QKV, O, gate/up, down
  double sum_prefill_ms = 0;
  // chained draft forwards (ps_draft): device tokens + pinned copy, timing events
  int32_t* d_chain = nullptr;
  int32_t* h_chain = nullptr;
  cudaEvent_t chain_ev[2] = {nullptr, nullptr};
};

// rows buckets: 16 and 32 (forwards with the lm_head: verify / draft), 64 (prefill chunks)
static int bucket_rp(int b) { return b == 0 ? 16 : b == 1 ? 32 : 64; }

// Device-wide setup of a stage's device: the shared GEMM/attention attributes
// plus the megakernel instantiations (per device, so every GPU of a process).
static ps_status init_stage_device(int device) {
  ps_status st;
  if ((st = init_device_globals(device)) != PS_OK) return st;
  CU_TRY(cudaFuncSetAttribute(mega_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, MegaSmem<16>::kBytes));
  CU_TRY(cudaFuncSetAttribute(mega_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, MegaSmem<32>::kBytes));
  CU_TRY(cudaFuncSetAttribute(mega_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, MegaSmem<64>::kBytes));
  CU_TRY(cudaFuncSetAttribute(mega_kernel<16, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, MegaSmem<16, 6>::kBytes));
  CU_TRY(cudaFuncSetAttribute(pf_gemm_kernel<PF_QKV, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              pf_smem_bytes<128>()));
  CU_TRY(cudaFuncSetAttribute(pf_gemm_kernel<PF_QKV, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              pf_smem_bytes<256>()));
  CU_TRY(cudaFuncSetAttribute(pf_gemm_kernel<PF_RESID, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              pf_smem_bytes<128>()));
  CU_TRY(cudaFuncSetAttribute(pf_gemm_kernel<PF_RESID, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              pf_smem_bytes<256>()));
  CU_TRY(cudaFuncSetAttribute(pf_gemm_kernel<PF_SWIGLU, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              pf_smem_bytes<256>()));
  CU_TRY(cudaFuncSetAttribute(pf_gemm_kernel<PF_SWIGLU, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              pf_smem_bytes<128>()));
  CU_TRY(cudaFuncSetAttribute(pf_gemm_kernel<PF_SWIGLU, 224>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              pf_smem_bytes<224>()));
  CU_TRY(cudaFuncSetAttribute(pf_attn_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, pf_attn_smem_bytes<64>()));
  CU_TRY(cudaFuncSetAttribute(pf_attn_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, pf_attn_smem_bytes<128>()));
  return PS_OK;
}
static int bucket_of(int R) { return R <= 16 ? 0 : R <= 32 ? 1 : 2; }

// Calls that change or use the stage are refused while an asynchronous pass
// is in flight (ps_verify_async ... ps_verify_wait).
#define PS_NOT_INFLIGHT(S) \
  if ((S)->inflight) return fail(PS_E_INVALID, "a ps_verify_async pass is in flight (call ps_verify_wait)")

extern "C" int64_t ps_kv_pool_bytes_tp(const ps_model_shape* s, int32_t max_seq, int32_t page_size, int32_t tp) {
  if (!s || page_size <= 0 || tp < 1 || s->n_kv_heads % tp) return -1;
  long long pages = (max_seq + page_size - 1) / page_size;
  // K_hi, K_lo, V_hi, V_lo planes (split-bf16 KV cache, ps_kernels.cuh)
  long long page_elems = (long long)s->n_layers * kKvPlanes * (s->n_kv_heads / tp) * page_size * s->head_dim;
  return pages * page_elems * 2;
}
extern "C" int64_t ps_kv_pool_bytes(const ps_model_shape* s, int32_t max_seq, int32_t page_size) {
  return ps_kv_pool_bytes_tp(s, max_seq, page_size, 1);
}

static void rope_table(const ps_model_shape& s, int max_seq, std::vector<float2>& out) {
  const int hd = s.head_dim, half = hd / 2;
  std::vector<double> inv(half);
  for (int i = 0; i < half; ++i) inv[i] = 1.0 / std::pow((double)s.rope_theta, (2.0 * i) / hd);
  if (s.rope_kind == 1) {   // llama3 frequency scaling (HF convention, reading R19)
    const double factor = s.rope_factor, lo = s.lo_ff, hi = s.hi_ff, old = s.rope_orig_max;
    const double low_wl = old / lo, high_wl = old / hi;
    for (int i = 0; i < half; ++i) {
      const double wl = 2.0 * M_PI / inv[i];
      double f = wl > low_wl ? inv[i] / factor : inv[i];
      if (wl >= high_wl && wl <= low_wl) {
        const double sm = (old / wl - lo) / (hi - lo);
        f = (1.0 - sm) * f / factor + sm * f;
      }
      inv[i] = f;
    }
  }
  out.resize((size_t)max_seq * half);
  for (int p = 0; p < max_seq; ++p)
    for (int i = 0; i < half; ++i) {
      const double a = (double)p * inv[i];
      out[(size_t)p * half + i] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
}

// ---------------------------------------------------------------- forward
// phases per forward: embed + L x {QKV, attn, combine, O, [TPRED], gate/up, down, [TPRED]} + lm_head + argmax
static int kMaxPhases(int L) { return 8 * L + 8; }
enum { K_EMBED = 0, K_QKV, K_ATTN, K_O, K_GU, K_DOWN, K_LMHEAD, K_ARGMAX };

// Host-side TMA maps of one GEMM step: A0..A2 (weights) and X (activations).
struct HostMaps {
  const CUtensorMap *a0 = nullptr, *a1 = nullptr, *a2 = nullptr, *x = nullptr;
};

// Parameters of one step of the forward (rows bucket b, layer l) -- shared by
// the megakernel phase table.
static void build_phase(ps_stage* S, int b, int kind, int l, MegaPhase& P, HostMaps& hm) {
  const ps_model_shape& sh = S->sh;
  const int d = sh.d_model, hq = sh.n_heads * sh.head_dim, hkv = sh.n_kv_heads * sh.head_dim;
  const float inv_d = 1.0f / d;
  const int ss_n = (d + 127) / 128;
  const __nv_bfloat16* const* W = sh.n_layers ? &S->lw[(size_t)l * 9] : nullptr;
  memset(&P, 0, sizeof P);
  GemmParams& p = P.g;
  p.step = S->d_in;
  p.ws = S->ws;
  p.counters = S->counters;
  p.ws_chunk = S->ws_chunk;
  p.cnt_chunk = S->cnt_chunk;
  p.ll = 1;
  p.ll_tag = 1 + kind + 8 * l;     // per-kernel path; the megakernel re-tags by phase index
  switch (kind) {
    case K_EMBED: {
      P.kind = PH_EMBED;
      P.em = EmbedParams{S->d_in, S->embed, d, S->vocab_full, sh.n_layers ? S->lw[PS_N_ATTN] : S->final_norm,
                         S->x, d, S->xg, S->xg_ld, S->ss, S->ss_ld};
      return;
    }
    case K_QKV: {   // QKV + RoPE + paged KV append (a4, a5)
      const LayerMaps& M = S->maps[l];
      P.kind = PH_GEMM;
      p.ss_in = S->ss; p.ss_n = ss_n; p.ss_ld = S->ss_ld; p.inv_d = inv_d; p.eps = sh.rms_eps;
      p.mode = EPI_QKV;
      p.N = hq + 2 * hkv;
      p.n_tiles = S->gs_qkv.n_tiles; p.kb_total = S->gs_qkv.kb_total; p.maxseg = S->gs_qkv.maxseg; p.grid = S->gs_qkv.grid;
      p.t1 = (hq + 127) / 128; p.t2 = p.t1 + (hkv + 127) / 128;
      p.nq = hq; p.nk = hkv;
      p.q = S->q; p.ld_q = hq;
      p.kv = S->kv; p.page_table = S->d_page_table; p.page_size = S->page_size; p.layer = l;
      p.hkv = sh.n_kv_heads; p.hd = sh.head_dim; p.page_stride = S->page_elems; p.rope_cs = S->rope_cs;
      hm = HostMaps{&M.q, &M.k, &M.v, &S->map_xg[b]};
      return;
    }
    case K_ATTN: {  // split-KV decode attention (a6)
      P.kind = PH_ATTN;
      AttnParams& a = P.a;
      a.step = S->d_in; a.q = S->q; a.ld_q = hq; a.page_table = S->d_page_table;
      a.page_size = S->page_size; a.page_shift = __builtin_ctz((unsigned)S->page_size);
      a.rows_per_page = S->page_elems / sh.head_dim; a.layer = l; a.hkv = sh.n_kv_heads;
      a.H = sh.n_heads; a.hd = sh.head_dim; a.scale_log2 = 1.4426950408889634f / std::sqrt((float)sh.head_dim);
      a.max_chunks = S->max_chunks; a.rows_cap = S->max_rb * kAttnRB; a.sc = S->attn_sc;
      a.ws_o = S->attn_o; a.ws_ml = S->attn_ml;
      a.out = S->att; a.ld_out = hq;
      a.dbg = S->attn_dbg;   // PS_TRACE builds only (null otherwise)
      hm = HostMaps{&S->map_kv, &S->map_kv, &S->map_kv, &S->map_kv};
      return;
    }
    case K_O: {     // O projection + residual; writes x∘g_mlp and sumsq (a7)
      const LayerMaps& M = S->maps[l];
      P.kind = PH_GEMM;
      p.mode = EPI_RESID; p.N = d;
      p.n_tiles = S->gs_o.n_tiles; p.kb_total = S->gs_o.kb_total; p.maxseg = S->gs_o.maxseg; p.grid = S->gs_o.grid;
      p.x = S->x; p.ld_x = d; p.xg = S->xg; p.ld_xg = S->xg_ld; p.gain = W[PS_N_MLP];
      p.ss_out = S->ss; p.ss_out_ld = S->ss_ld;
      if (S->tp_size > 1) {   // row-parallel: partial -> exchange slot 0, reduced by the TPRED phase
        p.mode = EPI_STORE;
        p.out = (float*)(S->xch + S->off_part); p.ld_out = d;
      }
      hm = HostMaps{&M.o, &M.o, &M.o, &S->map_att[b]};
      return;
    }
    case K_GU: {    // gate/up + SiLU*mul (a8)
      const LayerMaps& M = S->maps[l];
      P.kind = PH_GEMM;
      P.gu = 1;
      p.mode = EPI_SWIGLU; p.N = sh.d_ffn;
      p.n_tiles = S->gs_gu.n_tiles; p.kb_total = S->gs_gu.kb_total; p.maxseg = S->gs_gu.maxseg; p.grid = S->gs_gu.grid;
      p.ss_in = S->ss; p.ss_n = ss_n; p.ss_ld = S->ss_ld; p.inv_d = inv_d; p.eps = sh.rms_eps;
      p.h = S->h; p.ld_h = sh.d_ffn;
      hm = HostMaps{&M.g, &M.u, &M.u, &S->map_xg[b]};
      return;
    }
    case K_DOWN: {  // down + residual; writes x∘g_next and sumsq (a9)
      const LayerMaps& M = S->maps[l];
      P.kind = PH_GEMM;
      p.mode = EPI_RESID; p.N = d;
      p.n_tiles = S->gs_d.n_tiles; p.kb_total = S->gs_d.kb_total; p.maxseg = S->gs_d.maxseg; p.grid = S->gs_d.grid;
      p.x = S->x; p.ld_x = d; p.xg = S->xg; p.ld_xg = S->xg_ld;
      p.gain = (l + 1 < sh.n_layers) ? S->lw[(size_t)(l + 1) * 9 + PS_N_ATTN] : S->final_norm;
      p.ss_out = S->ss; p.ss_out_ld = S->ss_ld;
      if (S->tp_size > 1) {   // row-parallel: partial -> exchange slot 1
        p.mode = EPI_STORE;
        p.out = (float*)(S->xch + S->off_part) + (size_t)kRowsCap * d; p.ld_out = d;
      }
      hm = HostMaps{&M.d, &M.d, &M.d, &S->map_h[b]};
      return;
    }
    case K_LMHEAD: {  // final norm + lm_head + argmax partials (a10)
      P.kind = PH_GEMM;
      p.mode = EPI_LMHEAD; p.N = sh.vocab;
      p.n_tiles = S->gs_lm.n_tiles; p.kb_total = S->gs_lm.kb_total; p.maxseg = S->gs_lm.maxseg; p.grid = S->gs_lm.grid;
      p.ss_in = S->ss; p.ss_n = ss_n; p.ss_ld = S->ss_ld; p.inv_d = inv_d; p.eps = sh.rms_eps;
      p.logits = S->logits; p.ld_logits = sh.vocab; p.amax = S->amax; p.amax_ld = S->lm_tiles;
      if (S->tp_size > 1) {   // vocab-parallel: global ids, per-rank keys in the exchange buffer
        p.vocab_off = S->vocab_off;
        p.amax = (unsigned long long*)(S->xch + S->off_keys);
        p.amax_par = 1;
      }
      hm = HostMaps{&S->map_lm, &S->map_lm, &S->map_lm, &S->map_xg[b]};
      return;
    }
    case K_ARGMAX: {  // argmax + compare + first-mismatch scan (a11)
      P.kind = PH_ARGMAX;
      P.am = ArgmaxParams{S->d_in, S->amax, S->lm_tiles, S->lm_tiles, S->d_out, S->h_out_dev, S->d_syn, S->vocab_full,
                          0, {}};
      if (S->tp_size > 1) {
        P.am.amax = (unsigned long long*)(S->xch + S->off_keys);
        P.am.tp_n = S->tp_size;
        for (int q = 0; q < S->tp_size; ++q)
          P.am.tp_keys[q] = (const unsigned long long*)(S->peers[q] + S->off_keys);
      }
      return;
    }
  }
}

// ---------------------------------------------------------------- megakernel
// Phase table of one forward (bucket b; with_head adds LM_HEAD + ARGMAX), with
// tensor maps copied to device memory.
static ps_status build_mega(ps_stage* S, int b, bool with_head) {
  const int L = S->sh.n_layers;
  std::vector<MegaPhase> ph;
  std::vector<CUtensorMap> maps;
  auto add = [&](int kind, int l) {
    MegaPhase P;
    HostMaps hm;
    build_phase(S, b, kind, l, P, hm);
    if (P.kind == PH_ATTN) {   // the KV map; index patched to a pointer below
      P.a.kvmap = reinterpret_cast<const CUtensorMap*>(maps.size() + 1);
      maps.push_back(*hm.a0);
    }
    if (P.kind == PH_GEMM) {   // device map indices, patched to pointers below
      const size_t base = maps.size();
      maps.push_back(*hm.a0);
      maps.push_back(*hm.a1);
      maps.push_back(*hm.a2);
      maps.push_back(*hm.x);
      P.mA0 = reinterpret_cast<const CUtensorMap*>(base + 1);   // 1-based index
    }
    ph.push_back(P);
  };
  const bool tp = S->tp_size > 1;
  auto add_tpred = [&](int l, bool after_down) {   // all-reduce + residual + next norm operand (a14)
    ph.back().xpub = 1;
    const ps_model_shape& sh = S->sh;
    MegaPhase P;
    memset(&P, 0, sizeof P);
    P.kind = PH_TPRED;
    P.xwait = 1;
    TpParams& t = P.tp;
    t.n = S->tp_size;
    for (int q = 0; q < S->tp_size; ++q)
      t.part[q] = (const float*)(S->peers[q] + S->off_part) + (after_down ? (size_t)kRowsCap * sh.d_model : 0);
    t.x = S->x; t.ld_x = sh.d_model; t.xg = S->xg; t.ld_xg = S->xg_ld;
    t.gain = !after_down ? S->lw[(size_t)l * 9 + PS_N_MLP]
                         : (l + 1 < sh.n_layers ? S->lw[(size_t)(l + 1) * 9 + PS_N_ATTN] : S->final_norm);
    t.ss_out = S->ss; t.ss_out_ld = S->ss_ld; t.d = sh.d_model;
    ph.push_back(P);
  };
  add(K_EMBED, 0);
  for (int l = 0; l < L; ++l)
    for (int kind = K_QKV; kind <= K_DOWN; ++kind) {
      add(kind, l);
      if (kind == K_ATTN) {
        // chunk partials, then a separate combine phase (measured round 1: the
        // last-arriving CTA combining inline costs +6% on the 8B R=5 pass)
        ph.push_back(ph.back());
        ph.back().kind = PH_ACOMB;
      }
      if (tp && (kind == K_O || kind == K_DOWN)) add_tpred(l, kind == K_DOWN);
    }
  if (with_head) {
    add(K_LMHEAD, 0);
    ph.back().head = 1;
    ph.back().xpub = tp ? 1 : 0;
    add(K_ARGMAX, 0);
    ph.back().head = 1;
    ph.back().xwait = tp ? 1 : 0;
  }
  if ((int)ph.size() > kMaxPhases(L)) return fail(PS_E_INVALID, "phase table overflow");
  // LL stream-K flag tag: the phase index (< 1024)
  for (size_t i = 0; i < ph.size(); ++i)
    if (ph[i].kind == PH_GEMM) ph[i].g.ll_tag = 1 + (int)i;
  const int key = b * 2 + (with_head ? 1 : 0);
  if (S->mega_maps[key]) cudaFree(S->mega_maps[key]);
  if (S->mega_ph[key]) cudaFree(S->mega_ph[key]);
  CU_TRY(cudaMalloc(&S->mega_maps[key], std::max<size_t>(1, maps.size()) * sizeof(CUtensorMap)));
  CU_TRY(cudaMemcpy(S->mega_maps[key], maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  if (S->epi_dbg)   // PS_TRACE builds: per-phase stream-K fixup stamps [phase][cta][4]
    for (size_t i = 0; i < ph.size(); ++i) ph[i].g.dbg = S->epi_dbg + i * g_num_sms * 4;
  const CUtensorMap* dm = S->mega_maps[key];
  for (auto& P : ph) {
    if (P.kind == PH_ATTN) P.a.kvmap = dm + (reinterpret_cast<size_t>(P.a.kvmap) - 1);
    if (P.kind != PH_GEMM) continue;
    const size_t base = reinterpret_cast<size_t>(P.mA0) - 1;
    P.mA0 = dm + base;
    P.mA1 = dm + base + 1;
    P.mA2 = dm + base + 2;
    P.mX = dm + base + 3;
  }
  CU_TRY(cudaMalloc(&S->mega_ph[key], ph.size() * sizeof(MegaPhase)));
  CU_TRY(cudaMemcpy(S->mega_ph[key], ph.data(), ph.size() * sizeof(MegaPhase), cudaMemcpyHostToDevice));
  S->mega_n[key] = (int)ph.size();
  return PS_OK;
}

static ps_status launch_mega(ps_stage* S, int b, bool with_head) {
  const int key = b * 2 + (with_head ? 1 : 0);
  // (tables are built at create / connect time: a build here would allocate
  // after the forward's generation counters were prepared)
  if (!S->mega_ph[key]) return fail(PS_E_INVALID, "megakernel phase table %d missing", key);
  MegaParams mp{S->mega_ph[key], S->mega_n[key], S->d_in, S->mega_done, S->mega_dbg, S->tp_size, {}, S->d_chain};
  for (int q = 0; q < S->tp_size; ++q) mp.peer_done[q] = (const unsigned*)S->peers[q];
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(S->n_ctas);
  cfg.blockDim = dim3(kMegaThreads);
  cfg.stream = S->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  // A cooperative launch guarantees co-residency of the whole grid, but the
  // driver does not start a second cooperative kernel while one is running:
  // ranks of a tensor-parallel group sharing one GPU (max_ctas partitions)
  // would wait on each other forever.  A partial grid (one 200+ KB CTA per
  // SM, at most the free SMs) is launched as a plain kernel instead.
  cfg.numAttrs = S->n_ctas == g_num_sms ? 1 : 0;
  cudaError_t e;
  if (b == 0 && S->sh.d_model <= 2048) {
    // Small models: a 6-slot ring.  A deeper ring runs further ahead across
    // phase boundaries but queues the boundary's latency-critical loads
    // (stream-K partials, X tiles, attention) behind more weight bytes, and
    // the short phases of a small model lose more to that than they gain
    // (measured: 1B draft step 0.943 ms with 6 slots vs 0.958 with 8; the 8B
    // verify pass prefers 8: 3.597 vs 3.638 ms).
    cfg.dynamicSmemBytes = MegaSmem<16, 6>::kBytes;
    e = cudaLaunchKernelEx(&cfg, mega_kernel<16, 6>, mp);
  } else if (b == 0) {
    cfg.dynamicSmemBytes = MegaSmem<16>::kBytes;
    e = cudaLaunchKernelEx(&cfg, mega_kernel<16>, mp);
  } else if (b == 1) {
    cfg.dynamicSmemBytes = MegaSmem<32>::kBytes;
    e = cudaLaunchKernelEx(&cfg, mega_kernel<32>, mp);
  } else {
    cfg.dynamicSmemBytes = MegaSmem<64>::kBytes;
    e = cudaLaunchKernelEx(&cfg, mega_kernel<64>, mp);
  }
  if (e != cudaSuccess) return fail(PS_E_CUDA, "megakernel launch: %s", cudaGetErrorString(e));
  g_launches++;
  return PS_OK;
}

// ---------------------------------------------------------------- paging
// Mapped logical pages always form a prefix [0, n_mapped) of the page table:
// ensure_pages extends it, free_pages_from cuts it.
static ps_status ensure_pages(ps_stage* S, long long last_pos) {
  const int need = (int)(last_pos / S->page_size) + 1;
  if (need > (int)S->page_of.size()) return fail(PS_E_CAPACITY, "position %lld beyond max_seq", last_pos);
  if (need <= S->n_mapped) return PS_OK;
  if ((int)S->free_pages.size() < need - S->n_mapped) return fail(PS_E_CAPACITY, "KV pool exhausted");
  const int lo = S->n_mapped;
  for (int lp = lo; lp < need; ++lp) {
    S->page_of[lp] = S->free_pages.back();
    S->free_pages.pop_back();
    S->h_page_table[lp] = S->page_of[lp];
  }
  S->n_mapped = need;
  CU_TRY(cudaMemcpyAsync(S->d_page_table + lo, S->h_page_table + lo, (size_t)(need - lo) * 4, cudaMemcpyHostToDevice,
                         S->stream));
  return PS_OK;
}

// Free the pages lying wholly at or beyond kv_len: O(#freed pages).
static void free_pages_from(ps_stage* S, long long kv_len) {
  const int first = (int)((kv_len + S->page_size - 1) / S->page_size);
  for (int lp = S->n_mapped - 1; lp >= first; --lp) {
    S->free_pages.push_back(S->page_of[lp]);
    S->page_of[lp] = -1;   // the pinned mirror entry may still be in flight: leave it
  }
  if (first < S->n_mapped) S->n_mapped = first;
}

static long long pages_in_use(const ps_stage* S) {
  return (long long)S->pages_total - (long long)S->free_pages.size();
}

static void update_onpath(ps_stage* S) {
  if (S->S_host.empty()) return;
  const long long gen = (long long)S->tokens.size() - S->n_prompt;
  if (S->onpath > gen) S->onpath = (int)std::max(0LL, gen);
  while (S->onpath < gen && S->onpath < (int)S->S_host.size() &&
         S->tokens[S->n_prompt + S->onpath] == S->S_host[S->onpath])
    ++S->onpath;
}

// ============================================================================ C ABI
extern "C" {

const char* ps_last_error(void) { return g_err.c_str(); }
int32_t ps_version(void) { return 100; }
int64_t ps_kernel_launch_count(void) { return g_launches.load(); }

static ps_status validate_shape(const ps_model_shape* s) {
  if (!s) return fail(PS_E_INVALID, "shape is NULL");
  if (s->vocab < 2 || s->d_model <= 0 || s->n_layers < 0 || s->n_heads <= 0 || s->n_kv_heads <= 0)
    return fail(PS_E_INVALID, "bad shape sizes");
  if (s->n_heads % s->n_kv_heads) return fail(PS_E_INVALID, "n_heads %% n_kv_heads != 0");
  if (s->head_dim != 64 && s->head_dim != 128) return fail(PS_E_INVALID, "head_dim must be 64 or 128");
  if (s->d_model % 64 || s->d_ffn % 64 || (s->n_heads * s->head_dim) % 64)
    return fail(PS_E_INVALID, "d_model, d_ffn and n_heads*head_dim must be multiples of 64");
  if (s->d_ffn <= 0) return fail(PS_E_INVALID, "d_ffn must be positive");
  return PS_OK;
}

ps_status ps_stage_destroy(ps_stage* S) {
  if (!S) return PS_OK;
  cudaSetDevice(S->device);
  if (S->stream) cudaStreamSynchronize(S->stream);
  for (int k = 0; k < 6; ++k) {
    if (S->mega_ph[k]) cudaFree(S->mega_ph[k]);
    if (S->mega_maps[k]) cudaFree(S->mega_maps[k]);
  }
  for (int q = 0; q < 8; ++q)
    if (S->peer_ipc[q]) cudaIpcCloseMemHandle(S->peers[q]);
  if (S->xch) cudaFree(S->xch);
  if (S->mega_dbg) cudaFree(S->mega_dbg);
  if (S->attn_dbg) cudaFree(S->attn_dbg);
  void* dev[] = {S->d_page_table, S->d_in, S->d_out, S->x, S->q, S->ss, S->logits, S->ws, S->xg, S->att, S->h,
                 S->amax, S->counters, S->attn_counters, S->attn_o, S->attn_ml, S->rope_cs, S->d_syn, S->d_S};
  for (void* p : dev)
    if (p) cudaFree(p);
  void* pf[] = {S->pf_x, S->pf_q, S->pf_xs, S->pf_att, S->pf_h, S->pf_tok};
  for (void* p : pf)
    if (p) cudaFree(p);
  if (S->h_pf_tok) cudaFreeHost(S->h_pf_tok);
  if (S->d_chain) cudaFree(S->d_chain);
  if (S->h_chain) cudaFreeHost(S->h_chain);
  for (auto& ev : S->chain_ev)
    if (ev) cudaEventDestroy(ev);
  if (S->pf_tok_ev) cudaEventDestroy(S->pf_tok_ev);
  if (S->h_page_table) cudaFreeHost(S->h_page_table);
  if (S->h_in) cudaFreeHost(S->h_in);
  for (auto& ev : S->in_ev)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : S->fwd_ev)
    if (ev) cudaEventDestroy(ev);
  if (S->done_ev) cudaEventDestroy(S->done_ev);
  if (S->h_out) cudaFreeHost(S->h_out);
  if (S->own_stream && S->stream) cudaStreamDestroy(S->stream);
  delete S;
  return PS_OK;
}

// ---------------------------------------------------------------- tensor-parallel wiring
static void drop_tables(ps_stage* S) {   // phase tables embed peer pointers: rebuild after (re)connect
  for (int k = 0; k < 6; ++k) {
    if (S->mega_ph[k]) cudaFree(S->mega_ph[k]);
    if (S->mega_maps[k]) cudaFree(S->mega_maps[k]);
    S->mega_ph[k] = nullptr;
    S->mega_maps[k] = nullptr;
  }
}

// Build every phase table now: building one lazily inside a forward allocates
// and copies synchronously, which would wait for a peer rank's running
// megakernel that is itself waiting for this rank's forward.
static ps_status build_all_tables(ps_stage* S) {
  for (int b = 0; b < 3; ++b)
    for (int h = 0; h < (b < 2 ? 2 : 1); ++h) {   // the 64-row bucket never runs the lm_head
      ps_status st = build_mega(S, b, h != 0);
      if (st != PS_OK) return st;
    }
  CU_TRY(cudaDeviceSynchronize());
  return PS_OK;
}

// Exported handle: the IPC handle of the exchange buffer plus what every rank
// must agree on -- the megakernel grid (each rank waits for its peers' phase
// counters at ITS OWN target gen * n_ctas), the buffer size and the shard shape.
struct TpHandle {
  cudaIpcMemHandle_t ipc;
  uint32_t magic;
  int32_t tp_rank, tp_size, n_ctas;
  int64_t xch_bytes;
  ps_model_shape shard;
};
static_assert(sizeof(TpHandle) <= PS_TP_HANDLE_BYTES, "handle size");
constexpr uint32_t kTpMagic = 0x50535450u;   // "PSTP"

ps_status ps_tp_handle(ps_stage* S, void* handle_out) {
  if (!S || !handle_out) return fail(PS_E_INVALID, "NULL argument");
  CU_TRY(cudaSetDevice(S->device));
  TpHandle h;
  memset(&h, 0, sizeof h);
  CU_TRY(cudaIpcGetMemHandle(&h.ipc, S->xch));
  h.magic = kTpMagic;
  h.tp_rank = S->tp_rank;
  h.tp_size = S->tp_size;
  h.n_ctas = S->n_ctas;
  h.xch_bytes = (int64_t)S->xch_bytes;
  h.shard = S->sh;
  memset(handle_out, 0, PS_TP_HANDLE_BYTES);
  memcpy(handle_out, &h, sizeof h);
  return PS_OK;
}

ps_status ps_tp_connect(ps_stage* S, const void* handles) {
  if (!S || !handles) return fail(PS_E_INVALID, "NULL argument");
  if (S->tp_size < 2) return fail(PS_E_INVALID, "stage is not tensor parallel");
  for (int q = 0; q < S->tp_size; ++q) {   // every rank must match this one's grid and shard
    if (q == S->tp_rank) continue;
    TpHandle h;
    memcpy(&h, (const uint8_t*)handles + (size_t)q * PS_TP_HANDLE_BYTES, sizeof h);
    if (h.magic != kTpMagic || h.tp_rank != q || h.tp_size != S->tp_size)
      return fail(PS_E_INVALID, "handle %d is not rank %d of a tp_size %d group", q, q, S->tp_size);
    if (h.n_ctas != S->n_ctas || h.xch_bytes != (int64_t)S->xch_bytes || memcmp(&h.shard, &S->sh, sizeof S->sh) != 0)
      return fail(PS_E_INVALID, "rank %d: megakernel grid (%d vs %d CTAs) or shard shape differs from rank %d", q,
                  h.n_ctas, S->n_ctas, S->tp_rank);
  }
  CU_TRY(cudaSetDevice(S->device));
  CU_TRY(cudaStreamSynchronize(S->stream));
  drop_tables(S);
  for (int q = 0; q < S->tp_size; ++q) {
    if (q == S->tp_rank) continue;
    if (S->peer_ipc[q]) { cudaIpcCloseMemHandle(S->peers[q]); S->peer_ipc[q] = false; }
    TpHandle h;
    memcpy(&h, (const uint8_t*)handles + (size_t)q * PS_TP_HANDLE_BYTES, sizeof h);
    void* p = nullptr;
    CU_TRY(cudaIpcOpenMemHandle(&p, h.ipc, cudaIpcMemLazyEnablePeerAccess));
    S->peers[q] = (uint8_t*)p;
    S->peer_ipc[q] = true;
  }
  ps_status st = build_all_tables(S);
  if (st != PS_OK) return st;
  S->tp_connected = true;
  return PS_OK;
}

ps_status ps_tp_connect_local(ps_stage* const* stages, int32_t n) {
  if (!stages || n < 2 || n > 8) return fail(PS_E_INVALID, "need 2..8 stages");
  for (int r = 0; r < n; ++r) {
    const ps_stage* A = stages[r];
    if (!A) return fail(PS_E_INVALID, "NULL stage");
    if (A->tp_size != n || A->tp_rank != r) return fail(PS_E_INVALID, "stage %d: tp_rank/tp_size mismatch", r);
    if (A->n_ctas != stages[0]->n_ctas || A->xch_bytes != stages[0]->xch_bytes ||
        memcmp(&A->sh, &stages[0]->sh, sizeof A->sh) != 0)
      return fail(PS_E_INVALID, "stage %d: shard shape / grid differs from rank 0", r);
  }
  for (int r = 0; r < n; ++r) {
    ps_stage* A = stages[r];
    CU_TRY(cudaSetDevice(A->device));
    CU_TRY(cudaStreamSynchronize(A->stream));
    drop_tables(A);
    for (int q = 0; q < n; ++q) {
      const ps_stage* B = stages[q];
      if (B->device != A->device) {
        int ok = 0;
        CU_TRY(cudaDeviceCanAccessPeer(&ok, A->device, B->device));
        if (!ok) return fail(PS_E_CUDA, "no peer access %d -> %d", A->device, B->device);
        cudaError_t e = cudaDeviceEnablePeerAccess(B->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          return fail(PS_E_CUDA, "enable peer access: %s", cudaGetErrorString(e));
        cudaGetLastError();
      }
      A->peers[q] = B->xch;
    }
    ps_status st = build_all_tables(A);
    if (st != PS_OK) return st;
    A->tp_connected = true;
  }
  return PS_OK;
}

ps_status ps_stage_create(const ps_model_shape* shape, const ps_weights* w, const ps_placement* pl,
                          const ps_stage_opts* o, ps_stage** out) {
  ps_status st;
  if (!out || !w || !pl || !o) return fail(PS_E_INVALID, "NULL argument");
  if ((st = validate_shape(shape)) != PS_OK) return st;
  const int tp = pl->tp_size < 1 ? 1 : pl->tp_size;
  if (tp > 8 || pl->tp_rank < 0 || pl->tp_rank >= tp) return fail(PS_E_INVALID, "tp_rank/tp_size out of range (tp <= 8)");
  if (tp > 1) {
    if (shape->n_heads % tp || shape->n_kv_heads % tp || shape->vocab % tp || shape->d_ffn % (64 * tp) ||
        shape->d_model % 128)
      return fail(PS_E_INVALID, "tensor parallel needs heads, kv_heads, vocab divisible by tp, d_ffn by 64*tp, "
                                "d_model by 128");
  }
  if (o && o->max_ctas < 0) return fail(PS_E_INVALID, "max_ctas must be >= 0");
  if (o->max_seq < 2) return fail(PS_E_INVALID, "max_seq must be >= 2");
  if (o->max_window < 0 || o->max_window > kMaxRows - 1) return fail(PS_E_INVALID, "max_window must be 0..31");
  if (o->page_size != 64 && o->page_size != 128 && o->page_size != 256)
    return fail(PS_E_INVALID, "page_size must be 64, 128 or 256");
  if (!w->embed || !w->lm_head || !w->final_norm || (shape->n_layers > 0 && !w->layers))
    return fail(PS_E_INVALID, "NULL weight pointer");
  const int64_t need = ps_kv_pool_bytes_tp(shape, o->max_seq, o->page_size, tp);
  if ((need > 0 && !o->kv_pool) || o->kv_pool_bytes < need)
    return fail(PS_E_INVALID, "kv_pool too small (%lld < %lld bytes)", (long long)o->kv_pool_bytes, (long long)need);
  if ((st = init_stage_device(pl->device)) != PS_OK) return st;

  ps_stage* S = new (std::nothrow) ps_stage();
  if (!S) return fail(PS_E_INVALID, "out of host memory");
  auto bail = [&](ps_status s2) {
    std::string keep = g_err;
    ps_stage_destroy(S);
    g_err = keep;
    return s2;
  };
#define S_TRY(expr)                                                                             \
  do {                                                                                          \
    cudaError_t e_ = (expr);                                                                    \
    if (e_ != cudaSuccess)                                                                      \
      return bail(fail(PS_E_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)));                   \
  } while (0)
#define P_TRY(expr)                                                                             \
  do {                                                                                          \
    ps_status s_ = (expr);                                                                      \
    if (s_ != PS_OK) return bail(s_);                                                           \
  } while (0)

  // this rank's shard of the model: heads, KV heads, FFN columns, vocabulary
  ps_model_shape shl = *shape;
  shl.n_heads /= tp; shl.n_kv_heads /= tp; shl.d_ffn /= tp; shl.vocab /= tp;
  const ps_model_shape& sh = shl;
  S->sh = sh;
  S->tp_size = tp;
  S->tp_rank = pl->tp_rank;
  S->vocab_full = shape->vocab;
  S->vocab_off = pl->tp_rank * sh.vocab;
  S->tp_connected = tp == 1;
  S->n_ctas = o->max_ctas > 0 ? std::min(o->max_ctas, g_num_sms) : g_num_sms;
  S->device = pl->device;
  S->max_seq = o->max_seq;
  S->max_window = o->max_window;
  S->page_size = o->page_size;
  if (!o->use_megakernel) return bail(fail(PS_E_INVALID, "use_megakernel must be 1 (the only forward path)"));
  if (o->stream) {
    S->stream = (cudaStream_t)o->stream;
  } else {
    S_TRY(cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking));
    S->own_stream = true;
  }
  S->embed = (const __nv_bfloat16*)w->embed;
  S->lm_head = (const __nv_bfloat16*)w->lm_head;
  S->final_norm = (const __nv_bfloat16*)w->final_norm;
  S->lw.assign((size_t)std::max(sh.n_layers, 1) * 9, nullptr);
  for (int i = 0; i < sh.n_layers * 9; ++i) {
    S->lw[i] = (const __nv_bfloat16*)w->layers[i];
    if (!S->lw[i]) return bail(fail(PS_E_INVALID, "NULL layer weight %d", i));
  }
  const int d = sh.d_model, hq = sh.n_heads * sh.head_dim, hkv = sh.n_kv_heads * sh.head_dim, f = sh.d_ffn;
  // --- TMA maps over the borrowed weights
  S->maps.resize(sh.n_layers);
  for (int l = 0; l < sh.n_layers; ++l) {
    const __nv_bfloat16* const* W = &S->lw[(size_t)l * 9];
    LayerMaps& M = S->maps[l];
    P_TRY(make_map(&M.q, W[PS_WQ], hq, d, 128));
    P_TRY(make_map(&M.k, W[PS_WK], hkv, d, 128));
    P_TRY(make_map(&M.v, W[PS_WV], hkv, d, 128));
    P_TRY(make_map(&M.o, W[PS_WO], d, hq, 128));
    P_TRY(make_map(&M.g, W[PS_WG], f, d, 64));
    P_TRY(make_map(&M.u, W[PS_WU], f, d, 64));
    P_TRY(make_map(&M.d, W[PS_WD], d, f, 128));
  }
  P_TRY(make_map(&S->map_lm, S->lm_head, sh.vocab, d, 128));
  // --- scratch
  S->xg_ld = d;
  S->ss_ld = (d + 127) / 128;
  S_TRY(cudaMalloc(&S->d_in, sizeof(StepIn)));
  S_TRY(cudaMalloc(&S->d_out, sizeof(StepOut)));
  S_TRY(cudaHostAlloc(&S->h_in, 8 * sizeof(StepIn), cudaHostAllocDefault));
  for (auto& ev : S->in_ev) S_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  for (auto& ev : S->fwd_ev) S_TRY(cudaEventCreate(&ev));
  S_TRY(cudaEventCreateWithFlags(&S->done_ev, cudaEventDisableTiming));
  S_TRY(cudaHostAlloc(&S->h_out, sizeof(StepOut), cudaHostAllocMapped));
  S_TRY(cudaHostGetDevicePointer((void**)&S->h_out_dev, S->h_out, 0));
  memset(S->h_in, 0, 8 * sizeof(StepIn));
  S_TRY(cudaMalloc(&S->x, (size_t)kRowsCap * d * 4));
  // split-bf16 GEMM operands: hi rows [0, kRowsCap), lo rows [kRowsCap, 2 kRowsCap)
  S_TRY(cudaMalloc(&S->xg, (size_t)2 * kRowsCap * d * 2));
  S_TRY(cudaMalloc(&S->att, (size_t)2 * kRowsCap * hq * 2));
  S_TRY(cudaMalloc(&S->h, (size_t)2 * kRowsCap * f * 2));
  S_TRY(cudaMalloc(&S->q, (size_t)kRowsCap * hq * 4));
  S_TRY(cudaMalloc(&S->ss, (size_t)kRowsCap * S->ss_ld * 4));
  S_TRY(cudaMalloc(&S->logits, (size_t)kMaxRows * sh.vocab * 4));
  S_TRY(cudaMemset(S->x, 0, (size_t)kRowsCap * d * 4));
  S_TRY(cudaMemset(S->xg, 0, (size_t)2 * kRowsCap * d * 2));
  S_TRY(cudaMemset(S->att, 0, (size_t)2 * kRowsCap * hq * 2));
  S_TRY(cudaMemset(S->h, 0, (size_t)2 * kRowsCap * f * 2));
  S_TRY(cudaMemset(S->q, 0, (size_t)kRowsCap * hq * 4));
  S_TRY(cudaMemset(S->ss, 0, (size_t)kRowsCap * S->ss_ld * 4));
  for (int b = 0; b < 3; ++b) {
    P_TRY(make_map(&S->map_xg[b], S->xg, 2 * kRowsCap, d, bucket_rp(b)));
    P_TRY(make_map(&S->map_att[b], S->att, 2 * kRowsCap, hq, bucket_rp(b)));
    P_TRY(make_map(&S->map_h[b], S->h, 2 * kRowsCap, f, bucket_rp(b)));
  }
  // --- GEMM partitions (persistent grid = #SMs, stream-K)
  const int n = S->n_ctas;
  // tile-aligned partitions where they pay (gemm_shape): d_model > 2048 only
  // (round 2, split-bf16 operands and the keys-as-M attention: the 1B draft
  // step 0.955 ms with >= 60% aligned partitions, 0.946 with pure stream-K)
  const int align = d <= 2048 ? 0 : 95;
  S->gs_qkv = gemm_shape((hq + 127) / 128 + 2 * ((hkv + 127) / 128), d, n, align);
  S->gs_o = gemm_shape((d + 127) / 128, hq, n, align);
  S->gs_gu = gemm_shape((f + 63) / 64, d, n, align);
  S->gs_d = gemm_shape((d + 127) / 128, f, n, align);
  S->gs_lm = gemm_shape((sh.vocab + 127) / 128, d, n, align);
  S->lm_tiles = S->gs_lm.n_tiles;
  size_t ws_tiles = 0;
  int max_tiles = 0;
  for (const GemmShape* g : {&S->gs_qkv, &S->gs_o, &S->gs_gu, &S->gs_d, &S->gs_lm}) {
    ws_tiles = std::max(ws_tiles, (size_t)g->n_tiles * g->maxseg);
    max_tiles = std::max(max_tiles, g->n_tiles);
  }
  // stream-K partials [tile][segment][128][rows] of one forward (rows <= 32; 8-byte
  // LL words), or of each 16-row chunk of the 64-row bucket (regions of ws_chunk floats)
  const size_t ws_chunk = ws_tiles * 16 * 128 * 2;
  const size_t ws_elems = ws_tiles * kRowsCap * 128;
  S->ws_chunk = (long long)ws_chunk;
  S->cnt_chunk = max_tiles;
  // fp32 partials (release path) or (fp32, flag) words (LL path): 8 bytes each;
  // zeroed so no stale flag of a freed buffer can match
  S->ws_bytes = ws_elems * 8;
  S_TRY(cudaMalloc(&S->ws, S->ws_bytes));
  S_TRY(cudaMemset(S->ws, 0, S->ws_bytes));
  S_TRY(cudaMalloc(&S->counters, (size_t)max_tiles * (kRowsCap / 16) * 4));
  S_TRY(cudaMemset(S->counters, 0, (size_t)max_tiles * (kRowsCap / 16) * 4));
  S_TRY(cudaMalloc(&S->amax, (size_t)kMaxRows * 8));
  S_TRY(cudaMemset(S->amax, 0, (size_t)kMaxRows * 8));
  // --- attention workspace
  // keys per attention work item: sc 64-key chunks, a per-stage constant
  // (results must not depend on R or on the context length).  At max_seq, a
  // one-row-block window has kv_heads x ceil(chunks / sc) items of 4 sc ring
  // stages on n_ctas CTAs, and every query row combines ceil(chunks / sc)
  // partials: sc (a power of two <= 16) minimises the makespan in stages +
  // 0.2 per partial (ties to the larger sc), fitted to the 8B with sc forced
  // (`profiles/r02_attn_sc_sweep.log`: best at 4K keys sc 4, 8K 8, 16K 16 --
  // what this picks; R = 5 at 8K 5.83 ms with the previous rule (sc 1) vs
  // 5.22 with sc 8).
  {
    const int chunks = (S->max_seq + kRowsCap + kAttnChunk - 1) / kAttnChunk;
    long long best = -1;
    // up to 1.5K keys one-chunk items: a CTA's whole item (<= 4 stages) is
    // prefetched into the ring during the QKV phase (measured at 1K keys: sc 1
    // 0.696 of the HBM peak vs sc 2 0.648 for R = 1)
    for (int sc = 1; sc <= (chunks <= 24 ? 1 : 16); sc *= 2) {
      const long long items = (long long)sh.n_kv_heads * ((chunks + sc - 1) / sc);
      const long long cost = 10 * ((items + S->n_ctas - 1) / S->n_ctas) * 4 * sc + 2 * ((chunks + sc - 1) / sc);
      if (best < 0 || cost <= best) {
        best = cost;
        S->attn_sc = sc;
      }
    }
#ifdef PS_ATTN_SC                               // A/B builds: keys per item forced
    S->attn_sc = PS_ATTN_SC;
#endif
    S->max_chunks = kAttnWarps * ((chunks + S->attn_sc - 1) / S->attn_sc);   // item partials per (head, row block)   // item partials per (head, row block)
  }
  {
    const int g = sh.n_heads / sh.n_kv_heads;
    S->max_rb = (kRowsCap * g + kAttnRB - 1) / kAttnRB;   // attention row blocks of kAttnRB query rows
  }
  S->attn_grid = std::min(sh.n_kv_heads * S->max_rb * S->max_chunks, 2 * n);
  const size_t attn_rows = (size_t)sh.n_kv_heads * S->max_rb * S->max_chunks * kAttnRB;
  S_TRY(cudaMalloc(&S->attn_o, attn_rows * sh.head_dim * 4));
  S_TRY(cudaMalloc(&S->attn_ml, attn_rows * 2 * 4));
  // --- RoPE table
  {
    std::vector<float2> cs;
    rope_table(sh, S->max_seq + kRowsCap, cs);
    S_TRY(cudaMalloc(&S->rope_cs, cs.size() * sizeof(float2)));
    S_TRY(cudaMemcpy(S->rope_cs, cs.data(), cs.size() * sizeof(float2), cudaMemcpyHostToDevice));
  }
  // --- paged KV
  S->kv = (__nv_bfloat16*)o->kv_pool;
  S->page_elems = (long long)sh.n_layers * kKvPlanes * sh.n_kv_heads * S->page_size * sh.head_dim;
  const int lpages = (S->max_seq + kRowsCap + S->page_size - 1) / S->page_size;
  S->pages_total = S->page_elems ? (int)(o->kv_pool_bytes / (S->page_elems * 2)) : lpages;   // 0 layers: no KV
  if (S->page_elems) {
    // Attention stages load whole 16-key groups and mask the keys past the
    // context: those must hold finite values (0 * NaN = NaN in P V), so the
    // pool's pages start zeroed (later stale rows are finite K/V).
    S_TRY(cudaMemset(S->kv, 0, (size_t)S->pages_total * S->page_elems * 2));
    P_TRY(make_map_kv(&S->map_kv, S->kv, (uint64_t)S->pages_total * (S->page_elems / sh.head_dim), sh.head_dim,
                      (uint64_t)sh.n_kv_heads * S->page_size));
  }
  S->page_of.assign(lpages, -1);
  for (int p = S->pages_total - 1; p >= 0; --p) S->free_pages.push_back(p);
  S_TRY(cudaMalloc(&S->d_page_table, (size_t)lpages * 4));
  S_TRY(cudaMemset(S->d_page_table, 0, (size_t)lpages * 4));
  S_TRY(cudaHostAlloc(&S->h_page_table, (size_t)lpages * 4, cudaHostAllocDefault));
  memset(S->h_page_table, 0, (size_t)lpages * 4);
#if PS_TRACE
  S_TRY(cudaMalloc(&S->attn_dbg, (size_t)1024 * 8 * 8));
  S_TRY(cudaMemset(S->attn_dbg, 0, (size_t)1024 * 8 * 8));
  S_TRY(cudaMalloc(&S->mega_dbg, (size_t)g_num_sms * kMaxPhases(sh.n_layers) * 8 * 8));
  S_TRY(cudaMemset(S->mega_dbg, 0, (size_t)g_num_sms * kMaxPhases(sh.n_layers) * 8 * 8));
  S_TRY(cudaMalloc(&S->epi_dbg, (size_t)kMaxPhases(sh.n_layers) * g_num_sms * 4 * 8));
#endif
  // --- exchange buffer: megakernel phase-completion counters (cumulative; see
  // ps_mega.cuh), tensor-parallel partials and argmax keys (read by peers)
  S->off_part = ((size_t)kMaxPhases(sh.n_layers) * 4 + 255) / 256 * 256;
  S->off_keys = S->off_part + (size_t)2 * kRowsCap * d * 4;
  S->xch_bytes = S->off_keys + (size_t)2 * kMaxRows * 8;
  S_TRY(cudaMalloc(&S->xch, S->xch_bytes));
  S_TRY(cudaMemset(S->xch, 0, S->xch_bytes));
  S->mega_done = (unsigned*)S->xch;
  S->peers[S->tp_rank] = S->xch;
  // --- chained draft forwards
  S_TRY(cudaMalloc(&S->d_chain, kMaxChain * 4));
  S_TRY(cudaMemset(S->d_chain, 0, kMaxChain * 4));
  S_TRY(cudaHostAlloc(&S->h_chain, kMaxChain * 4, cudaHostAllocDefault));
  for (auto& ev : S->chain_ev) S_TRY(cudaEventCreate(&ev));
  // --- synthetic override (disabled)
  S_TRY(cudaMalloc(&S->d_syn, sizeof(SynthParams)));
  S->h_syn = SynthParams{};
  S_TRY(cudaMemcpy(S->d_syn, &S->h_syn, sizeof(SynthParams), cudaMemcpyHostToDevice));
  S_TRY(cudaStreamSynchronize(S->stream));
  // --- NEXT-3 prefill kernels (single-GPU stages with layers)
  if (tp == 1 && sh.n_layers > 0) {
    const size_t R = kPfRows;
    S_TRY(cudaMalloc(&S->pf_x, R * d * 4));
    S_TRY(cudaMalloc(&S->pf_q, R * hq * 4));
    S_TRY(cudaMalloc(&S->pf_xs, 2 * R * d * 2));
    S_TRY(cudaMalloc(&S->pf_att, 2 * R * hq * 2));
    S_TRY(cudaMalloc(&S->pf_h, 2 * R * f * 2));
    S_TRY(cudaMalloc(&S->pf_tok, R * 4));
    S_TRY(cudaMemset(S->pf_xs, 0, 2 * R * d * 2));
    S_TRY(cudaMemset(S->pf_att, 0, 2 * R * hq * 2));
    S_TRY(cudaMemset(S->pf_h, 0, 2 * R * f * 2));
    S_TRY(cudaHostAlloc(&S->h_pf_tok, R * 4, cudaHostAllocDefault));
    S_TRY(cudaEventCreateWithFlags(&S->pf_tok_ev, cudaEventDisableTiming));
    CUtensorMap mxs, matt, mh;
    P_TRY(make_map(&mxs, S->pf_xs, 2 * R, d, 128));
    P_TRY(make_map(&matt, S->pf_att, 2 * R, hq, 128));
    P_TRY(make_map(&mh, S->pf_h, 2 * R, f, 128));
    int shift = 0;
    while ((1 << shift) < S->page_size) ++shift;
    S->pf_gemm.resize((size_t)sh.n_layers * 4);
    for (int l = 0; l < sh.n_layers; ++l) {
      const __nv_bfloat16* const* W = &S->lw[(size_t)l * 9];
      const LayerMaps& M = S->maps[l];
      PfGemmParams* g = &S->pf_gemm[(size_t)l * 4];
      for (int k = 0; k < 4; ++k) memset(&g[k], 0, sizeof(PfGemmParams));
      // QKV: q tiles, then k, then v (each matrix's rows padded to 128)
      g[0].mX = mxs; g[0].mW0 = M.q; g[0].mW1 = M.k; g[0].mW2 = M.v;
      g[0].K = d;
      g[0].N = hq + 2 * hkv;                          // (tiles per matrix set at launch, per tile width)
      g[0].nq = hq; g[0].nk = hkv;
      g[0].q = S->pf_q; g[0].ld_q = hq;
      g[0].kv = S->kv; g[0].page_table = S->d_page_table; g[0].page_size = S->page_size; g[0].page_shift = shift;
      g[0].layer = l; g[0].hkv = sh.n_kv_heads; g[0].hd = sh.head_dim; g[0].page_stride = S->page_elems;
      g[0].rope_cs = S->rope_cs;
      // O (+ residual): x += att Wo^T
      g[1].mX = matt; g[1].mW0 = M.o; g[1].K = hq; g[1].N = d; g[1].x = S->pf_x; g[1].ld_x = d;
      // gate/up (+ SiLU * mul): 128-row boxes of Wg and Wu
      g[2].mX = mxs; g[2].K = d; g[2].N = f; g[2].h = S->pf_h; g[2].ld_h = f;
      P_TRY(make_map(&g[2].mW0, W[PS_WG], f, d, 128));
      P_TRY(make_map(&g[2].mW1, W[PS_WU], f, d, 128));
      g[2].mG64 = M.g;                                 // (the megakernel's 64-row boxes)
      g[2].mU64 = M.u;
      P_TRY(make_map(&g[2].mG112, W[PS_WG], f, d, 112));
      P_TRY(make_map(&g[2].mU112, W[PS_WU], f, d, 112));
      // down (+ residual)
      g[3].mX = mh; g[3].mW0 = M.d; g[3].K = f; g[3].N = d; g[3].x = S->pf_x; g[3].ld_x = d;
    }
    S->pf_ready = (d % 64 == 0) && (hq % 64 == 0) && (f % 64 == 0) && (sh.head_dim == 64 || sh.head_dim == 128) &&
                  64 % (sh.n_heads / sh.n_kv_heads) == 0;
  }
  // phase tables now (tensor-parallel groups build theirs at connect time)
  if (tp == 1) P_TRY(build_all_tables(S));
  *out = S;
#undef S_TRY
#undef P_TRY
  return PS_OK;
}

// One forward over tokens [start, start+R) at positions [start, start+R);
// with_head computes logits/argmax for all rows.  dev_window (optional): a
// DEVICE array of w draft tokens copied on-stream into rows row0+1.. (the host
// rows there are placeholders).  The stage's forward counters (gen, gen_head:
// the megakernel's cumulative phase targets) are committed only once the
// forward is enqueued, so a failed launch leaves them consistent with the
// device counters.
// chain_flags / chain_idx / syn_g: chained draft forwards (ps_draft): the
// forward's slot in the chain array and its generated index (the host's token
// buffer does not hold the chain's earlier tokens yet).
static ps_status forward_rows(ps_stage* S, const int32_t* toks, int R, long long pos0, int w, bool with_head,
                              bool want_logits, int row0 = 0, const int32_t* dev_window = nullptr,
                              int chain_flags = 0, int chain_idx = 0, long long syn_g = -1) {
  ps_status st;
  if (!S->tp_connected) return fail(PS_E_INVALID, "tensor-parallel stage not connected (ps_tp_connect)");
  if ((st = ensure_pages(S, pos0 + R - 1)) != PS_OK) return st;
  CU_TRY(cudaEventSynchronize(S->in_ev[S->in_slot]));   // slot's previous copy done
  const unsigned gen = S->gen + 1, gen_head = S->gen_head + (with_head ? 1 : 0);
  // LL stream-K flags carry gen mod 2^22 (ps_kernels.cuh): clear the partial
  // workspace every 2^20 forwards so no slot can hold a flag old enough to alias
  if ((gen & ((1u << 20) - 1)) == 0) CU_TRY(cudaMemsetAsync(S->ws, 0, S->ws_bytes, S->stream));
  StepIn* in = S->h_in + S->in_slot;
  in->R = R;
  in->pos0 = (int32_t)pos0;
  in->w = w;
  in->flags = (want_logits ? kFlagLogits : 0) | chain_flags;
  in->chain_idx = chain_idx;
  in->syn_p0 = 0;
  in->syn_onpath = 0;
  in->row0 = row0;
  in->gen = (int32_t)gen;
  in->gen_head = (int32_t)gen_head;
  if (with_head && !S->S_host.empty()) {
    in->flags |= kFlagSynth;
    const long long g = syn_g >= 0 ? syn_g : (long long)S->tokens.size() - S->n_prompt;
    in->syn_p0 = (int32_t)g;
    in->syn_onpath = (g >= 0 && S->onpath == g) ? 1 : 0;   // (a kFlagChainIn forward takes it from the chain)
  }
  for (int j = 0; j < kRowsCap; ++j) in->tokens[j] = j < R ? toks[j] : 0;
  const int b = bucket_of(R);
  S->last_bucket = b;
  // Forwards are enqueued back to back (prefill chunks): each uses its own
  // staging slot, and a slot is rewritten only after its previous copy ran.
  CU_TRY(cudaMemcpyAsync(S->d_in, S->h_in + S->in_slot, sizeof(StepIn), cudaMemcpyHostToDevice, S->stream));
  if (dev_window && w > 0)
    CU_TRY(cudaMemcpyAsync(S->d_in->tokens + row0 + 1, dev_window, (size_t)w * 4, cudaMemcpyDeviceToDevice,
                           S->stream));
  CU_TRY(cudaEventRecord(S->in_ev[S->in_slot], S->stream));
  S->in_slot = (S->in_slot + 1) % 8;
  if (with_head) CU_TRY(cudaEventRecord(S->fwd_ev[0], S->stream));
  st = launch_mega(S, b, with_head);
  if (st != PS_OK) return st;
  S->gen = gen;                        // the forward is enqueued: commit the counters
  S->gen_head = gen_head;
  if (with_head) CU_TRY(cudaEventRecord(S->fwd_ev[1], S->stream));
  return PS_OK;
}

// NEXT-3: positions [pos0, pos0 + T) (T <= kPfRows) through the prefill
// kernels (ps_prefill.cuh): per layer norm, QKV GEMM (+ RoPE, KV append),
// causal attention, O GEMM (+ residual), norm, gate/up GEMM (+ SwiGLU), down
// GEMM (+ residual).  No lm_head (prefill predicts nothing: the last prompt
// token stays pending).
static ps_status prefill_chunk(ps_stage* S, const int32_t* toks, int T, long long pos0) {
  ps_status st;
  if ((st = ensure_pages(S, pos0 + T - 1)) != PS_OK) return st;
  const ps_model_shape& sh = S->sh;
  const int d = sh.d_model, hq = sh.n_heads * sh.head_dim;
  const int mt = (T + 127) / 128;
  CU_TRY(cudaEventSynchronize(S->pf_tok_ev));              // the staging buffer's previous copy ran
  memcpy(S->h_pf_tok, toks, (size_t)T * 4);
  CU_TRY(cudaMemcpyAsync(S->pf_tok, S->h_pf_tok, (size_t)T * 4, cudaMemcpyHostToDevice, S->stream));
  CU_TRY(cudaEventRecord(S->pf_tok_ev, S->stream));
  int shift = 0;
  while ((1 << shift) < S->page_size) ++shift;
  PfAttnParams ap{};
  ap.q = S->pf_q; ap.ld_q = hq;
  ap.kv = S->kv; ap.page_table = S->d_page_table; ap.page_size = S->page_size; ap.page_shift = shift;
  ap.hkv = sh.n_kv_heads; ap.H = sh.n_heads; ap.page_stride = S->page_elems;
  ap.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)sh.head_dim));
  ap.T = T; ap.pos0 = (int)pos0; ap.out = S->pf_att; ap.ld_out = hq;
  const int QB = 64 / (sh.n_heads / sh.n_kv_heads);
  const dim3 agrid((T + QB - 1) / QB, sh.n_kv_heads);
  // Tile width: 256 features (half the activation re-reads per FLOP) unless the
  // 128-wide tiling finishes in fewer tile-times on the persistent grid (wave
  // quantisation: cost = ceil(tiles / SMs) x width, by at least 25%); a SwiGLU tile holds
  // width / 2 gate rows and the same up rows.
  auto gemm = [&](int mode, PfGemmParams& g) -> ps_status {
    g.T = T;
    g.pos0 = (int)pos0;
    g.m_tiles = mt;
    const int hkv = sh.n_kv_heads * sh.head_dim;
    auto tiles = [&](int bn) {
      return mode == PF_QKV ? (hq + bn - 1) / bn + 2 * ((hkv + bn - 1) / bn)
             : mode == PF_SWIGLU ? (g.N + bn / 2 - 1) / (bn / 2) : (g.N + bn - 1) / bn;
    };
    auto cost = [&](int bn) { return (long long)((tiles(bn) * mt + g_num_sms - 1) / g_num_sms) * bn; };
    int bn = 256;
    if (mode == PF_SWIGLU && cost(224) < cost(256)) bn = 224;   // (gate/up: 112 + 112 rows)
    if (4 * cost(128) <= 3 * cost(bn)) bn = 128;   // (a 128-wide tile moves more operand bytes per FLOP:
                                                   // 8B gate/up 128-wide on 7 waves slower than 256-wide on 4)
    g.n_tiles = tiles(bn);
    g.t1 = (hq + bn - 1) / bn;
    g.t2 = g.t1 + (hkv + bn - 1) / bn;
    const int grid = std::min(g.n_tiles * mt, g_num_sms);
    if (mode == PF_QKV && bn == 128) pf_gemm_kernel<PF_QKV, 128><<<grid, kPfThreads, pf_smem_bytes<128>(), S->stream>>>(g);
    else if (mode == PF_QKV) pf_gemm_kernel<PF_QKV, 256><<<grid, kPfThreads, pf_smem_bytes<256>(), S->stream>>>(g);
    else if (mode == PF_RESID && bn == 128)
      pf_gemm_kernel<PF_RESID, 128><<<grid, kPfThreads, pf_smem_bytes<128>(), S->stream>>>(g);
    else if (mode == PF_RESID) pf_gemm_kernel<PF_RESID, 256><<<grid, kPfThreads, pf_smem_bytes<256>(), S->stream>>>(g);
    else if (bn == 128) pf_gemm_kernel<PF_SWIGLU, 128><<<grid, kPfThreads, pf_smem_bytes<128>(), S->stream>>>(g);
    else if (bn == 224) pf_gemm_kernel<PF_SWIGLU, 224><<<grid, kPfThreads, pf_smem_bytes<224>(), S->stream>>>(g);
    else pf_gemm_kernel<PF_SWIGLU, 256><<<grid, kPfThreads, pf_smem_bytes<256>(), S->stream>>>(g);
    g_launches++;
    CU_TRY(cudaGetLastError());
    return PS_OK;
  };
  for (int l = 0; l < sh.n_layers; ++l) {
    const __nv_bfloat16* const* W = &S->lw[(size_t)l * 9];
    PfGemmParams* g = &S->pf_gemm[(size_t)l * 4];
    // h = RMSNorm(x) (layer 0: x = E[tok] first)
    pf_norm_kernel<<<T, kPfNormThreads, 0, S->stream>>>(l == 0 ? S->pf_tok : nullptr, S->embed, S->vocab_full, S->pf_x,
                                                         d, W[PS_N_ATTN], sh.rms_eps, S->pf_xs);
    g_launches++;
    if ((st = gemm(PF_QKV, g[0])) != PS_OK) return st;
    ap.layer = l;
    if (sh.head_dim == 128) pf_attn_kernel<128><<<agrid, 128, pf_attn_smem_bytes<128>(), S->stream>>>(ap);
    else pf_attn_kernel<64><<<agrid, 128, pf_attn_smem_bytes<64>(), S->stream>>>(ap);
    g_launches++;
    if ((st = gemm(PF_RESID, g[1])) != PS_OK) return st;
    pf_norm_kernel<<<T, kPfNormThreads, 0, S->stream>>>(nullptr, S->embed, S->vocab_full, S->pf_x, d, W[PS_N_MLP],
                                                         sh.rms_eps, S->pf_xs);
    g_launches++;
    if ((st = gemm(PF_SWIGLU, g[2])) != PS_OK) return st;
    if ((st = gemm(PF_RESID, g[3])) != PS_OK) return st;
  }
  CU_TRY(cudaGetLastError());
  return PS_OK;
}

ps_status ps_set_prefill_path(ps_stage* S, int32_t path) {
  if (!S) return fail(PS_E_INVALID, "NULL argument");
  if (path != PS_PREFILL_AUTO && path != PS_PREFILL_ROWS) return fail(PS_E_INVALID, "unknown prefill path %d", path);
  S->prefill_path = path;
  return PS_OK;
}

ps_status ps_prefill(ps_stage* S, const int32_t* tokens, int32_t n) {
  if (!S || !tokens) return fail(PS_E_INVALID, "NULL argument");
  PS_NOT_INFLIGHT(S);
  if (n < 1 || n > S->max_seq) return fail(PS_E_INVALID, "prefill length %d not in [1, max_seq]", n);
  for (int i = 0; i < n; ++i)
    if (tokens[i] < 0 || tokens[i] >= S->vocab_full) return fail(PS_E_INVALID, "token %d out of range", tokens[i]);
  CU_TRY(cudaSetDevice(S->device));
  // keep the KV of the longest common prefix
  long long m = 0;
  while (m < (long long)S->tokens.size() && m < n && S->tokens[m] == tokens[m]) ++m;
  // KV at position p depends on tokens[0..p] only: valid for p < m
  const long long keep_kv = std::min<long long>(S->kv_len, std::min<long long>(m, n - 1));
  S->tokens.assign(tokens, tokens + n);
  S->kv_len = keep_kv;
  free_pages_from(S, S->kv_len);
  update_onpath(S);
  // forward positions [kv_len, n-1): runs of >= 64 positions in chunks of up to
  // kPfRows tokens through the prefill kernels; the rest (and every position
  // with PS_PREFILL_ROWS) in chunks of up to kRowsCap rows through the decode
  // megakernel's 64-row bucket (no lm_head)
  const bool gemm_path = S->pf_ready && S->prefill_path == PS_PREFILL_AUTO;
  while (S->kv_len < n - 1) {
    const long long left = n - 1 - S->kv_len;
    ps_status st;
    int R;
    if (gemm_path && left >= kRowsCap) {
      R = (int)std::min<long long>(kPfRows, left);
      st = prefill_chunk(S, &S->tokens[S->kv_len], R, S->kv_len);
    } else {
      R = (int)std::min<long long>(kRowsCap, left);
      st = forward_rows(S, &S->tokens[S->kv_len], R, S->kv_len, 0, false, false);
    }
    if (st != PS_OK) {
      S->kv_len = 0;   // KV state unknown: force a full recompute next time
      free_pages_from(S, 0);
      return st;
    }
    S->kv_len += R;
  }
  CU_TRY(cudaStreamSynchronize(S->stream));
  return PS_OK;
}

// Rows of one verify forward: the KV catch-up suffix tokens[kv_len .. n-2]
// (non-empty only after a lazy ps_resync), the pending token x[n-1], then the
// window; predictions are read from rows row0 = n-1-kv_len onwards.
static ps_status catch_up(ps_stage* S, int reserve_rows) {
  const long long n = (long long)S->tokens.size();
  while ((n - 1 - S->kv_len) + reserve_rows > kMaxRows) {
    const int R = (int)std::min<long long>(kRowsCap, n - 1 - S->kv_len);
    ps_status st = forward_rows(S, &S->tokens[S->kv_len], R, S->kv_len, 0, false, false);
    if (st != PS_OK) return st;
    S->kv_len += R;
  }
  return PS_OK;
}

ps_status ps_resync(ps_stage* S, const int32_t* tokens, int32_t n) {
  if (!S || !tokens) return fail(PS_E_INVALID, "NULL argument");
  PS_NOT_INFLIGHT(S);
  if (n < 1 || n > S->max_seq) return fail(PS_E_INVALID, "resync length %d not in [1, max_seq]", n);
  for (int i = 0; i < n; ++i)
    if (tokens[i] < 0 || tokens[i] >= S->vocab_full) return fail(PS_E_INVALID, "token %d out of range", tokens[i]);
  long long m = 0;
  while (m < (long long)S->tokens.size() && m < n && S->tokens[m] == tokens[m]) ++m;
  S->kv_len = std::min<long long>(S->kv_len, std::min<long long>(m, n - 1));
  S->tokens.assign(tokens, tokens + n);
  free_pages_from(S, S->kv_len);
  update_onpath(S);
  return PS_OK;
}

// Enqueue one verification pass (rows = KV catch-up suffix, pending x[n-1],
// window) without waiting.  `window` is host memory, or (dev) device memory.
static ps_status verify_launch(ps_stage* S, const int32_t* window, int w, bool dev, float* logits_out) {
  const long long n = (long long)S->tokens.size();
  if (n < 1) return fail(PS_E_CONTRACT, "verify on an empty token buffer (call ps_prefill first)");
  if (w < 0 || w > S->max_window) return fail(PS_E_INVALID, "window %d > max_window %d", w, S->max_window);
  if (n + w > S->max_seq) return fail(PS_E_CAPACITY, "n + w = %lld exceeds max_seq", n + w);
  if (S->kv_len > n - 1) return fail(PS_E_CONTRACT, "KV covers %lld positions > n-1 = %lld", S->kv_len, n - 1);
  if (!dev)
    for (int j = 0; j < w; ++j)
      if (window[j] < 0 || window[j] >= S->vocab_full) return fail(PS_E_INVALID, "draft token %d out of range", window[j]);
  ps_status st = catch_up(S, 1 + w);
  if (st != PS_OK) return st;
  const int row0 = (int)(n - 1 - S->kv_len);
  int32_t rows[kMaxRows];
  for (int j = 0; j <= row0; ++j) rows[j] = S->tokens[S->kv_len + j];
  for (int j = 0; j < w; ++j) rows[row0 + 1 + j] = dev ? 0 : window[j];
  st = forward_rows(S, rows, row0 + 1 + w, S->kv_len, w, true, logits_out != nullptr, row0, dev ? window : nullptr);
  if (st != PS_OK) return st;
  if (logits_out) {
    cudaPointerAttributes at{};
    cudaMemcpyKind kind = cudaMemcpyDeviceToHost;
    if (cudaPointerGetAttributes(&at, logits_out) == cudaSuccess && at.type == cudaMemoryTypeDevice)
      kind = cudaMemcpyDeviceToDevice;
    cudaGetLastError();
    CU_TRY(cudaMemcpyAsync(logits_out, S->logits + (size_t)row0 * S->sh.vocab, (size_t)(w + 1) * S->sh.vocab * 4,
                           kind, S->stream));
  }
  S->if_n = n;
  S->if_w = w;
  return PS_OK;
}

// Commit the finished pass (its result is in the mapped pinned mirror).
static ps_status verify_commit(ps_stage* S, int32_t* a_out, int32_t* next_out) {
  {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, S->fwd_ev[0], S->fwd_ev[1]) == cudaSuccess) {
      S->last_fwd_ms = ms;
      S->sum_fwd_ms += ms;
      ++S->n_fwd;
    }
    cudaGetLastError();
  }
  const StepOut* r = S->h_out;
  const long long n = S->if_n;
  const int w = S->if_w;
  if (r->R == -1) return fail(PS_E_INVALID, "device window holds a token outside [0, vocab)");
  const int a = r->a, nxt = r->next;
  if (a < 0 || a > w || nxt < 0 || nxt >= S->vocab_full || r->kv_len != n + a)
    return fail(PS_E_CUDA, "corrupt verify result a=%d next=%d kv_len=%d", a, nxt, r->kv_len);
  for (int j = 0; j < a; ++j) S->tokens.push_back(r->pred[j]);   // accepted drafts: pred_j == d_j
  S->tokens.push_back(nxt);
  S->kv_len = n + a;
  free_pages_from(S, S->kv_len);
  update_onpath(S);
  *a_out = a;
  *next_out = nxt;
  return PS_OK;
}

static bool is_device_ptr(const void* p) {
  cudaPointerAttributes at{};
  const bool dev = p && cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeDevice;
  cudaGetLastError();
  return dev;
}

static ps_status verify_host(ps_stage* S, const int32_t* window, int w, int32_t* a_out, int32_t* next_out,
                             float* logits_out) {
  ps_status st = verify_launch(S, window, w, false, logits_out);
  if (st != PS_OK) return st;
  CU_TRY(cudaStreamSynchronize(S->stream));
  return verify_commit(S, a_out, next_out);
}

ps_status ps_verify(ps_stage* S, const int32_t* window, int32_t w, int32_t* accepted_len, int32_t* next_token,
                    float* opt_logits) {
  if (!S || !accepted_len || !next_token || (w > 0 && !window)) return fail(PS_E_INVALID, "NULL argument");
  PS_NOT_INFLIGHT(S);
  if (w < 0 || w > S->max_window) return fail(PS_E_INVALID, "window %d not in [0, max_window=%d]", w, S->max_window);
  CU_TRY(cudaSetDevice(S->device));
  int32_t host_window[kMaxRows];
  const int32_t* win = window;
  if (w > 0 && is_device_ptr(window)) {
    CU_TRY(cudaMemcpyAsync(host_window, window, (size_t)w * 4, cudaMemcpyDeviceToHost, S->stream));
    CU_TRY(cudaStreamSynchronize(S->stream));
    win = host_window;
  }
  return verify_host(S, win, w, accepted_len, next_token, opt_logits);
}

ps_status ps_verify_async(ps_stage* S, const int32_t* window, int32_t w, ps_verify_ticket* ticket) {
  if (!S || (w > 0 && !window)) return fail(PS_E_INVALID, "NULL argument");
  PS_NOT_INFLIGHT(S);
  if (w < 0 || w > S->max_window) return fail(PS_E_INVALID, "window %d not in [0, max_window=%d]", w, S->max_window);
  CU_TRY(cudaSetDevice(S->device));
  ps_status st = verify_launch(S, window, w, w > 0 && is_device_ptr(window), nullptr);
  if (st != PS_OK) return st;
  CU_TRY(cudaEventRecord(S->done_ev, S->stream));
  S->inflight = true;
  if (ticket) {
    ticket->d_result = reinterpret_cast<const ps_verify_result*>(S->d_out);
    ticket->h_result = reinterpret_cast<const ps_verify_result*>(S->h_out);
    ticket->event = S->done_ev;
  }
  return PS_OK;
}

ps_status ps_verify_wait(ps_stage* S, int32_t* accepted_len, int32_t* next_token) {
  if (!S || !accepted_len || !next_token) return fail(PS_E_INVALID, "NULL argument");
  if (!S->inflight) return fail(PS_E_INVALID, "no ps_verify_async pass in flight");
  CU_TRY(cudaSetDevice(S->device));
  S->inflight = false;
  CU_TRY(cudaEventSynchronize(S->done_ev));
  return verify_commit(S, accepted_len, next_token);
}

ps_status ps_verify_query(ps_stage* S, int32_t* done) {
  if (!S || !done) return fail(PS_E_INVALID, "NULL argument");
  if (!S->inflight) { *done = 1; return PS_OK; }
  CU_TRY(cudaSetDevice(S->device));
  const cudaError_t e = cudaEventQuery(S->done_ev);
  if (e == cudaSuccess) { *done = 1; return PS_OK; }
  if (e == cudaErrorNotReady) { cudaGetLastError(); *done = 0; return PS_OK; }
  return fail(PS_E_CUDA, "ps_verify_query: %s", cudaGetErrorString(e));
}

// n greedy steps as a chain of forwards launched back to back: forward i > 0
// takes its row token from forward i - 1's result on the device (kFlagChainIn),
// so the host waits once for the chain instead of once per token.  Same
// forwards, same arithmetic and results as n single steps.
static ps_status draft_chain(ps_stage* S, int32_t n_steps, int32_t* out_tokens) {
  const long long n = (long long)S->tokens.size();
  ps_status st = catch_up(S, 1);
  if (st != PS_OK) return st;
  const long long kv0 = S->kv_len;
  const int row0 = (int)(n - 1 - kv0);
  int32_t rows[kMaxRows];
  for (int j = 0; j <= row0; ++j) rows[j] = S->tokens[kv0 + j];
  CU_TRY(cudaEventRecord(S->chain_ev[0], S->stream));
  for (int i = 0; i < n_steps; ++i) {
    const long long g = n + i - S->n_prompt;
    if (i == 0) st = forward_rows(S, rows, row0 + 1, kv0, 0, true, false, row0, nullptr, kFlagChainOut, 0, g);
    else st = forward_rows(S, rows, 1, n - 1 + i, 0, true, false, 0, nullptr, kFlagChainIn | kFlagChainOut, i, g);
    if (st != PS_OK) {
      cudaStreamSynchronize(S->stream);
      S->kv_len = 0;                     // KV state unknown: recompute on the next forward
      free_pages_from(S, 0);
      return st;
    }
  }
  CU_TRY(cudaEventRecord(S->chain_ev[1], S->stream));
  CU_TRY(cudaMemcpyAsync(S->h_chain, S->d_chain, (size_t)n_steps * 4, cudaMemcpyDeviceToHost, S->stream));
  CU_TRY(cudaStreamSynchronize(S->stream));
  {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, S->chain_ev[0], S->chain_ev[1]) == cudaSuccess) {
      S->last_fwd_ms = ms / n_steps;
      S->sum_fwd_ms += ms;
      S->n_fwd += n_steps;
    }
    cudaGetLastError();
  }
  const StepOut* r = S->h_out;           // the last forward's result
  const long long kv_end = n - 1 + n_steps;
  if (r->R == -1 || r->kv_len != kv_end)
    return fail(PS_E_CUDA, "corrupt chained draft result R=%d kv_len=%d (want %lld)", r->R, r->kv_len, kv_end);
  for (int i = 0; i < n_steps; ++i) {
    const int t = S->h_chain[i] & 0x7FFFFFFF;
    if (t < 0 || t >= S->vocab_full) return fail(PS_E_CUDA, "corrupt chained draft token %d", t);
    S->tokens.push_back(t);
    out_tokens[i] = t;
  }
  S->kv_len = kv_end;
  update_onpath(S);
  return PS_OK;
}

ps_status ps_draft(ps_stage* S, int32_t n_steps, int32_t* out_tokens) {
  if (!S || (n_steps > 0 && !out_tokens)) return fail(PS_E_INVALID, "NULL argument");
  PS_NOT_INFLIGHT(S);
  if (n_steps < 0) return fail(PS_E_INVALID, "n_steps < 0");
  CU_TRY(cudaSetDevice(S->device));
  const long long n = (long long)S->tokens.size();
  if (n_steps > 1 && n >= 1 && n - 1 + n_steps <= S->max_seq && S->kv_len <= n - 1) {
    for (int done = 0; done < n_steps;) {          // chains of up to kMaxChain forwards
      const int c = std::min(n_steps - done, kMaxChain);
      ps_status st = c > 1 ? draft_chain(S, c, out_tokens + done) : PS_OK;
      if (c == 1) {
        int32_t a, nxt;
        st = verify_host(S, nullptr, 0, &a, &nxt, nullptr);
        if (st == PS_OK) out_tokens[done] = nxt;
      }
      if (st != PS_OK) return st;
      done += c;
    }
    return PS_OK;
  }
  for (int i = 0; i < n_steps; ++i) {
    int32_t a, nxt;
    ps_status st = verify_host(S, nullptr, 0, &a, &nxt, nullptr);
    if (st != PS_OK) return st;
    out_tokens[i] = nxt;
  }
  return PS_OK;
}

ps_status ps_kv_rollback(ps_stage* S, int64_t keep) {
  if (!S) return fail(PS_E_INVALID, "NULL stage");
  PS_NOT_INFLIGHT(S);
  if (keep < 1 || keep > (int64_t)S->tokens.size())
    return fail(PS_E_CONTRACT, "rollback keep=%lld not in [1, len=%zu]", (long long)keep, S->tokens.size());
  S->tokens.resize((size_t)keep);
  S->kv_len = std::min<long long>(S->kv_len, keep - 1);
  free_pages_from(S, S->kv_len);
  update_onpath(S);
  return PS_OK;
}

ps_status ps_stage_tokens(const ps_stage* S, int32_t* out, int64_t cap, int64_t* len) {
  if (!S || !len || (cap > 0 && !out)) return fail(PS_E_INVALID, "NULL argument");
  const int64_t n = (int64_t)S->tokens.size();
  const int64_t m = std::min(cap, n);
  if (m > 0) memcpy(out, S->tokens.data(), (size_t)m * 4);
  *len = n;
  return PS_OK;
}

ps_status ps_stage_get_info(const ps_stage* S, ps_stage_info* info) {
  if (!S || !info) return fail(PS_E_INVALID, "NULL argument");
  memset(info, 0, sizeof *info);
  info->n_tokens = (int64_t)S->tokens.size();
  info->kv_len = S->kv_len;
  info->pages_in_use = pages_in_use(S);
  info->pages_total = S->pages_total;
  info->launches_per_verify = 1;   // one persistent megakernel per forward
  info->rows_buckets[0] = 16;
  info->rows_buckets[1] = 32;
  info->last_fwd_ms = S->last_fwd_ms;
  info->sum_fwd_ms = S->sum_fwd_ms;
  info->n_fwd = S->n_fwd;
  info->max_window = S->max_window;
  info->max_seq = S->max_seq;
  info->attn_sc = S->attn_sc;
  return PS_OK;
}

ps_status ps_stage_reset_timers(ps_stage* S) {
  if (!S) return fail(PS_E_INVALID, "NULL stage");
  S->sum_fwd_ms = 0;
  S->n_fwd = 0;
  return PS_OK;
}

ps_status ps_set_synthetic(ps_stage* S, const int32_t* Sv, int32_t len_S, int32_t n_prompt, int32_t level,
                           int32_t top, const double* alphas, uint64_t seed) {
  if (!S) return fail(PS_E_INVALID, "NULL stage");
  PS_NOT_INFLIGHT(S);
  CU_TRY(cudaSetDevice(S->device));
  CU_TRY(cudaStreamSynchronize(S->stream));
  if (S->d_S) { cudaFree(S->d_S); S->d_S = nullptr; }
  S->S_host.clear();
  S->h_syn = SynthParams{};
  if (len_S > 0) {
    if (!Sv || !alphas || level < 0 || top <= level || top > 8 || n_prompt < 0)
      return fail(PS_E_INVALID, "bad synthetic parameters");
    S->S_host.resize(len_S);
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, Sv) == cudaSuccess && at.type == cudaMemoryTypeDevice)
      CU_TRY(cudaMemcpy(S->S_host.data(), Sv, (size_t)len_S * 4, cudaMemcpyDeviceToHost));
    else
      memcpy(S->S_host.data(), Sv, (size_t)len_S * 4);
    cudaGetLastError();
    CU_TRY(cudaMalloc(&S->d_S, (size_t)len_S * 4));
    CU_TRY(cudaMemcpy(S->d_S, S->S_host.data(), (size_t)len_S * 4, cudaMemcpyHostToDevice));
    S->h_syn.S = S->d_S;
    S->h_syn.len_S = len_S;
    S->h_syn.level = level;
    S->h_syn.top = top;
    S->h_syn.vocab = S->vocab_full;
    S->h_syn.seed = seed;
    for (int j = level; j < top; ++j) {
      const double a = alphas[j - level];
      if (!(a >= 0.0 && a <= 1.0)) return fail(PS_E_INVALID, "alpha out of [0,1]");
      S->h_syn.thr[j] = (uint64_t)std::ldexp(a, 53);
    }
    S->n_prompt = n_prompt;
    S->onpath = 0;
    update_onpath(S);
  }
  CU_TRY(cudaMemcpy(S->d_syn, &S->h_syn, sizeof(SynthParams), cudaMemcpyHostToDevice));
  return PS_OK;
}

}  // extern "C"

#if PS_TRACE
extern "C" ps_status ps_trace_read(ps_stage* S, int32_t which, void* dst, int64_t bytes) {
  if (!S || !dst) return fail(PS_E_INVALID, "NULL argument");
  const void* src = nullptr;
  switch (which) {
    case 0: src = S->x; break;
    case 1: src = S->xg; break;
    case 2: src = S->q; break;
    case 3: src = S->att; break;
    case 4: src = S->h; break;
    case 5: src = S->ss; break;
    case 6: src = S->kv; break;
    case 7: src = S->attn_ml; break;
    case 8: src = S->d_page_table; break;
    case 9: src = S->mega_dbg; break;
    case 11: src = S->epi_dbg; break;
    case 10: src = S->attn_dbg; break;
    case 12: src = S->xch + S->off_part; break;
    default: return fail(PS_E_INVALID, "unknown buffer %d", which);
  }
  CU_TRY(cudaStreamSynchronize(S->stream));
  CU_TRY(cudaMemcpy(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost));
  return PS_OK;
}
#endif

extern "C" ps_status ps_pipeline_run(ps_stage* const* stages, int32_t k, const int32_t* prompt, int32_t n_prompt,
                                     const ps_run_opts* opts, int32_t* out, int32_t* out_len, ps_run_stats* stats);
