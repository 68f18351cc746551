// ps_mega.cuh — the whole verify forward as ONE persistent cooperative kernel.
//
// Batch-1 verification is a chain of ~5L+3 HBM-bound steps, each only a few
// microseconds long at the roofline; launched as separate kernels every step
// pays a launch, a prologue, a cold TMA pipeline and a drained tail.  Here one
// CTA per SM walks the phase table
//     EMBED, {QKV, ATTN, O, GATE/UP, DOWN} x L, [LM_HEAD, ARGMAX]
// with the same warp roles as the standalone GEMM:
//   warp 0      TMA producer: streams the weight tiles of every GEMM phase in
//               order through one STAGES-deep ring.  Weights do not depend on
//               activations, so it runs AHEAD across phase boundaries and only
//               the small activation tile of a stage waits for the previous
//               phase to complete (grid-wide counter, acquire) -- the HBM pipe
//               never drains between phases.
//   warp 1      TMEM owner + tcgen05.mma issuer (double-buffered accumulators).
//   warps 2-5   epilogues (stream-K fixup + fused epilogue), the attention
//               phase (mma.sync, 4 warps), embed and argmax/scan; after each
//               phase a CTA publishes completion with a release atomic.
// Phase completion counters are cumulative (target = gen * gridDim.x, gen
// from StepIn), so the graph-captured kernel needs no reset.  Cooperative
// launch guarantees every CTA is resident (the waits would deadlock otherwise).
#pragma once
#include "ps_kernels.cuh"

namespace ps {

enum { PH_EMBED = 0, PH_GEMM = 1, PH_ATTN = 2, PH_ARGMAX = 3, PH_ACOMB = 4, PH_TPRED = 5 };

struct MegaPhase {
  int kind;
  int gu;                          // GEMM: gate/up (two 64-row boxes per A tile)
  int head;                        // 1: runs only in forwards with lm_head (counter target gen_head)
  int xpub;                        // tensor parallel: peers read this phase's output (publish at sys scope)
  int xwait;                       // tensor parallel: also wait for every peer's previous phase
  const CUtensorMap* mA0;          // global-memory tensor maps (64-byte aligned)
  const CUtensorMap* mA1;
  const CUtensorMap* mA2;
  const CUtensorMap* mX;
  GemmParams g;
  AttnParams a;
  EmbedParams em;
  ArgmaxParams am;
  TpParams tp;
};

struct MegaParams {
  const MegaPhase* ph;
  int n_ph;
  const StepIn* step;
  unsigned* done;                  // [n_ph] cumulative CTA completion counters
  unsigned long long* dbg;         // PS_TRACE builds: [G][n_ph][8] %globaltimer stamps
  int tp_n;                        // tensor-parallel group size (1: none)
  const unsigned* peer_done[8];    // every rank's phase counters (peer memory for other ranks)
  int32_t* chain;                  // chained draft forwards' tokens (see kFlagChainIn / kFlagChainOut)
};

// Phase-wait poll back-off cap (ns; measured: 1024 +5-8%, 256 / 64 / 32 within noise).
constexpr unsigned kSpinCapNs = 64;

constexpr int kMegaThreads = 224;   // 7 warps: W producer, MMA, 4 epilogue, X loader
// ring depth per rows bucket (fills the SM's shared memory next to the 53 KB attention area)
// (RP = 64: the prefill bucket, 64 rows per forward, epilogues in 16-row chunks)
template <int RP> constexpr int mega_stages() { return RP == 16 ? 7 : RP == 32 ? 5 : 4; }
template <int RP> constexpr int epi_rows() { return RP < 32 ? RP : 32; }   // rows per epilogue pass (scratch)

template <int RP, int STAGES = mega_stages<RP>()>
struct MegaSmem {
  static constexpr int kMegaStages = STAGES;
  static constexpr int kABytes = 128 * 64 * 2;
  static constexpr int kXBytes = 2 * RP * 64 * 2;   // split-bf16 activation tiles: hi, then lo
  static constexpr int kOffX = kMegaStages * kABytes;
  static constexpr int kOffScratch = kOffX + kMegaStages * kXBytes;
  static constexpr int kOffRed = kOffScratch + 128 * (epi_rows<RP>() + 1) * 4;
  static constexpr int kOffRstd = kOffRed + 4 * RP * 8;
  static constexpr int kOffKvRow = kOffRstd + RP * 4;
  static constexpr int kOffAttn = (kOffKvRow + RP * 8 + 1023) / 1024 * 1024;   // TMA 128B-swizzle dst
  // the attention's S exchange lives in the activation slots (idle in an attention phase)
  static_assert(kMegaStages * kXBytes >= kAttnXAreaBytes, "attention Q fragments live in the X slots");
  static constexpr int kAttnBytes = attn_smem_bytes(4);
  static constexpr int kOffBar = kOffAttn + kAttnBytes;
  static constexpr int kOffMisc = kOffBar + (2 * kMegaStages + 4) * 8;
  static constexpr int kOffPhase = (kOffMisc + 64 + 127) / 128 * 128;   // MegaPhase copy (epilogue warps)
  static constexpr int kOffStep = kOffPhase + (int)((sizeof(MegaPhase) + 127) / 128 * 128);   // StepIn copy
  static constexpr int kBytes = kOffStep + (int)((sizeof(StepIn) + 127) / 128 * 128) + 1024;
};

PS_DEV unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
PS_DEV void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
PS_DEV unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
PS_DEV void fence_acquire_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// Poll with relaxed loads and a short back-off (a tight acquire spin from 148
// SMs hammers one L2 line and invalidates L1 on every poll), then acquire once.
PS_DEV void spin_until(const unsigned* p, unsigned target, unsigned cap = 256) {
  unsigned ns = 32, polls = 0;
  unsigned long long t0 = 0;
  while ((int)(ld_relaxed_u32(p) - target) < 0) {
    __nanosleep(ns);
    ns = ns < cap ? ns * 2 : cap;
    spin_check(polls, t0);
  }
  fence_acquire_gpu();
}
PS_DEV bool poll_ready(const unsigned* p, unsigned target) {
  if ((int)(ld_relaxed_u32(p) - target) < 0) return false;
  fence_acquire_gpu();
  return true;
}

// Attention K/V ring producer (one thread of the X-loader warp): this CTA's
// stream of 16-key stages of attention phase pa, each issued once its buffer
// is released by its consumer (warp w for slot w, arriving for all 4).  Stages whose keys are all below pos0
// go out immediately; the first one reaching the window's rows waits for the
// QKV phase (pa - 1) to be published grid-wide (its K/V rows are new).
template <int HD>
__device__ __noinline__ void attn_produce(const MegaParams& P, int pa, const AttnParams& p, uint8_t* ring,
                                          uint64_t* full, uint64_t* empty, uint32_t& seq, int cta, int ncta,
                                          unsigned tgt_head, unsigned tgt_body) {
  const AttnGeom gm(p);
  const int it0 = gm.first(cta, ncta), it_end = gm.first(cta + 1, ncta);
  AttnProducer u;
  attn_producer_init(p, gm, it0, it_end, u);
  const int pos0 = p.step->pos0;
  const uint32_t ring_u32 = smem_u32(ring), full_u32 = smem_u32(full);
  // The ring shares its shared memory with the stream-K staging of > 16-row
  // epilogues (every GEMM phase but QKV).  A CTA without units in the phases
  // just before this attention reaches it early, while its own epilogue warps
  // may still be in the phase before QKV: wait until that phase is published
  // grid-wide (then this CTA's epilogue is in QKV or later, which stages
  // nothing until the attention is consumed).  A CTA with units everywhere
  // gets here only after that point anyway.
  if (it0 < it_end && pa >= 2)
    spin_until(P.done + (pa - 2), P.ph[pa - 2].head ? tgt_head : tgt_body, kSpinCapNs);
  bool qkv_seen = false;
  while (u.more) {
    if (!qkv_seen && u.kbeg + (u.s + 1) * kAttnStep > pos0) {
      spin_until(P.done + (pa - 1), P.ph[pa - 1].head ? tgt_head : tgt_body, kSpinCapNs);
      fence_proxy_async_global();
      qkv_seen = true;
    }
    const int buf = seq % kAttnStages;
    mbar_wait(&empty[buf], ((seq / kAttnStages) & 1) ^ 1);
    attn_issue<HD>(p, ring_u32, full_u32, seq, u.row);
    ++seq;
    attn_producer_seek(p, gm, it_end, u);
  }
}

template <int RP, int STAGES = mega_stages<RP>()>
__global__ void __launch_bounds__(kMegaThreads, 1) mega_kernel(const __grid_constant__ MegaParams P) {
  using L = MegaSmem<RP, STAGES>;
  constexpr int kMegaStages = L::kMegaStages;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned, derived from smem_raw by an offset (keeps the shared
  // address space visible to the compiler: LDS/STS instead of generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sX = smem + L::kOffX;
  float* scratch = (float*)(smem + L::kOffScratch);
  unsigned long long* red = (unsigned long long*)(smem + L::kOffRed);
  float* rstd = (float*)(smem + L::kOffRstd);
  long long* kvrow = (long long*)(smem + L::kOffKvRow);
  uint8_t* attn_smem = smem + L::kOffAttn;
  uint64_t* afull = (uint64_t*)(attn_smem + kAttnStages * attn_stage_bytes<128>());   // attention ring barriers
  uint64_t* aempty = afull + kAttnStages;
  uint64_t* full = (uint64_t*)(smem + L::kOffBar);
  uint64_t* empty = full + kMegaStages;
  uint64_t* tfull = empty + kMegaStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(smem + L::kOffMisc);
  volatile int* flag = (volatile int*)(smem + L::kOffMisc + 4);
  MegaPhase* sph = (MegaPhase*)(smem + L::kOffPhase);
  StepIn* sstep = (StepIn*)(smem + L::kOffStep);

  constexpr int kTmemCols = 4 * RP;                     // 2 accumulators x N = 2 RP columns
  constexpr uint32_t kIdesc = idesc_bf16_f32<128, 2 * RP>();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, c = blockIdx.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMegaStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 128); }
    for (int s = 0; s < kAttnStages; ++s) { mbar_init(&afull[s], 1); mbar_init(&aempty[s], 4); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // phase ph is complete when all G CTAs of every forward that ran it so far
  // have published it: target = (#forwards containing ph) * G
  const unsigned tgt_body = (unsigned)P.step->gen * (unsigned)G;
  const unsigned tgt_head = (unsigned)P.step->gen_head * (unsigned)G;

  // Unit walk shared by the two TMA warps: fn(ph, Q, u, t, kb) for this CTA's
  // units of every GEMM phase, in ring order.
  auto for_units = [&](auto&& fn) {
    for (int ph = 0; ph < P.n_ph; ++ph) {
      const MegaPhase& Q = P.ph[ph];
      if (Q.kind != PH_GEMM) continue;
      const int kbt = Q.g.kb_total;
      const long long U = (long long)Q.g.n_tiles * kbt;
      const int Gp = (int)min((long long)min(G, Q.g.grid), U);
      if (c >= Gp) continue;
      const long long ub = sk_begin(U, Gp, c), ue = sk_begin(U, Gp, c + 1);
      for (long long u = ub; u < ue; ++u) fn(ph, Q, u, (int)(u / kbt), (int)(u % kbt));
    }
  };

  if (warp == 0) {
    // ================= W producer: weight tiles of every GEMM phase, never waits
    // on activations (weights do not depend on them), so it streams ahead across
    // phase boundaries as far as the ring allows.
    if (lane == 0) {
      uint32_t it = 0;
      int last_ph = -1;
      for_units([&](int ph, const MegaPhase& Q, long long, int t, int kb) {
        if (ph != last_ph) { tma_prefetch_desc(Q.mA0); last_ph = ph; }
        const int slot = it % kMegaStages;
        mbar_wait(&empty[slot], ((it / kMegaStages) & 1) ^ 1);
        uint8_t* dst = sA + slot * L::kABytes;
        mbar_arrive_expect_tx(&full[slot], L::kABytes + L::kXBytes);
        if (Q.gu) {
          tma_load_2d(dst, Q.mA0, &full[slot], kb * 64, t * 64, kEvictFirst);
          tma_load_2d(dst + 64 * 128, Q.mA1, &full[slot], kb * 64, t * 64, kEvictFirst);
        } else if (Q.g.mode == EPI_QKV) {
          if (t < Q.g.t1) tma_load_2d(dst, Q.mA0, &full[slot], kb * 64, t * 128, kEvictFirst);
          else if (t < Q.g.t2) tma_load_2d(dst, Q.mA1, &full[slot], kb * 64, (t - Q.g.t1) * 128, kEvictFirst);
          else tma_load_2d(dst, Q.mA2, &full[slot], kb * 64, (t - Q.g.t2) * 128, kEvictFirst);
        } else {
          tma_load_2d(dst, Q.mA0, &full[slot], kb * 64, t * 128, kEvictFirst);
        }
        ++it;
      });
    }
  } else if (warp == 6) {
    // ================= X loader: the activation tile of each unit, issued once
    // the whole previous phase has been published (grid-wide cumulative
    // counter: relaxed polls, one acquire, then a proxy fence so this CTA's
    // TMA (async proxy) sees the other CTAs' generic-proxy epilogue stores).
    if (lane == 0) {
      uint32_t it = 0, aseq = 0;
      int cur_ph = -1;
      for_units([&](int ph, const MegaPhase& Q, long long, int, int kb) {
        if (ph != cur_ph) {
          // attention phases between the last GEMM phase and this one: this
          // warp feeds their K/V ring (keys below pos0 at once, while QKV still
          // runs; the rest once QKV is published)
          for (int pa = cur_ph + 1; pa < ph; ++pa)
            if (P.ph[pa].kind == PH_ATTN) {
              const AttnParams& ap = P.ph[pa].a;
              if (ap.hd == 128) attn_produce<128>(P, pa, ap, attn_smem, afull, aempty, aseq, c, G, tgt_head, tgt_body);
              else attn_produce<64>(P, pa, ap, attn_smem, afull, aempty, aseq, c, G, tgt_head, tgt_body);
            }
          tma_prefetch_desc(Q.mX);
          cur_ph = ph;
          spin_until(P.done + (ph - 1), P.ph[ph - 1].head ? tgt_head : tgt_body, kSpinCapNs);
          fence_proxy_async_global();
          PS_TRACE_STAMP(P.dbg, ((size_t)c * P.n_ph + ph) * 8 + 2);
        }
        const int slot = it % kMegaStages;
        mbar_wait(&empty[slot], ((it / kMegaStages) & 1) ^ 1);
        // hi rows [0, RP) and lo rows [kRowsCap, kRowsCap + RP) of the operand
        tma_load_2d(sX + slot * L::kXBytes, Q.mX, &full[slot], kb * 64, 0, kEvictLast);
        tma_load_2d(sX + slot * L::kXBytes + RP * 128, Q.mX, &full[slot], kb * 64, kRowsCap, kEvictLast);
        ++it;
      });
      // attention phases after this CTA's last GEMM unit (none in the current
      // phase tables; kept so a CTA without later GEMM units still feeds them)
      for (int pa = cur_ph + 1; pa < P.n_ph; ++pa)
        if (P.ph[pa].kind == PH_ATTN) {
          const AttnParams& ap = P.ph[pa].a;
          if (ap.hd == 128) attn_produce<128>(P, pa, ap, attn_smem, afull, aempty, aseq, c, G, tgt_head, tgt_body);
          else attn_produce<64>(P, pa, ap, attn_smem, afull, aempty, aseq, c, G, tgt_head, tgt_body);
        }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    if (lane == 0) {
      uint32_t it = 0, nacc = 0;
      for (int ph = 0; ph < P.n_ph; ++ph) {
        const MegaPhase& Q = P.ph[ph];
        if (Q.kind != PH_GEMM) continue;
        const int kbt = Q.g.kb_total;
        const long long U = (long long)Q.g.n_tiles * kbt;
        const int Gp = (int)min((long long)min(G, Q.g.grid), U);
        if (c >= Gp) continue;
        const long long ub = sk_begin(U, Gp, c), ue = sk_begin(U, Gp, c + 1);
        long long u = ub;
        bool first = true;
        while (u < ue) {
          const int t = (int)(u / kbt);
          const long long seg_begin = u;
          const long long seg_end = min(ue, (long long)(t + 1) * kbt);
          const int acc = nacc & 1;
          mbar_wait(&tempty[acc], ((nacc >> 1) & 1) ^ 1);
#if PS_TRACE
          if (first) {
            mbar_wait(&full[it % kMegaStages], (it / kMegaStages) & 1);
            PS_TRACE_STAMP(P.dbg, ((size_t)c * P.n_ph + ph) * 8 + 3);
          }
#endif
          first = false;
          tc_fence_after();
          const uint32_t dcol = tmem + acc * 2 * RP;
          for (; u < seg_end; ++u, ++it) {
            const int slot = it % kMegaStages;
            mbar_wait(&full[slot], (it / kMegaStages) & 1);
            tc_fence_after();
            const uint32_t a0 = smem_u32(sA + slot * L::kABytes);
            const uint32_t x0 = smem_u32(sX + slot * L::kXBytes);
#pragma unroll
            for (int k = 0; k < 4; ++k)   // N = 2 RP: the hi and lo rows of the split operand in one MMA
              mma_bf16(dcol, smem_desc_sw128(a0 + 32 * k), smem_desc_sw128(x0 + 32 * k), kIdesc,
                       (u != seg_begin || k > 0) ? 1u : 0u);
            mma_commit(&empty[slot]);
          }
          mma_commit(&tfull[acc]);
          ++nacc;
        }
        PS_TRACE_STAMP(P.dbg, ((size_t)c * P.n_ph + ph) * 8 + 4);
      }
    }
  } else {
    // ================= epilogue / attention / embed / argmax (warps 2-5) =================
    const int et0 = threadIdx.x - 64;                  // 0..127 in warp order 2..5
    uint32_t nacc = 0;
    uint32_t attn_seq = 0;                             // attention ring stages consumed so far
    // StepIn -> smem once: every later read of the step (rows, positions,
    // generation, flags) in the epilogues / attention / argmax is a shared-
    // memory hit instead of a global round trip on a phase's critical path.
    {
      static_assert(sizeof(StepIn) % 4 == 0, "StepIn words");
      const int* src = reinterpret_cast<const int*>(P.step);
      int* dst = reinterpret_cast<int*>(sstep);
      for (int i = et0; i < (int)(sizeof(StepIn) / 4); i += 128) dst[i] = src[i];
      named_bar(1, 128);
      if (et0 == 0 && (sstep->flags & kFlagChainIn)) {   // row 0 = the previous chained forward's token
        const int v = __ldcg(P.chain + sstep->chain_idx - 1);
        sstep->tokens[0] = v & 0x7FFFFFFF;
        sstep->syn_onpath = (int)(((unsigned)v) >> 31);
      }
    }
    const StepIn* st = P.step;
    const int R = st->R;
    const int pos0 = st->pos0;
    for (int ph = 0; ph < P.n_ph; ++ph) {
      // per-thread indices re-read every phase (opaque to the compiler): values
      // derived from them are not hoisted out of the loop and kept live
      // across the attention call
      const int et = (int)opaque_tid_x() - 64;
      const int lane = et & 31;
      const int quarter = (et >> 5) ^ 2;               // warps 2..5 -> TMEM lane quarters 2, 3, 0, 1
      const int e = quarter * 32 + lane;
      // phase descriptor -> smem (one batch of 8-byte loads; every later
      // parameter access is a shared-memory hit instead of an L2 round trip)
      {
        const unsigned long long* src = reinterpret_cast<const unsigned long long*>(P.ph + ph);
        unsigned long long* dst = reinterpret_cast<unsigned long long*>(sph);
        constexpr int NW8 = (int)(sizeof(MegaPhase) / 8);
        for (int i = et; i < NW8; i += 128) dst[i] = src[i];
      }
      const int prev_head = ph > 0 ? P.ph[ph - 1].head : 0;
      // Wait for the whole previous phase (its outputs, and for QKV / gate-up
      // epilogues its row statistics); for a GEMM phase this is off the
      // critical path -- the first accumulator needs the X tiles, which the
      // X loader issues only after the same publication.
      named_bar(1, 128);
      if (et == 0) {   // the phase's step pointers -> the smem copy (read after the next barrier)
        sph->g.step = sstep;
        sph->a.step = sstep;
        sph->em.step = sstep;
        sph->am.step = sstep;
      }
      if (ph > 0 && et == 0) {
        spin_until(P.done + (ph - 1), prev_head ? tgt_head : tgt_body, kSpinCapNs);
        if (sph->xwait)           // tensor parallel: every peer's partial is published
          for (int q = 0; q < P.tp_n; ++q) spin_until_sys(P.peer_done[q] + (ph - 1), prev_head ? tgt_head : tgt_body);
      }
      named_bar(1, 128);
      if (et == 0) PS_TRACE_STAMP(P.dbg, ((size_t)c * P.n_ph + ph) * 8 + 0);
      const MegaPhase& Q = *sph;
      const int kind = Q.kind;
      if (kind == PH_EMBED) {
        for (int r = c; r < R; r += G) embed_row(Q.em, r, et);
      } else if (kind == PH_ATTN) {          // chunk partials; combined in the next phase
        // (the Q fragments use the X slots: during an attention phase this CTA's
        // previous GEMM phase is consumed, and the next one's X tiles load only
        // after the combine phase is published)
        const int nr = attn_nr(sstep->R * (Q.a.H / Q.a.hkv), sstep->pos0 + sstep->R);
        if (Q.a.hd == 128) {
          if (nr == 1) attn_run<128, 1>(Q.a, attn_smem, afull, aempty, sX, et, c, G, attn_seq);
          else if (nr == 2) attn_run<128, 2>(Q.a, attn_smem, afull, aempty, sX, et, c, G, attn_seq);
          else attn_run<128, 3>(Q.a, attn_smem, afull, aempty, sX, et, c, G, attn_seq);
        } else {
          if (nr == 1) attn_run<64, 1>(Q.a, attn_smem, afull, aempty, sX, et, c, G, attn_seq);
          else if (nr == 2) attn_run<64, 2>(Q.a, attn_smem, afull, aempty, sX, et, c, G, attn_seq);
          else attn_run<64, 3>(Q.a, attn_smem, afull, aempty, sX, et, c, G, attn_seq);
        }
      } else if (kind == PH_ACOMB) {
        if (Q.a.hd == 128) attn_combine<128>(Q.a, scratch, et, c, G);
        else attn_combine<64>(Q.a, scratch, et, c, G);
      } else if (kind == PH_TPRED) {
        const int nt = Q.tp.d >> 7;
        for (int u = c * 4 + (et >> 5); u < R * nt; u += G * 4) tp_reduce_unit(Q.tp, u / nt, u % nt, lane);
      } else if (kind == PH_ARGMAX) {
        if (c == 0) {
          argmax_run<128>(Q.am, et, (int*)scratch, 1);
          if (et == 0 && (sstep->flags & kFlagChainOut)) {   // (et 0 wrote out->next)
            const int nx = Q.am.out->next;
            const SynthParams* sp = Q.am.syn;
            const int g = sstep->syn_p0;
            const bool on = (sstep->flags & kFlagSynth) && sp != nullptr && sstep->syn_onpath && g >= 0 &&
                            g < sp->len_S && nx == sp->S[g];
            P.chain[sstep->chain_idx] = (int)((unsigned)nx | (on ? 0x80000000u : 0u));
          }
        }
      } else {
        const GemmParams& gp = Q.g;
        const int kbt = gp.kb_total;
        const long long U = (long long)gp.n_tiles * kbt;
        const int Gp = (int)min((long long)min(G, Q.g.grid), U);
        if (c < Gp) {
          epi_prepare<RP>(gp, e, R, pos0, scratch, rstd, kvrow);
          const long long ub = sk_begin(U, Gp, c), ue = sk_begin(U, Gp, c + 1);
          long long u = ub;
          while (u < ue) {
            const int t = (int)(u / kbt);
            const long long seg_begin = u;
            const long long seg_end = min(ue, (long long)(t + 1) * kbt);
            const int acc = nacc & 1;
            mbar_wait(&tfull[acc], (nacc >> 1) & 1);
            tc_fence_after();
            if (et == 0) {
              if (u == ub) PS_TRACE_STAMP(P.dbg, ((size_t)c * P.n_ph + ph) * 8 + 5);
              PS_TRACE_STAMP(P.dbg, ((size_t)c * P.n_ph + ph) * 8 + 6);
            }
            const uint32_t tacc = tmem + ((uint32_t)(quarter * 32) << 16) + acc * 2 * RP;
            if constexpr (RP <= 32) {
              float v[RP];
              load_acc<RP>(tacc, v);
              tc_fence_before();
              mbar_arrive(&tempty[acc]);
              ++nacc;
              u = seg_end;
              // (the attention area stages stream-K partials, except in QKV phases:
              // the next attention phase's K/V chunk is prefetched into it then)
              epi_segment<RP, true>(gp, t, seg_begin, seg_end, U, Gp, c, kbt, v, e, lane, quarter, R, pos0, scratch,
                                    red, rstd, kvrow, flag,
                                    gp.mode == EPI_QKV ? nullptr : reinterpret_cast<float4*>(attn_smem),
                                    kAttnStages * attn_stage_bytes<128>() / 16);   // not the ring barriers
            } else {
              // 64-row bucket: the epilogue in 16-row chunks (hi columns [16q, 16q + 16),
              // lo columns RP + 16q ..); the accumulator is released after the last chunk
              u = seg_end;
              for (int r0 = 0; r0 < R; r0 += 16) {
                float v[16], lo[16];
                tmem_ld16(tacc + r0, v);
                tmem_ld16(tacc + RP + r0, lo);
#pragma unroll
                for (int r = 0; r < 16; ++r) v[r] += lo[r];
                if (r0 + 16 >= R) {
                  tc_fence_before();
                  mbar_arrive(&tempty[acc]);
                }
                epi_segment<16, false>(gp, t, seg_begin, seg_end, U, Gp, c, kbt, v, e, lane, quarter,
                                       min(16, R - r0), pos0 + r0, scratch, red, rstd + r0, kvrow + r0, flag,
                                       nullptr, 0, r0);
              }
              ++nacc;
            }
            if (et == 0) PS_TRACE_STAMP(P.dbg, ((size_t)c * P.n_ph + ph) * 8 + 7);
          }
        }
      }
      // publish this CTA's completion of phase ph (release: orders all of the
      // CTA's phase writes, observed through the named barrier, before it)
      named_bar(1, 128);
      if (et == 0) {
        fence_proxy_async_global();
        if (Q.xpub) red_release_add_sys(P.done + ph, 1u);
        else red_release_add(P.done + ph, 1u);
        PS_TRACE_STAMP(P.dbg, ((size_t)c * P.n_ph + ph) * 8 + 1);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<kTmemCols>(tmem);
}

}  // namespace ps
