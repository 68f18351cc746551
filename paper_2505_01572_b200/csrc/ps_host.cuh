// ps_host.cuh — host helpers shared by the product library (ps_stage.cu) and
// the test library (ps_testlib.cu): errors, TMA descriptors, stream-K
// partitions, device setup.  Internal; not part of the ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>

#include "../../include/pipespec.h"
#include "ps_mega.cuh"

using namespace ps;

// ============================================================================ errors
// Each library defines its own thread-local error string and launch counter.
ps_status fail(ps_status code, const char* fmt, ...);
extern std::atomic<long long> g_launches;

#define CU_TRY(expr)                                                                       \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(PS_E_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

// ============================================================================ TMA maps
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static ps_status get_encoder() {
  if (g_encode) return PS_OK;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  CU_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) return fail(PS_E_CUDA, "cuTensorMapEncodeTiled not found");
  g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  return PS_OK;
}

// Row-major bf16 [rows, cols] matrix; box = box_rows x 64 columns, SWIZZLE_128B
// (128-byte rows, the canonical K-major UMMA layout).
static ps_status make_map(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  if (((uintptr_t)ptr & 15) || (cols * 2) % 16) return fail(PS_E_INVALID, "tensor not 16-byte aligned");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PS_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return PS_OK;
}

// The paged KV pool for the attention ring: [plane 4][rows][hd] bf16 viewed as
// a 3D tensor {hd, rows, plane} (the plane stride = one plane of one page's
// layer block: hkv * page_size rows), box {64, 16, 4}: one TMA moves 16 keys
// x 64 dims of all four planes (K_hi, K_lo, V_hi, V_lo), SWIZZLE_128B.
static ps_status make_map_kv(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t hd, uint64_t plane_rows) {
  if (((uintptr_t)ptr & 15) || (hd * 2) % 16) return fail(PS_E_INVALID, "KV pool not 16-byte aligned");
  cuuint64_t dims[3] = {hd, rows, 4};
  cuuint64_t strides[2] = {hd * 2, plane_rows * hd * 2};
  cuuint32_t box[3] = {64, 16, 4};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PS_E_CUDA, "cuTensorMapEncodeTiled (KV) failed (%d)", (int)r);
  return PS_OK;
}

// ============================================================================ GEMM launch
static int g_num_sms = 0;

struct GemmShape {
  int n_tiles, kb_total, grid, maxseg;
};

// Stream-K partition of one GEMM over the persistent grid.  align_pct > 0:
// if k = floor(#SMs / n_tiles) CTAs per tile keep >= align_pct% of the SMs
// busy, use n_tiles * k CTAs: every CTA then owns one tile-aligned segment
// and each tile exactly k partials.  Large models' phases are bandwidth-bound
// and take it at >= 95% (8B: QKV on 144 CTAs -0.25%; O / down on 128 CTAs
// would cost +1.4%; 80% +1.3%).  (Round 1 also aligned small models at 60%:
// 1B 0.940 -> 0.919 ms then; with round 2's kernels pure stream-K is 1% faster.)
static GemmShape gemm_shape(int n_tiles, int K, int num_sms, int align_pct = 0) {
  GemmShape g;
  g.n_tiles = n_tiles;
  g.kb_total = K / 64;
  long long U = (long long)n_tiles * g.kb_total;
  g.grid = (int)std::min<long long>(num_sms, U);
  if (align_pct > 0 && n_tiles <= num_sms) {
    // sk_begin splits at kb_total*c/k: tile-aligned for any k (<= kb_total: no empty CTA ranges)
    const int k = std::min(num_sms / n_tiles, g.kb_total);
    if ((long long)n_tiles * k * 100 >= (long long)num_sms * align_pct) g.grid = n_tiles * k;
  }
  auto owner = [&](long long u) { return (int)(((u + 1) * g.grid - 1) / U); };
  g.maxseg = 1;
  for (int t = 0; t < n_tiles; ++t) {
    int ns = owner((long long)t * g.kb_total + g.kb_total - 1) - owner((long long)t * g.kb_total) + 1;
    g.maxseg = std::max(g.maxseg, ns);
  }
  return g;
}

static ps_status init_device_globals(int device) {
  CU_TRY(cudaSetDevice(device));
  int major = 0, minor = 0;
  CU_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  CU_TRY(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
  if (major != 10 || minor != 0)
    return fail(PS_E_CUDA, "device %d is sm_%d%d; this library is built for sm_100a only", device, major, minor);
  CU_TRY(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, device));
  ps_status st;
  if ((st = get_encoder()) != PS_OK) return st;
  return PS_OK;
}

