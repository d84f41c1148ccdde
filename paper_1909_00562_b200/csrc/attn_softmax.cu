// attn_softmax.cu -- libattnsm.so: the C ABI of include/attn_softmax.h, the
// host planner (validation, workspace carving, TMA descriptors, V-chunk
// schedule, streams / events) and the kernel launches of the stage.
//
// Stage order (bf16 path, default options):
//   F1-F2  attention scores, masked softmax, context       Eqs. 1-3   attn_fwd_kernel
//   F3     proj_tanh  H_c = tanh([H|C] W_c^T)              Eq. 4      gemm_tc
//   F4     vocab_fwd  per-tile (max, sumexp) + target logit (logits not stored),
//          then lse_reduce                                 Eqs. 5-6   gemm_tc, lse_reduce_kernel
//   B1     one persistent launch: per V-chunk c the logits recomputed into
//          dL_c (L2 scratch), dHc += dL_c W_out[c], dW_out[c] = dL_c^T H_c   vocab_kernel
//   B1'    dz = dHc (1 - H_c^2)                                          dz_kernel
//   B2a    dC = dz W_c[:, d:], dW_c = dz^T [H|C] (split-K)               gemm_tc
//   B3     attention backward -> dQ, dH_enc                              attn_bwd_kernel
//   B2b    dH_dec = dz W_c[:, :d] + dQ                                   gemm_tc
//   X      dW_out chunks, dW_c, loss allreduced (comm != NULL)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <set>
#include <functional>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/attn_softmax.h"
#include "nvtx.cuh"
#include "../../include/attn_softmax_debug.h"
#include "comm.h"
#include "gemm_simt.cuh"
#include "gemm_tc.cuh"
#include "small_kernels.cuh"
#include "vocab.cuh"
#include "attn_tc.cuh"

using namespace attnsm;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;

static attn_status_t fail(attn_status_t code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(ATTN_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                  \
  } while (0)

extern "C" const char* attn_last_error(void) { return g_err.c_str(); }
attn_status_t attn_set_error(attn_status_t code, const char* msg) {
  g_err = msg;
  return code;
}
extern "C" const char* attn_version(void) { return "attnsm 0.1 sm_100a"; }

// ------------------------------------------------------------------ stage events / launch count
// Debug surface (attn_softmax_debug.h): when "stage_events" is on, the stage
// records a CUDA event on the caller's stream after each step so a harness
// can time every step of the path on the launching stream.
struct Prof {
  bool on = false;
  bool vocab_only = false;   // option value 2: only the marks around the vocab GEMMs
  bool created = false;
  int n = 0;
  cudaEvent_t ev[32];
  const char* name[32];
};
static Prof g_prof;
static long long g_launches = 0;

static void prof_mark(const char* name, cudaStream_t s, bool vocab_mark = false) {
  nvtxMarkA(name);   // end of stage `name` (host enqueue order)
  if (!g_prof.on || (g_prof.vocab_only && !vocab_mark)) return;
  if (!g_prof.created) {
    for (int i = 0; i < 32; ++i) cudaEventCreate(&g_prof.ev[i]);
    g_prof.created = true;
  }
  if (g_prof.n >= 32) return;
  cudaEventRecord(g_prof.ev[g_prof.n], s);
  g_prof.name[g_prof.n++] = name;
}

extern "C" int attn_softmax_stage_count(void) { return g_prof.n > 0 ? g_prof.n - 1 : 0; }

extern "C" attn_status_t attn_softmax_stage_time(int i, const char** name, float* ms) {
  if (i < 0 || i + 1 >= g_prof.n) return fail(ATTN_ERR_INVALID_ARG, "stage index %d out of range", i);
  CUDA_TRY(cudaEventSynchronize(g_prof.ev[i + 1]));
  float t = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&t, g_prof.ev[i], g_prof.ev[i + 1]));
  if (name) *name = g_prof.name[i + 1];
  if (ms) *ms = t;
  return ATTN_OK;
}

extern "C" long long attn_softmax_last_launches(void) { return g_launches; }

// ------------------------------------------------------------------ options
// GEMM groups, the bits of the wide_tiles option: forward vocab +
// projection, vocab backward chunks (stored-logits ablation), projection
// backward, the debug GEMM entry
enum : int { PAIR_FWD = 1, PAIR_VBWD = 2, PAIR_PBWD = 4, PAIR_DEBUG = 8 };
// debug_epilogue option: 0 = fp32 TMA store, 1 = accumulator read only (no store)
static int g_debug_epi = 0;
static int g_opt_mn3d = 1;  // MN-major operands via one 3D TMA box
// "wide_tiles": bitmask of GEMM groups on 256 x 256 single-CTA tiles; default
// the stored-logits ablation's vocab-backward launches
static int g_opt_wide = PAIR_VBWD;
// "db_gemm" (stored-logits ablation only): db_out summed by 0 column-sum
// kernels after each launch, 2 the dlogits kernels (default -1 = 2)
static int g_opt_db_gemm = -1;
constexpr int kEwParts = 320;   // row-group partial rows of the dlogits kernels' column sums
// "store_logits" (ABLATION, not the product path -- north_star forbids
// round-tripping the logits through HBM): the forward vocab GEMM also stores
// the logits as fp16 [T, V] and the backward turns each V-chunk into dL with
// an elementwise kernel; 1: chunk c+1's kernel beside launch c, 2: serialised.
// 0 (default): the persistent vocab kernel recomputes the logits per chunk.
static int g_opt_store_logits = 0;
// "dl_budget_mb": bytes of the dL chunk scratch (all NB buffers) the V-chunk
// width is sized to (an L2-sized budget; the dL lines are still written back
// to DRAM); "dl_buffers": NB
// 200 (C1: Vc = 5376, 10 chunks): re-measured with the final kernel (wide
// tiles, late claim, 48 KB stages) -- 2.09-2.17 vs 2.15-2.26 ms per step
// against 120 MB (Vc = 3072), alternating same-box pairs; C4 (Vc 4352 vs
// 2560) within noise, C3 unchanged (the 25-chunk cap sets Vc = 4096).  The
// dL lines reach DRAM anyway, so the L2-sized budget no
// longer decides
static int64_t g_opt_dl_budget_mb = 200;
static int g_opt_dl_nbuf = 3;
// "vb_last_g2_first": last block of the persistent backward dispatches the
// long dW_out tiles before the dHc tiles (shorter tail)
static int g_opt_vb_g2first = 1;
static long long* g_vb_trace = nullptr;   // "vb_trace": device buffer, 32 int64 per tile
// "vb_pair": the persistent vocab backward on CTA pairs (cta_group::2, 256 x 256 tiles)
static int g_opt_vb_pair = 1;
// "vb_order": dispatch blocks of the persistent vocab backward: 0 = [G3(c),
// G2(c), G1(c+1)]; 1 = [G1(c+1), G3(c), G2(c)] (chunk c's consumers run a
// whole G1 set after its producers; needs dl_buffers >= 3)
static int g_opt_vb_order = 1;
// order 2 (row-interleaved): "vb_lag" = row blocks between G1 and G3 of a row
// block, "vb_g2split" = G2 split over T in two row halves
static int g_opt_vb_lag = 2;
static int g_opt_vb_g2split = 1;
// "vb_claim": when a pair claims its next tile: 0 = right after the current
// tile's first load, 1 = two k-blocks before the end of its loads (default: a
// claimed tile never waits behind a long one; C1 vocab backward 1.57-1.59 ->
// 1.52 ms, two alternating same-box pairs), -1 = 1 for order 2 only
static int g_opt_vb_claim = 1;
// "vb_g1wide": G1 (dL) tiles 512 columns wide on CTA pairs (VbParams::g1wide)
static int g_opt_vb_g1wide = 0;
// "gemm_claim": bitmask of GEMM groups (the PAIR_* bits of "wide_tiles") whose
// tiles are claimed late (TcParams::claim_late).  Default: the projection
// backward (B2a's mix of 16- and 50-k-block tiles: 46.6 / 49.1 / 54.3 ->
// 41.0 / 43.9 / 45.5 us, alternating pairs); the uniform forward GEMMs were
// neutral to slightly slower
static int g_opt_gemm_claim = PAIR_PBWD;
static int g_vb_debug = 0;    // "vb_debug": timing experiments (vocab.cuh VbParams::debug)
static int g_opt_vb_wide = 1; // "vb_wide": 512-column G2 / G3 tiles on CTA pairs (VbParams::wide)
static int g_opt_vb_l2 = 3;   // "vb_l2hints": VbParams::l2hints
// "vb_fwd_fused": F4 + F5 inside the persistent launch (G0 tiles on CTA pairs,
// LSE by its warps 8-9) instead of the single-CTA forward GEMM + lse_reduce
// kernel before it (same-box C1: 2.28 vs 2.17 ms per step -- the power-capped
// clock runs lower under the pair tiles' forward)
static int g_opt_vb_fwd = 0;
// "n_fast": dispatch the vocab-backward GEMMs' column tiles of one row block
// back to back (their shared A block -- the dlogits chunk -- then leaves HBM once)
static int g_opt_n_fast = 1;
static int g_debug_skip_ew = 0;   // "debug_skip_dlogits": timing only -- skip the elementwise dlogits of chunks >= 1 (WRONG gradients)
static long long* g_trace = nullptr;   // "gemm_trace": device pointer of a per-tile trace buffer
static long long g_trace_launch = -1;  // "gemm_trace_launch": trace only this launch index of a call (-1 = all)
static int64_t g_opt_vocab_chunk = 0;
static int64_t g_opt_gemm_ctas = 0;
// "pdl": launch the bf16 path's kernels as programmatic dependents of the
// previous kernel (their prologue overlaps its tail; they griddepcontrol.wait
// before touching its results)
static int g_opt_pdl = 1;
// "attn_fused": the attention steps as one kernel per direction, one CTA per
// sentence (attn_tc.cuh; N, M <= 128, d % 64 == 0), else the generic engine's
// batched score / context GEMMs
static int g_opt_attn_fused = 1;
// "proj_bn": tile width of the Eq. 4 projection GEMM (K-major W_c allows
// 64, 128, 192, 256).  128 (400 tiles at C1, 2.7 waves on 148 SMs instead of
// 1.35) was measured slower: 43.6 vs 36.0 us (same box); 192: 43.3 us
static int g_opt_proj_bn = 256;
// "attn_trace": device buffer of globaltimer stamps, [2][B][16] int64 (forward,
// backward) + [B][64][4] backward chunk stamps (scripts/attn_trace.py)
static long long* g_attn_trace = nullptr;
namespace attnsm { extern long long* g_lstm_trace; }

// Options are read by a call from its start to its last enqueue under this
// lock (and written under it), so a concurrent set_option never changes a call
// in flight; recursive because entry points call each other.
static std::recursive_mutex g_opt_mu;
#define OPT_LOCK std::lock_guard<std::recursive_mutex> opt_lock_(g_opt_mu)

extern "C" attn_status_t attn_softmax_set_option(const char* key, int64_t value) {
  OPT_LOCK;
  if (!key) return fail(ATTN_ERR_INVALID_ARG, "set_option: key is NULL");
  if (!strcmp(key, "vocab_chunk")) {
    if (value < 0 || value % 256 != 0)
      return fail(ATTN_ERR_INVALID_ARG, "vocab_chunk must be a non-negative multiple of 256 (got %lld)",
                  (long long)value);
    g_opt_vocab_chunk = value;
    return ATTN_OK;
  }
  if (!strcmp(key, "gemm_trace_launch")) {
    g_trace_launch = value;
    return ATTN_OK;
  }
  if (!strcmp(key, "gemm_trace")) {
    g_trace = reinterpret_cast<long long*>(value);
    return ATTN_OK;
  }
  if (!strcmp(key, "debug_skip_dlogits")) {
    g_debug_skip_ew = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "n_fast")) {
    g_opt_n_fast = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "dl_budget_mb")) {
    if (value < 1) return fail(ATTN_ERR_INVALID_ARG, "dl_budget_mb must be >= 1");
    g_opt_dl_budget_mb = value;
    return ATTN_OK;
  }
  if (!strcmp(key, "dl_buffers")) {
    if (value < 1 || value > 4) return fail(ATTN_ERR_INVALID_ARG, "dl_buffers must be in [1, 4]");
    g_opt_dl_nbuf = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "vb_fwd_fused")) {
    g_opt_vb_fwd = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "vb_l2hints")) {
    g_opt_vb_l2 = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "vb_wide")) {
    g_opt_vb_wide = value != 0;
    return ATTN_OK;
  }
  if (!strcmp(key, "vb_debug")) {
    g_vb_debug = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "vb_order")) {
    if (value < 0 || value > 2) return fail(ATTN_ERR_INVALID_ARG, "vb_order must be 0, 1 or 2");
    g_opt_vb_order = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "vb_lag")) {
    if (value < 0 || value > 64) return fail(ATTN_ERR_INVALID_ARG, "vb_lag must be in [0, 64]");
    g_opt_vb_lag = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "gemm_claim")) {
    g_opt_gemm_claim = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "vb_g1wide")) {
    g_opt_vb_g1wide = value != 0;
    return ATTN_OK;
  }
  if (!strcmp(key, "vb_claim")) {
    g_opt_vb_claim = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "vb_g2split")) {
    g_opt_vb_g2split = value != 0;
    return ATTN_OK;
  }
  if (!strcmp(key, "vb_pair")) {
    g_opt_vb_pair = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "vb_trace")) {
    g_vb_trace = reinterpret_cast<long long*>(value);
    return ATTN_OK;
  }
  if (!strcmp(key, "vb_last_g2_first")) {
    g_opt_vb_g2first = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "store_logits")) {
    g_opt_store_logits = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "db_gemm")) {
    g_opt_db_gemm = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "wide_tiles")) {
    g_opt_wide = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "mn_3d_tma")) {
    g_opt_mn3d = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "debug_epilogue")) {
    g_debug_epi = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "stage_events")) {
    g_prof.on = value != 0;
    g_prof.vocab_only = value == 2;
    return ATTN_OK;
  }
  if (!strcmp(key, "comm_reserve_1rank")) {
    g_comm_reserve_1rank = value != 0;
    return ATTN_OK;
  }
  if (!strcmp(key, "comm_max_ctas")) {
    if (value < 0 || value > 64) return fail(ATTN_ERR_INVALID_ARG, "comm_max_ctas must be in [0, 64]");
    g_comm_max_ctas = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "pdl")) {
    g_opt_pdl = value != 0;
    return ATTN_OK;
  }
  if (!strcmp(key, "lstm_trace")) {
    attnsm::g_lstm_trace = reinterpret_cast<long long*>(value);
    return ATTN_OK;
  }
  if (!strcmp(key, "attn_trace")) {
    g_attn_trace = reinterpret_cast<long long*>(value);
    return ATTN_OK;
  }
  if (!strcmp(key, "proj_bn")) {
    if (value < 64 || value > 256 || value % 64) return fail(ATTN_ERR_INVALID_ARG, "proj_bn must be 64, 128, 192 or 256");
    g_opt_proj_bn = (int)value;
    return ATTN_OK;
  }
  if (!strcmp(key, "attn_fused")) {
    g_opt_attn_fused = value != 0;
    return ATTN_OK;
  }
  if (!strcmp(key, "gemm_ctas")) {
    if (value < 0) return fail(ATTN_ERR_INVALID_ARG, "gemm_ctas must be >= 0");
    g_opt_gemm_ctas = value;
    return ATTN_OK;
  }
  return fail(ATTN_ERR_INVALID_ARG, "unknown option '%s'", key);
}

// ------------------------------------------------------------------ device info
struct DevInfo {
  int sms = 148;
  size_t l2 = 126u << 20;
};
static DevInfo dev_info() {
  DevInfo d;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      d.sms = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev) == cudaSuccess && v > 0) d.l2 = v;
  }
  return d;
}

// ------------------------------------------------------------------ TMA maps
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

// rank-r tensor map, 128-byte swizzle, zero fill out of bounds.
// dt: 0 = bf16, 1 = fp32, 2 = fp16
static attn_status_t encode(CUtensorMap* m, const void* ptr, int dt, int rank,
                            const cuuint64_t* dims, const cuuint64_t* strides_bytes,
                            const cuuint32_t* box,
                            CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return fail(ATTN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(m, dt == 1 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                   : dt == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank,
                   const_cast<void*>(ptr), dims, strides_bytes, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(ATTN_ERR_CUDA,
                "cuTensorMapEncodeTiled failed (%d): rank %d ptr=%p dims=[%llu,%llu,%llu,%llu]",
                (int)r, rank, ptr, (unsigned long long)dims[0],
                (unsigned long long)(rank > 1 ? dims[1] : 0), (unsigned long long)(rank > 2 ? dims[2] : 0),
                (unsigned long long)(rank > 3 ? dims[3] : 0));
  return ATTN_OK;
}

// src_len[0..B) then tgt_len[0..B) (zeros when tgt is NULL) into dst[0..2B),
// as kernel parameters (capturable, no host staging; see lens_kernel).
static attn_status_t upload_lens(int* dst, const int32_t* src, const int32_t* tgt, int B,
                                 cudaStream_t stream) {
  for (int base = 0; base < 2 * B; base += 512) {
    LensChunk c;
    c.dst = dst + base;
    c.n = std::min(512, 2 * B - base);
    for (int i = 0; i < c.n; ++i) {
      const int k = base + i;
      c.vals[i] = k < B ? src[k] : (tgt ? tgt[k - B] : 0);
    }
    lens_kernel<<<1, 512, 0, stream>>>(c);
    CUDA_TRY(cudaGetLastError());
  }
  return ATTN_OK;
}

// ------------------------------------------------------------------ GEMM descriptions
// C[M,N] = A[M,K] B[N,K]^T per batch item.  A K-major operand is [rows, K]
// (row stride ld), an MN-major one [K, cols]; batch items are bstride
// elements apart.  k_ext is the operand's K extent (TMA zero-fills beyond
// it); mn_ext its M / N extent (rows for K-major, columns for MN-major).
struct Operand {
  const void* p = nullptr;
  long long ld = 0, bstride = 0, k_ext = 0, mn_ext = 0;
};
struct GemmDesc {
  int M = 0, N = 0, K = 0, batch = 1;
  int a_mn = 0, b_mn = 0;
  Operand a0, a1, b0, b1;
  int kseg = 0;      // two K segments: k-blocks [0,kseg) read a0/b0, the rest a1/(b1 if b_seg)
  int b_seg = 0;
  int b_nsplit = 0;  // MN-major B: columns >= b_nsplit come from b1
  int b_koff = 0;
  long long out_bstride = 0;   // batch stride of the epilogue output (elements)
  int bn = 0;        // tile columns (0 = 256); < 256 only for K-major B on single CTAs
  int n_fast = 0;    // dispatch the column tiles of a row block together (A read once via L2)
  EpiParams epi{};
};

static attn_status_t operand_map(CUtensorMap* m, const Operand& o, bool mn, int box_rows, int batch,
                                 int* mode, bool is_b = false) {
  const long long bs = batch > 1 ? o.bstride : (o.mn_ext + 1) * o.ld;
  if (!mn) {
    cuuint64_t dims[3] = {(cuuint64_t)std::max(1ll, o.k_ext), (cuuint64_t)std::max(1ll, o.mn_ext),
                          (cuuint64_t)batch};
    cuuint64_t st[2] = {(cuuint64_t)(o.ld * 2), (cuuint64_t)(bs * 2)};
    cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
    *mode = 0;
    return encode(m, o.p, false, 3, dims, st, box);
  }
  if (g_opt_mn3d && o.mn_ext % 64 == 0) {
    cuuint64_t dims[4] = {64, (cuuint64_t)std::max(1ll, o.k_ext), (cuuint64_t)(o.mn_ext / 64),
                          (cuuint64_t)batch};
    cuuint64_t st[3] = {(cuuint64_t)(o.ld * 2), 128, (cuuint64_t)(bs * 2)};
    cuuint32_t box[4] = {64, 64, (cuuint32_t)(box_rows / 64), 1};
    *mode = 1;
    return encode(m, o.p, false, 4, dims, st, box);
  }
  cuuint64_t dims[3] = {(cuuint64_t)std::max(1ll, o.mn_ext), (cuuint64_t)std::max(1ll, o.k_ext),
                        (cuuint64_t)batch};
  cuuint64_t st[2] = {(cuuint64_t)(o.ld * 2), (cuuint64_t)(bs * 2)};
  cuuint32_t box[3] = {64, 64, 1};
  *mode = 2;
  return encode(m, o.p, false, 3, dims, st, box);
}

// pair: 1 = 128 x 256 tiles, 4 = wide single CTA (256 rows, whole B tile)
static attn_status_t fill_tc(const GemmDesc& g, CUtensorMap* maps, TcProblem& pr, int tile_begin,
                             int pair) {
  memset(&pr, 0, sizeof(pr));
  const int bn = g.bn > 0 ? g.bn : TC_BN;
  // narrower tiles: K-major B only.  The generic epilogues need widths that
  // are multiples of 64 (160 and 224 were measured broken); the attention
  // softmax epilogues (tile width = the source positions rounded to 32) handle
  // any multiple of 32 up to 256
  const bool attn_epi = g.epi.kind == EPI_ATTN_SOFTMAX || g.epi.kind == EPI_ATTN_SOFTMAX_BWD;
  if (bn != TC_BN && (bn % (attn_epi ? 32 : 64) != 0 || bn > TC_BN || g.b_mn || g.b_nsplit))
    return fail(ATTN_ERR_UNSUPPORTED, "tile width %d: needs a multiple of %d and a K-major B", bn,
                attn_epi ? 32 : 64);
  const int tile_m = pair == 1 ? TC_BM : 2 * TC_BM;
  const int b_rows = bn;
  pr.M = g.M; pr.N = g.N; pr.K = g.K; pr.batch = g.batch;
  pr.bn = bn;
  pr.n_fast = g.n_fast && g_opt_n_fast;
  pr.tiles_m = (g.M + tile_m - 1) / tile_m;
  pr.tiles_n = (g.N + bn - 1) / bn;
  pr.kseg = g.kseg;
  pr.kb_total = g.kseg > 0 ? g.kseg + (int)((g.a1.k_ext + TC_BK - 1) / TC_BK)
                           : (g.K + TC_BK - 1) / TC_BK;
  pr.tile_begin = tile_begin;
  pr.a_mn = g.a_mn; pr.b_mn = g.b_mn;
  pr.b_seg = g.b_seg;
  pr.b_nsplit = g.b_nsplit;
  pr.b_koff = g.b_koff;
  pr.epi = g.epi;
  attn_status_t st;
  int mode0 = 0, mode1 = 0;
  if ((st = operand_map(&maps[0], g.a0, g.a_mn, TC_BM, g.batch, &mode0)) != ATTN_OK) return st;
  if (g.kseg > 0) {
    if ((st = operand_map(&maps[1], g.a1, g.a_mn, TC_BM, g.batch, &mode1)) != ATTN_OK) return st;
    if (mode1 != mode0) return fail(ATTN_ERR_UNSUPPORTED, "A segments need the same tile mode");
  } else {
    maps[1] = maps[0];
  }
  pr.a_mode = mode0;
  if ((st = operand_map(&maps[2], g.b0, g.b_mn, b_rows, g.batch, &mode0, true)) != ATTN_OK) return st;
  if (g.b_seg || g.b_nsplit) {
    if ((st = operand_map(&maps[3], g.b1, g.b_mn, b_rows, g.batch, &mode1, true)) != ATTN_OK) return st;
    if (mode1 != mode0) {
      // keep both halves on the per-atom path
      int m2;
      const int save = g_opt_mn3d;
      g_opt_mn3d = 0;
      st = operand_map(&maps[2], g.b0, g.b_mn, b_rows, g.batch, &m2);
      if (st == ATTN_OK) st = operand_map(&maps[3], g.b1, g.b_mn, b_rows, g.batch, &m2);
      g_opt_mn3d = save;
      if (st != ATTN_OK) return st;
      mode0 = m2;
    }
    if (g.b_nsplit && mode0 == 1 && g.b_nsplit % b_rows != 0) {
      int m2;
      const int save = g_opt_mn3d;
      g_opt_mn3d = 0;
      st = operand_map(&maps[2], g.b0, g.b_mn, b_rows, g.batch, &m2);
      if (st == ATTN_OK) st = operand_map(&maps[3], g.b1, g.b_mn, b_rows, g.batch, &m2);
      g_opt_mn3d = save;
      if (st != ATTN_OK) return st;
      mode0 = m2;
    }
  } else {
    maps[3] = maps[2];
  }
  pr.b_mode = mode0;
  // epilogue output: TMA store / reduce-add boxes of 32 rows x 128 bytes
  const int k = g.epi.kind;
  if (k == EPI_ATTN_SOFTMAX || k == EPI_ATTN_SOFTMAX_BWD) {
    // bf16 alpha / de [batch][rows, ldo] (box 32 x 32, 64-byte swizzle) and, for
    // the forward, the fp32 alpha stash [batch][rows, stash_ld] in maps[3]
    // (box 32 x 32, 128-byte swizzle; B has one segment, so maps[3] is free)
    cuuint64_t dims[3] = {(cuuint64_t)g.epi.ncols_store, (cuuint64_t)g.M, (cuuint64_t)g.batch};
    cuuint64_t strides[2] = {(cuuint64_t)(g.epi.ldo * 2), (cuuint64_t)(g.out_bstride * 2)};
    cuuint32_t box[3] = {32, 32, 1};
    if ((st = encode(&maps[4], g.epi.out, false, 3, dims, strides, box,
                     CU_TENSOR_MAP_SWIZZLE_64B)) != ATTN_OK)
      return st;
    if (k == EPI_ATTN_SOFTMAX) {
      if (g.b_seg || g.b_nsplit) return fail(ATTN_ERR_UNSUPPORTED, "softmax epilogue needs one B map");
      cuuint64_t d2[3] = {(cuuint64_t)g.epi.ncols_valid, (cuuint64_t)g.M, (cuuint64_t)g.batch};
      cuuint64_t s2[2] = {(cuuint64_t)(g.epi.stash_ld * 4),
                          (cuuint64_t)(g.epi.stash_ld * 4 * (long long)g.M)};
      if ((st = encode(&maps[3], g.epi.stash_f32, true, 3, d2, s2, box)) != ATTN_OK) return st;
    }
  } else if ((k != EPI_LSE || g.epi.out) && k != EPI_NONE && k != EPI_TOPK) {
    // (LSE with `out`: the fp16 logits of option store_logits)
    const bool f32 = epi_out_is_f32(k);
    const int esz = f32 ? 4 : 2;
    const long long bs = g.batch > 1 ? g.out_bstride : (long long)(g.M + 1) * g.epi.ldo;
    cuuint64_t dims[3] = {(cuuint64_t)g.epi.ncols_store, (cuuint64_t)g.M, (cuuint64_t)g.batch};
    cuuint64_t strides[2] = {(cuuint64_t)(g.epi.ldo * esz), (cuuint64_t)(bs * esz)};
    cuuint32_t box[3] = {(cuuint32_t)(f32 ? 32 : 64), 32, 1};
    if ((st = encode(&maps[4], g.epi.out, f32 ? 1 : k == EPI_LSE ? 2 : 0, 3, dims, strides, box)) !=
        ATTN_OK)
      return st;
  } else {
    maps[4] = maps[0];
  }
  return ATTN_OK;
}

// fp32 CUDA-core engine: same description, pointer + strides.
static void fill_simt(const GemmDesc& g, SimtProblem& pr, int tile_begin) {
  memset(&pr, 0, sizeof(pr));
  pr.M = g.M; pr.N = g.N; pr.K = g.K;
  pr.tiles_m = (g.M + SG_BM - 1) / SG_BM;
  pr.tiles_n = (g.N + SG_BN - 1) / SG_BN;
  pr.k_per_split = ((g.K + SG_BK - 1) / SG_BK) * SG_BK;
  pr.k_splits = 1;
  pr.tile_begin = tile_begin;
  pr.a0 = (const float*)g.a0.p;
  pr.a1 = g.kseg > 0 ? (const float*)g.a1.p : nullptr;
  pr.a_ksplit = (int)g.a0.k_ext;
  if (!g.a_mn) { pr.sam = g.a0.ld; pr.sak = 1; } else { pr.sam = 1; pr.sak = g.a0.ld; }
  pr.b0 = (const float*)g.b0.p;
  pr.b1 = g.b_nsplit ? (const float*)g.b1.p : nullptr;
  pr.b_nsplit = g.b_nsplit;
  pr.b_koff = g.b_koff;
  if (!g.b_mn) { pr.sbn = g.b0.ld; pr.sbk = 1; } else { pr.sbn = 1; pr.sbk = g.b0.ld; }
  pr.epi = g.epi;
}

static int tc_smem_bytes() { return TC_SMEM_BYTES; }

// Per-device "max dynamic shared memory" attribute of a kernel (set once per
// device, under a lock: the attribute belongs to the device's context).
template <typename K>
static attn_status_t ensure_smem_attr(K kernel, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;   // (kernel, device)
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  const void* key = reinterpret_cast<const void*>(kernel);
  std::lock_guard<std::mutex> lk(mu);
  for (auto& e : done)
    if (e.first == key && e.second == dev) return ATTN_OK;
  CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.emplace_back(key, dev);
  return ATTN_OK;
}



template <typename OutT, int kPair, bool kDecode = false>
static attn_status_t launch_tc_group_k(const GemmDesc* gs, int n, int* counter, cudaStream_t stream,
                                       int ctas = 0, int group_bit = 0) {
  attn_status_t st;
  if ((st = ensure_smem_attr(gemm_tc_kernel<OutT, true, kPair, kDecode>, tc_smem_bytes())) !=
      ATTN_OK)
    return st;
  TcParams P;
  memset(&P, 0, sizeof(P));
  int tiles = 0;
  for (int i = 0; i < n; ++i) {
    st = fill_tc(gs[i], P.maps[i], P.prob[i], tiles, kPair);
    if (st != ATTN_OK) return st;
    tiles += P.prob[i].tiles_m * P.prob[i].tiles_n * P.prob[i].batch;
  }
  P.nprob = n;
  P.total_tiles = tiles;
  P.tile_counter = counter;
  P.claim_late = (g_opt_gemm_claim & group_bit) ? 1 : 0;
  P.trace = (g_trace_launch < 0 || g_trace_launch == g_launches) ? g_trace : nullptr;
  if (tiles == 0) return ATTN_OK;
  const DevInfo di = dev_info();
  int units = ctas > 0 ? ctas : g_opt_gemm_ctas > 0 ? (int)g_opt_gemm_ctas : di.sms;
  units = std::max(1, std::min(units, tiles));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(units);
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = tc_smem_bytes();
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_opt_pdl ? 1 : 0;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<OutT, true, kPair, kDecode>, P));
  ++g_launches;
  return ATTN_OK;
}

// `group_bit` selects the bit of the "wide_tiles" option that puts this GEMM
// group on wide 256 x 256 tiles (0 = never); batched (attention) groups stay
// on 128 x 256 tiles (a sentence has <= 128 decoder rows).
template <typename OutT>
static attn_status_t launch_tc_group(const GemmDesc* gs, int n, int* counter, cudaStream_t stream,
                                     int group_bit = 0, int ctas = 0) {
  if (group_bit && (g_opt_wide & group_bit))
    return launch_tc_group_k<OutT, 4>(gs, n, counter, stream, ctas, group_bit);
  return launch_tc_group_k<OutT, 1>(gs, n, counter, stream, ctas, group_bit);
}

// Launch a plain kernel, as a programmatic dependent of the previous kernel
// when the "pdl" option is on (the kernel must pdl_wait() first).
template <typename... KArgs, typename... Args>
static attn_status_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t stream,
                                Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_opt_pdl ? 1 : 0;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
  ++g_launches;
  return ATTN_OK;
}

static attn_status_t launch_simt_group(const GemmDesc* gs, int n, cudaStream_t stream) {
  SimtParams P;
  memset(&P, 0, sizeof(P));
  int tiles = 0;
  for (int i = 0; i < n; ++i) {
    fill_simt(gs[i], P.prob[i], tiles);
    tiles += P.prob[i].tiles_m * P.prob[i].tiles_n * P.prob[i].k_splits;
  }
  P.nprob = n;
  if (tiles == 0) return ATTN_OK;
  gemm_simt_kernel<float><<<tiles, 256, 0, stream>>>(P);
  CUDA_TRY(cudaGetLastError());
  ++g_launches;
  return ATTN_OK;
}

// operand helpers: dense row-major [rows, cols] tensors
static Operand kmaj(const void* p, long long rows, long long k, long long ld, long long bstride = 0) {
  Operand o;
  o.p = p; o.ld = ld; o.bstride = bstride; o.k_ext = k; o.mn_ext = rows;
  return o;
}
static Operand mnmaj(const void* p, long long k_rows, long long mn_cols, long long ld,
                     long long bstride = 0) {
  Operand o;
  o.p = p; o.ld = ld; o.bstride = bstride; o.k_ext = k_rows; o.mn_ext = mn_cols;
  return o;
}

// ------------------------------------------------------------------ shapes / workspace
static size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

static attn_status_t check_shape(const attn_shape_t* s) {
  if (!s) return fail(ATTN_ERR_INVALID_ARG, "shape is NULL");
  if (s->dtype != ATTN_F32 && s->dtype != ATTN_BF16)
    return fail(ATTN_ERR_UNSUPPORTED, "dtype %d is not ATTN_F32 (0) or ATTN_BF16 (1)", (int)s->dtype);
  if (s->batch <= 0 || s->tgt_len <= 0 || s->src_len <= 0 || s->hidden <= 0 || s->vocab <= 0)
    return fail(ATTN_ERR_SHAPE,
                "shape [B=%d, N=%d, M=%d, d=%d, V=%d]: every extent must be >= 1", s->batch,
                s->tgt_len, s->src_len, s->hidden, s->vocab);
  const long long T = (long long)s->batch * s->tgt_len;
  if (T > (1ll << 30) || (long long)s->vocab > (1ll << 30) || s->hidden > (1 << 16))
    return fail(ATTN_ERR_UNSUPPORTED, "shape [B=%d, N=%d, d=%d, V=%d] exceeds the supported range",
                s->batch, s->tgt_len, s->hidden, s->vocab);
  if (s->dtype == ATTN_BF16 && s->hidden % 64 != 0)
    return fail(ATTN_ERR_UNSUPPORTED,
                "bf16 path needs hidden %% 64 == 0 (TMA / UMMA K blocks); got d=%d", s->hidden);
  if (s->dtype == ATTN_BF16 && s->src_len > 128)
    return fail(ATTN_ERR_UNSUPPORTED,
                "bf16 path needs M <= 128 source positions (one attention tile per sentence); "
                "got M=%d", s->src_len);
  return ATTN_OK;
}

constexpr int kNumCounters = 1024;
struct Plan {
  int B, N, M, d, V;
  long long T;
  bool bf16;
  size_t elt;
  int tileN;          // column tile of the vocab GEMM engine
  int ntn;            // column tiles over V
  int part_ld;        // LSE partial slots per row (tcgen05: 2 column halves per tile)
  int Vc;             // V-chunk width (multiple of 256)
  int nchunks;
  size_t off_lens, off_counters, off_blockpart, off_alpha, off_dalpha, off_ctx, off_hc, off_part,
      off_tgtlogit, off_lse, off_nll, off_rowscale, off_dl, off_dhc, off_dz, off_dhc2, off_abf,
      off_debf, off_q, off_dbpart, off_logits;
  int Mp;             // bf16 path: row stride of the bf16 alpha / de operands (64-multiple)
  int ald;            // row stride of the fp32 alpha stash (bf16 path: Mp, for TMA stores)
  bool store_logits;  // bf16 path, option store_logits: fp16 logits [T, Vld] in the workspace
  bool vb;            // bf16 path: persistent vocabulary launch (vocab.cuh)
  int nbuf;           // dL chunk buffers
  size_t off_vbctr, n_vbctr;   // its dependency counters (unsigned), zeroed per call
  long long Vld;
  size_t total;
};

// V-chunk width for the stored-logits backward on wide tiles: the balanced
// width (ceil(V / n) rounded up to 256) for the chunk count n in [2, 24] that
// minimises a model of the stage -- the persistent scheduler replayed on 148
// SMs (tiles in dispatch order, each SM takes the next tile when free; a wide
// tile costs 1024 cycles per 64-deep k-block + 8k epilogue + 1.5k boundary),
// + 35k cycles per launch (launch, prologue, and the visible share of the
// overlapped dlogits kernel, fitted), + chunk 0's serialised dlogits kernel
// (4 B per logit at 6 TB/s).  Its choices match the measured sweeps: C1
// 12544, C3 20224 (8.54-8.63 ms vs 8.97-9.09 at 10240), C4 10752 (4.78-4.88
// ms vs 5.10 at the old rule's 5376).  Deterministic in
// the shape (fixed SM count), so the workspace size does not depend on the
// device; memoised.
static long long model_chunk_width(long long T, long long d, long long V) {
  static std::mutex mu;
  static long long key[3] = {-1, -1, -1}, memo = 0;
  std::lock_guard<std::mutex> lock(mu);
  if (key[0] == T && key[1] == d && key[2] == V) return memo;
  const long long ntd = (d + 255) / 256, kbT = (T + 63) / 64;
  const double epi = 8000, bound = 1500, launch = 35000, clk = 1.9e9, bw = 6.0e12;
  std::vector<double> heap;
  double best = 1e300;
  long long best_vc = (V + 255) / 256 * 256;
  long long prev = -1;
  for (int n = 2; n <= 24; ++n) {
    const long long vc = ((V + n - 1) / n + 255) / 256 * 256;
    if (vc == prev || vc < 256) continue;
    prev = vc;
    double total = 0;
    for (long long c0 = 0; c0 < V; c0 += vc) {
      const long long vcc = std::min(vc, V - c0);
      heap.assign(148, 0.0);   // min-heap of SM finish times
      auto take = [&](double cost) {
        std::pop_heap(heap.begin(), heap.end(), std::greater<double>());
        heap.back() += cost;
        std::push_heap(heap.begin(), heap.end(), std::greater<double>());
      };
      const double tw = kbT * 1024.0 + epi + bound;                     // dW_out tile
      const double th = ((vcc + 63) / 64) * 1024.0 + epi + bound;       // dHc tile
      for (long long i = 0; i < ((vcc + 255) / 256) * ntd; ++i) take(tw);
      for (long long i = 0; i < ((T + 255) / 256) * ntd; ++i) take(th);
      total += *std::max_element(heap.begin(), heap.end()) + launch;
    }
    total += (double)std::min(vc, V) * T * 4.0 / bw * clk;
    if (total < best) { best = total; best_vc = vc; }
  }
  key[0] = T; key[1] = d; key[2] = V;
  memo = best_vc;
  return best_vc;
}

static size_t vb_ctr_words(const Plan& p);

static Plan make_plan(const attn_shape_t* s) {
  Plan p;
  p.B = s->batch; p.N = s->tgt_len; p.M = s->src_len; p.d = s->hidden; p.V = s->vocab;
  p.T = (long long)p.B * p.N;
  p.bf16 = s->dtype == ATTN_BF16;
  p.elt = p.bf16 ? 2 : 4;
  p.tileN = p.bf16 ? TC_BN : SG_BN;
  p.ntn = (p.V + p.tileN - 1) / p.tileN;
  p.part_ld = p.bf16 ? 2 * p.ntn : p.ntn;
  const long long vpad = (p.V + 255) / 256 * 256;
  long long vc = g_opt_vocab_chunk;
  p.store_logits = p.bf16 && g_opt_store_logits;
  p.vb = p.bf16 && !p.store_logits;
  p.nbuf = p.vb ? g_opt_dl_nbuf : 2;
  if (vc <= 0) {
    if (p.vb) {
      // the NB dL buffers [T, Vc] bf16 fit the L2 budget (DESIGN.md "V-chunk
      // schedule"), but at most 25 chunks: each chunk re-reads and re-writes
      // dHc [T, d] fp32, which outweighs L2 residency of dL at large T
      // (C3, T = 16384: 1280 -> 4096 columns, measured 8.77 -> 8.40 ms)
      vc = (g_opt_dl_budget_mb << 20) / ((long long)p.nbuf * p.T * 2) / 256 * 256;
      vc = std::max(vc, ((long long)(p.V + 24) / 25 + 255) / 256 * 256);
      vc = std::max(vc, 256ll);
    } else if (p.store_logits && (g_opt_wide & PAIR_VBWD)) {
      vc = model_chunk_width(p.T, p.d, p.V);
    } else {
      // fp32 path (and the stored-logits ablation on 128 x 256 tiles): about
      // 12 chunks per step
      vc = ((p.V + 11) / 12 + 255) / 256 * 256;
      vc = std::max(vc, 1024ll);
    }
  }
  vc = std::min(vc, vpad);
  // one tile counter per tcgen05 launch: keep the chunk count well inside
  while ((p.V + vc - 1) / vc > kNumCounters - 64) vc += 256;
  while (p.vb && (p.V + vc - 1) / vc > VB_MAX_BLOCKS - 1) vc += 256;
  p.Vc = (int)vc;
  p.nchunks = (int)((p.V + p.Vc - 1) / p.Vc);
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes); return r; };
  p.off_lens = take(2 * sizeof(int) * p.B);
  p.off_counters = take(sizeof(int) * kNumCounters);
  p.off_blockpart = take(sizeof(double) * ((p.T + 7) / 8 + 1));
  p.Mp = (p.M + 63) / 64 * 64;
  p.ald = p.bf16 ? p.Mp : p.M;
  p.off_alpha = take(sizeof(float) * p.T * p.ald);
  p.off_dalpha = take(sizeof(float) * p.T * p.M);
  p.off_ctx = take(p.elt * p.T * p.d);
  p.off_hc = take(p.elt * p.T * p.d);
  p.off_part = take(sizeof(float2) * p.T * p.part_ld);
  p.off_tgtlogit = take(sizeof(float) * p.T);
  p.off_lse = take(sizeof(float) * p.T);
  p.off_nll = take(sizeof(float) * p.T);
  p.off_rowscale = take(sizeof(float) * p.T);
  p.off_dl = take((size_t)std::max(2, p.nbuf) * p.elt * p.T * (size_t)p.Vc);
  p.off_dhc = take(sizeof(float) * p.T * p.d);
  p.off_dz = take(p.elt * p.T * p.d);
  p.off_dhc2 = take(sizeof(float) * p.T * 2 * p.d);
  p.off_abf = take(p.bf16 ? 2 * p.T * p.Mp : 0);
  p.off_debf = take(p.bf16 ? 2 * p.T * p.Mp : 0);
  p.off_q = take(p.elt * p.T * p.d);   // Eq. 2 general score: Q = H W_alpha
  // F_c bias: column-sum partials ([T/32][V] for the persistent launch's dL column sums)
  p.off_dbpart = take(sizeof(float) * std::max<size_t>(
      16 * (size_t)p.Vc, p.bf16 ? (size_t)std::max<long long>(kEwParts, (p.T + 31) / 32) * p.V : 0));
  p.Vld = (p.V + 7) / 8 * 8;
  p.off_logits = take(p.store_logits ? 2 * (size_t)p.T * p.Vld : 0);
  p.n_vbctr = p.vb ? vb_ctr_words(p) : 0;   // counters of the persistent vocabulary launch
  p.off_vbctr = take(sizeof(unsigned) * p.n_vbctr);
  p.total = o;
  return p;
}

extern "C" size_t attn_softmax_workspace_size(const attn_shape_t* s) {
  OPT_LOCK;
  if (check_shape(s) != ATTN_OK) return 0;
  return make_plan(s).total;
}

extern "C" attn_status_t attn_softmax_workspace_views(const attn_shape_t* s, attn_ws_views_t* out) {
  OPT_LOCK;
  attn_status_t st = check_shape(s);
  if (st != ATTN_OK) return st;
  if (!out) return fail(ATTN_ERR_INVALID_ARG, "out is NULL");
  Plan p = make_plan(s);
  out->alpha = p.off_alpha;
  out->alpha_ld = p.ald;
  out->ctx = p.off_ctx;
  out->hc = p.off_hc;
  out->lse = p.off_lse;
  out->nll = p.off_nll;
  out->vocab_chunk = p.Vc;
  return ATTN_OK;
}

// ------------------------------------------------------------------ attention (bgemm) launches
template <typename TA0, typename TB0, typename TA1, typename TB1, typename OutT>
static attn_status_t launch_bgemm(const BGemm<TA0, TB0, TA1, TB1, OutT>& g, cudaStream_t stream) {
  if (g.batch == 0 || g.M == 0 || g.N == 0) return ATTN_OK;
  dim3 grid((g.N + SG_BN - 1) / SG_BN, (g.M + SG_BM - 1) / SG_BM, g.batch);
  bgemm_kernel<TA0, TB0, TA1, TB1, OutT><<<grid, 256, 0, stream>>>(g);
  CUDA_TRY(cudaGetLastError());
  ++g_launches;
  return ATTN_OK;
}

template <typename T>
static attn_status_t attention_forward(const Plan& p, const T* H, const T* S, const int* src_len,
                                       float* alpha, T* ctx, cudaStream_t stream) {
  // F1: scores e_b = H_b S_b^T (Eq. 2, dot form)
  {
    BGemm<T, T, T, T, float> g{};
    g.batch = p.B; g.M = p.N; g.N = p.M; g.K0 = p.d; g.K1 = 0;
    g.s0 = {H, (long long)p.N * p.d, p.d, 1, S, (long long)p.M * p.d, p.d, 1};
    g.s1 = {H, 0, 0, 0, S, 0, 0, 0};
    g.out = alpha; g.sob = (long long)p.N * p.M; g.som = p.M; g.son = 1;
    attn_status_t st = launch_bgemm(g, stream);
    if (st != ATTN_OK) return st;
  }
  // Eq. 1: masked row softmax (in place)
  {
    const int rows = (int)p.T;
    softmax_fwd_kernel<<<(rows + 7) / 8, 256, 0, stream>>>(alpha, src_len, rows, p.N, p.M);
    CUDA_TRY(cudaGetLastError());
    ++g_launches;
  }
  // F2: C_b = alpha_b S_b (Eq. 3)
  {
    BGemm<float, T, float, T, T> g{};
    g.batch = p.B; g.M = p.N; g.N = p.d; g.K0 = p.M; g.K1 = 0;
    g.s0 = {alpha, (long long)p.N * p.M, p.M, 1, S, (long long)p.M * p.d, 1, p.d};
    g.s1 = {alpha, 0, 0, 0, S, 0, 0, 0};
    g.out = ctx; g.sob = (long long)p.N * p.d; g.som = p.d; g.son = 1;
    return launch_bgemm(g, stream);
  }
}

template <typename T>
static attn_status_t attention_backward(const Plan& p, const T* Q, const T* S, const float* alpha,
                                        float* dalpha, const float* dhc2, T* dH, T* dS, T* dq,
                                        cudaStream_t stream) {
  const long long ld2 = 2ll * p.d;
  const float* dC = dhc2 + p.d;   // columns [d, 2d) of [dH_part | dC]
  // dalpha_b = dC_b S_b^T
  {
    BGemm<float, T, float, T, float> g{};
    g.batch = p.B; g.M = p.N; g.N = p.M; g.K0 = p.d; g.K1 = 0;
    g.s0 = {dC, (long long)p.N * ld2, ld2, 1, S, (long long)p.M * p.d, p.d, 1};
    g.s1 = {dC, 0, 0, 0, S, 0, 0, 0};
    g.out = dalpha; g.sob = (long long)p.N * p.M; g.som = p.M; g.son = 1;
    attn_status_t st = launch_bgemm(g, stream);
    if (st != ATTN_OK) return st;
  }
  {
    const int rows = (int)p.T;
    softmax_bwd_kernel<<<(rows + 7) / 8, 256, 0, stream>>>(alpha, dalpha, rows, p.M);
    CUDA_TRY(cudaGetLastError());
    ++g_launches;
  }
  // dot score: dH_dec_b = dH_part_b + de_b S_b;  general score (dq != NULL):
  // dQ_b = de_b S_b (the caller adds dQ W_alpha^T to dH_part)
  {
    BGemm<float, T, float, T, T> g{};
    g.batch = p.B; g.M = p.N; g.N = p.d; g.K0 = p.M; g.K1 = 0;
    g.s0 = {dalpha, (long long)p.N * p.M, p.M, 1, S, (long long)p.M * p.d, 1, p.d};
    g.s1 = {dalpha, 0, 0, 0, S, 0, 0, 0};
    g.out = dq ? dq : dH; g.sob = (long long)p.N * p.d; g.som = p.d; g.son = 1;
    if (!dq) { g.add = dhc2; g.sadd_b = (long long)p.N * ld2; g.sadd_m = ld2; g.sadd_n = 1; }
    attn_status_t st = launch_bgemm(g, stream);
    if (st != ATTN_OK) return st;
  }
  // dH_enc_b = alpha_b^T dC_b + de_b^T H_b  (two K segments over the decoder rows)
  {
    BGemm<float, float, float, T, T> g{};
    g.batch = p.B; g.M = p.M; g.N = p.d; g.K0 = p.N; g.K1 = p.N;
    g.s0 = {alpha, (long long)p.N * p.M, 1, p.M, dC, (long long)p.N * ld2, 1, ld2};
    g.s1 = {dalpha, (long long)p.N * p.M, 1, p.M, Q, (long long)p.N * p.d, 1, p.d};
    g.out = dS; g.sob = (long long)p.M * p.d; g.som = p.d; g.son = 1;
    return launch_bgemm(g, stream);
  }
}

// ------------------------------------------------------------------ the stage
struct Bufs {
  int* src_len; int* tgt_len; unsigned int* counters; double* blockpart;
  float* alpha; float* dalpha; void* ctx; void* hc; float2* part; float* tgt_logit;
  float* lse; float* nll; float* rowscale; void* dl[2]; float* dhc; void* dz; float* dhc2;
  void* abf; void* debf; float* dhpart; void* dcbf;   // bf16 path
  float* dbpart;   // F_c bias: [16, Vc] column-sum partials (when not a GEMM)
  void* logits;    // option store_logits: fp16 [T, Vld]
  unsigned* vbctr; // persistent vocab backward: tile counter + dependency counters
  void* q;    // Eq. 2 general score: Q = H W_alpha [T, d] (dtype)
  void* dq;   // its gradient [T, d] (dtype); aliases dz, which is dead by then
  void* dq2;  // fused attention, dot score: dQ = de S bf16 [T, d] (the dH_part slot, unused then)
};

static Bufs carve(const Plan& p, void* ws) {
  char* w = (char*)ws;
  Bufs b;
  b.src_len = (int*)(w + p.off_lens);
  b.tgt_len = b.src_len + p.B;
  b.counters = (unsigned int*)(w + p.off_counters);
  b.blockpart = (double*)(w + p.off_blockpart);
  b.alpha = (float*)(w + p.off_alpha);
  b.dalpha = (float*)(w + p.off_dalpha);
  b.ctx = w + p.off_ctx;
  b.hc = w + p.off_hc;
  b.part = (float2*)(w + p.off_part);
  b.tgt_logit = (float*)(w + p.off_tgtlogit);
  b.lse = (float*)(w + p.off_lse);
  b.nll = (float*)(w + p.off_nll);
  b.rowscale = (float*)(w + p.off_rowscale);
  b.dl[0] = w + p.off_dl;
  b.dl[1] = w + p.off_dl + p.elt * p.T * (size_t)p.Vc;
  b.dhc = (float*)(w + p.off_dhc);
  b.dz = w + p.off_dz;
  b.dhc2 = (float*)(w + p.off_dhc2);
  b.abf = w + p.off_abf;
  b.debf = w + p.off_debf;
  b.dhpart = b.dhc2;                          // bf16 path: dH_part fp32 [T, d]
  b.dcbf = (char*)(b.dhc2 + p.T * p.d);       //            dC bf16 [T, d]
  b.q = w + p.off_q;
  b.dbpart = (float*)(w + p.off_dbpart);
  b.logits = p.store_logits ? w + p.off_logits : nullptr;
  b.vbctr = (unsigned*)(w + p.off_vbctr);
  b.dq = b.dz;
  b.dq2 = b.dhc2;
  return b;
}

static bool misaligned(const void* ptr) { return ptr && (reinterpret_cast<uintptr_t>(ptr) & 15); }

static attn_status_t validate(const attn_shape_t* s, const void* H_dec, const void* H_enc,
                              const int32_t* src_lens, const int32_t* tgt_lens,
                              const int32_t* tgt_ids, const void* W_c, const void* W_out,
                              const void* W_alpha, const float* loss, const void* dH_dec,
                              const void* dH_enc, const float* dW_c, const float* dW_out,
                              const float* dW_alpha, size_t ws_bytes, const void* ws) {
  attn_status_t st = check_shape(s);
  if (st != ATTN_OK) return st;
  struct { const void* p; const char* n; } req[] = {
      {H_dec, "H_dec"}, {H_enc, "H_enc"}, {src_lens, "src_lens_host"}, {tgt_lens, "tgt_lens_host"},
      {tgt_ids, "tgt_ids"}, {W_c, "W_c"}, {W_out, "W_out"}, {loss, "loss"}, {dH_dec, "dH_dec"},
      {dH_enc, "dH_enc"}, {dW_c, "dW_c"}, {dW_out, "dW_out"}, {ws, "workspace"}};
  for (auto& r : req)
    if (!r.p) return fail(ATTN_ERR_INVALID_ARG, "%s is NULL", r.n);
  if ((W_alpha == nullptr) != (dW_alpha == nullptr))
    return fail(ATTN_ERR_INVALID_ARG,
                "W_alpha and dW_alpha go together: both NULL (dot score, DESIGN.md R1) or both "
                "set (Eq. 2 general score); got W_alpha=%p dW_alpha=%p", W_alpha, (const void*)dW_alpha);
  long long total_tgt = 0;
  for (int b = 0; b < s->batch; ++b) {
    if (src_lens[b] < 1)
      return fail(ATTN_ERR_EMPTY_SOURCE, "src_lens_host[%d] = %d: every sentence needs >= 1 source position",
                  b, src_lens[b]);
    if (src_lens[b] > s->src_len)
      return fail(ATTN_ERR_SHAPE, "src_lens_host[%d] = %d exceeds the padded source length M = %d of "
                  "H_enc [%d, %d, %d]", b, src_lens[b], s->src_len, s->batch, s->src_len, s->hidden);
    if (tgt_lens[b] < 0 || tgt_lens[b] > s->tgt_len)
      return fail(ATTN_ERR_SHAPE, "tgt_lens_host[%d] = %d is outside [0, N = %d] of H_dec [%d, %d, %d]",
                  b, tgt_lens[b], s->tgt_len, s->batch, s->tgt_len, s->hidden);
    total_tgt += tgt_lens[b];
  }
  if (total_tgt == 0) return fail(ATTN_ERR_NO_TARGETS, "no valid target tokens (sum of tgt_lens_host is 0)");
  Plan p = make_plan(s);
  if (ws_bytes < p.total)
    return fail(ATTN_ERR_WORKSPACE, "workspace_bytes = %zu < required %zu", ws_bytes, p.total);
  if (s->dtype == ATTN_BF16) {
    const void* al[] = {H_dec, H_enc, W_c, W_out, dH_dec, dH_enc, dW_c, dW_out, ws, W_alpha,
                        dW_alpha};
    for (const void* a : al)
      if (misaligned(a)) return fail(ATTN_ERR_UNSUPPORTED, "bf16 path needs 16-byte aligned pointers");
  }
  return ATTN_OK;
}

// ---------------------------------------------------------------- GEMM plans
// Every GEMM of the stage, described once for both engines.  T = B*N rows.

// F3 (Eq. 4): H_c = tanh([H | C] W_c^T): two K segments (H, then C).
static GemmDesc g_proj(const Plan& p, const void* H, const void* ctx, const void* W_c, void* hc) {
  GemmDesc g;
  const int d = p.d;
  g.M = (int)p.T; g.N = d; g.K = 2 * d;
  g.a0 = kmaj(H, p.T, d, d);
  g.a1 = kmaj(ctx, p.T, d, d);
  g.kseg = (d + TC_BK - 1) / TC_BK;
  g.b0 = kmaj(W_c, d, 2 * d, 2 * d);
  g.bn = p.bf16 ? g_opt_proj_bn : 0;
  g.epi.kind = EPI_TANH; g.epi.out = hc; g.epi.ldo = d; g.epi.ncols_valid = d; g.epi.ncols_store = d;
  return g;
}
// F4 (Eq. 5): logits tile -> (max, sumexp) partials + target logit
static GemmDesc g_vocab_fwd(const Plan& p, const Bufs& b, const void* W_out, const int* tgt,
                            const void* b_out) {
  GemmDesc g;
  g.M = (int)p.T; g.N = p.V; g.K = p.d;
  g.a0 = kmaj(b.hc, p.T, p.d, p.d);
  g.b0 = kmaj(W_out, p.V, p.d, p.d);
  g.epi.kind = EPI_LSE; g.epi.ncols_valid = p.V; g.epi.ncols_store = p.V; g.epi.col_base = 0;
  g.epi.part = b.part; g.epi.part_ld = p.part_ld; g.epi.tgt_logit = b.tgt_logit; g.epi.tgt = tgt;
  g.epi.bias = b_out;
  if (p.store_logits) { g.epi.out = b.logits; g.epi.ldo = p.Vld; }
  return g;
}
// B1, chunk c: dlogits_c = rowscale (softmax - onehot) of the recomputed logits
static GemmDesc g_dlogits(const Plan& p, const Bufs& b, const void* W_out, const int* tgt, int c,
                          const void* b_out) {
  GemmDesc g;
  const int c0 = c * p.Vc, vcc = std::min(p.Vc, p.V - c0);
  g.M = (int)p.T; g.N = vcc; g.K = p.d;
  g.a0 = kmaj(b.hc, p.T, p.d, p.d);
  g.b0 = kmaj((const char*)W_out + (size_t)c0 * p.d * p.elt, vcc, p.d, p.d);
  g.epi.kind = EPI_DLOGITS; g.epi.out = b.dl[c & 1]; g.epi.ldo = p.Vc;
  g.epi.ncols_valid = vcc; g.epi.ncols_store = p.bf16 ? vcc : p.Vc; g.epi.col_base = c0;
  g.epi.lse = b.lse; g.epi.rowscale = b.rowscale; g.epi.tgt = tgt;
  g.epi.tgt_logit = b.tgt_logit;
  g.epi.bias = b_out;
  return g;
}
// B1, chunk c: dW_out[c] = dlogits_c^T H_c   (both operands MN-major)
static GemmDesc g_dwout(const Plan& p, const Bufs& b, float* dW_out, int c) {
  GemmDesc g;
  const int c0 = c * p.Vc, vcc = std::min(p.Vc, p.V - c0);
  g.M = vcc; g.N = p.d; g.K = (int)p.T;
  g.a_mn = 1; g.a0 = mnmaj(b.dl[c & 1], p.T, vcc, p.Vc);
  g.b_mn = 1; g.b0 = mnmaj(b.hc, p.T, p.d, p.d);
  g.epi.kind = EPI_STORE_F32; g.epi.out = dW_out + (size_t)c0 * p.d; g.epi.ldo = p.d;
  g.epi.ncols_valid = p.d; g.epi.ncols_store = p.d;
  g.n_fast = 1;
  return g;
}
// B1, chunk c: dHc (+)= dlogits_c W_out[c]   (B MN-major, K offset c0)
static GemmDesc g_dhc(const Plan& p, const Bufs& b, const void* W_out, int c) {
  GemmDesc g;
  const int c0 = c * p.Vc, vcc = std::min(p.Vc, p.V - c0);
  g.M = (int)p.T; g.N = p.d; g.K = vcc;
  g.a0 = kmaj(b.dl[c & 1], p.T, vcc, p.Vc);
  g.b_mn = 1; g.b0 = mnmaj(W_out, p.V, p.d, p.d); g.b_koff = c0;
  g.epi.kind = (c == 0) ? EPI_STORE_F32 : EPI_ACCUM_F32; g.epi.out = b.dhc; g.epi.ldo = p.d;
  g.epi.ncols_valid = p.d; g.epi.ncols_store = p.d;
  g.n_fast = 1;
  return g;
}
// B2: dW_c = dz^T [H | C]   (A MN-major, B MN-major split at column d)
static GemmDesc g_dwc(const Plan& p, const Bufs& b, const void* H, float* dW_c) {
  GemmDesc g;
  const int d = p.d;
  g.M = d; g.N = 2 * d; g.K = (int)p.T;
  g.a_mn = 1; g.a0 = mnmaj(b.dz, p.T, d, d);
  g.b_mn = 1; g.b0 = mnmaj(H, p.T, d, d); g.b1 = mnmaj(b.ctx, p.T, d, d); g.b_nsplit = d;
  g.epi.kind = EPI_STORE_F32; g.epi.out = dW_c; g.epi.ldo = 2ll * d;
  g.epi.ncols_valid = 2 * d; g.epi.ncols_store = 2 * d;
  return g;
}
// B2, split-K half `h` of dW_c (K = rows [k0, k1) of T): reduce-added into
// the zeroed dW_c (two addends onto 0: the sum is order-independent, exact
// IEEE commutativity, so deterministic)
static GemmDesc g_dwc_half(const Plan& p, const Bufs& b, const void* H, float* dW_c, int h) {
  GemmDesc g;
  const int d = p.d;
  // h = -1: one problem over all of T (small T)
  const long long mid = ((p.T / 2 + 63) / 64) * 64;
  const long long k0 = h == 1 ? mid : 0, k1 = h == 0 ? mid : p.T;
  const size_t off = (size_t)k0 * d * p.elt;
  g.M = d; g.N = 2 * d; g.K = (int)(k1 - k0);
  g.a_mn = 1; g.a0 = mnmaj((const char*)b.dz + off, k1 - k0, d, d);
  g.b_mn = 1; g.b0 = mnmaj((const char*)H + off, k1 - k0, d, d);
  g.b1 = mnmaj((const char*)b.ctx + off, k1 - k0, d, d); g.b_nsplit = d;
  g.epi.kind = EPI_ACCUM_F32; g.epi.out = dW_c; g.epi.ldo = 2ll * d;
  g.epi.ncols_valid = 2 * d; g.epi.ncols_store = 2 * d;
  return g;
}
// B2: dz W_c restricted to output columns [col0, col0 + ncol) (W_c MN-major)
static GemmDesc g_dzwc(const Plan& p, const Bufs& b, const void* W_c, int col0, int ncol,
                       int kind, void* out, long long ldo) {
  GemmDesc g;
  const int d = p.d;
  g.M = (int)p.T; g.N = ncol; g.K = d;
  g.a0 = kmaj(b.dz, p.T, d, d);
  g.b_mn = 1; g.b0 = mnmaj((const char*)W_c + (size_t)col0 * p.elt, d, ncol, 2ll * d);
  g.epi.kind = kind; g.epi.out = out; g.epi.ldo = ldo;
  g.epi.ncols_valid = ncol; g.epi.ncols_store = ncol;
  return g;
}

// Eq. 2 general score: Q = H W_alpha  (W_alpha [d,d] as MN-major B)
static GemmDesc g_query(const Plan& p, const Bufs& b, const void* H, const void* Wa) {
  GemmDesc g;
  const int d = p.d;
  g.M = (int)p.T; g.N = d; g.K = d;
  g.a0 = kmaj(H, p.T, d, d);
  g.b_mn = 1; g.b0 = mnmaj(Wa, d, d, d);
  g.epi.kind = p.bf16 ? EPI_STORE_BF16 : EPI_STORE_F32; g.epi.out = b.q; g.epi.ldo = d;
  g.epi.ncols_valid = d; g.epi.ncols_store = d;
  return g;
}
// its backward: dH_dec (+)= dQ W_alpha^T  (W_alpha K-major as stored)
static GemmDesc g_query_bwd_dh(const Plan& p, const Bufs& b, const void* Wa, void* dH, int kind) {
  GemmDesc g;
  const int d = p.d;
  g.M = (int)p.T; g.N = d; g.K = d;
  g.a0 = kmaj(b.dq, p.T, d, d);
  g.b0 = kmaj(Wa, d, d, d);
  g.epi.kind = kind; g.epi.out = dH; g.epi.ldo = d; g.epi.ncols_valid = d; g.epi.ncols_store = d;
  g.epi.addend = b.dhpart; g.epi.add_ld = d;
  return g;
}
// dW_alpha = H^T dQ  (both operands MN-major)
static GemmDesc g_query_bwd_dw(const Plan& p, const Bufs& b, const void* H, float* dWa) {
  GemmDesc g;
  const int d = p.d;
  g.M = d; g.N = d; g.K = (int)p.T;
  g.a_mn = 1; g.a0 = mnmaj(H, p.T, d, d);
  g.b_mn = 1; g.b0 = mnmaj(b.dq, p.T, d, d);
  g.epi.kind = EPI_STORE_F32; g.epi.out = dWa; g.epi.ldo = d; g.epi.ncols_valid = d;
  g.epi.ncols_store = d;
  return g;
}

// ---------------------------------------------------------------- fused attention kernels (attn_tc.cuh)
static bool attn_fused_ok(const Plan& p) {
  return g_opt_attn_fused && p.bf16 && p.N <= 128 && p.M <= 128 && p.d % 64 == 0;
}
// [B][rows][d] bf16 activations as a 3D map, box {64, box_rows, 1}
static attn_status_t map_rows3(CUtensorMap* m, const void* ptr, int d, int rows, int B, int box_rows) {
  cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)rows, (cuuint64_t)B};
  cuuint64_t str[2] = {(cuuint64_t)d * 2, (cuuint64_t)d * 2 * rows};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  return encode(m, ptr, 0, 3, dims, str, box);
}
template <typename P>
static attn_status_t launch_attn_k(void (*kernel)(P), const P& prm, int B, int smem, cudaStream_t stream) {
  attn_status_t st;
  if ((st = ensure_smem_attr(kernel, smem)) != ATTN_OK) return st;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(B);
  cfg.blockDim = dim3(AT_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_opt_pdl ? 1 : 0;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kernel, prm));
  ++g_launches;
  return ATTN_OK;
}
// F1 + Eq. 1 + F2 (Eqs. 1-3): alpha (fp32 stash + bf16 copy) and C
static attn_status_t attn_fused_fwd(const Plan& p, const void* Q, const void* S, const Bufs& b,
                                    cudaStream_t stream) {
  static AttnFwdParams P;   // large (5 tensor maps): filled under the option lock
  memset(&P, 0, sizeof(P));
  const int mbox = (p.M + 63) / 64 * 64, qrows = (p.N + 15) / 16 * 16;
  attn_status_t st;
  if ((st = map_rows3(&P.m_q, Q, p.d, p.N, p.B, qrows)) != ATTN_OK) return st;
  if ((st = map_rows3(&P.m_s, S, p.d, p.M, p.B, mbox)) != ATTN_OK) return st;
  if ((st = map_rows3(&P.m_c, b.ctx, p.d, p.N, p.B, 32)) != ATTN_OK) return st;
  {
    cuuint64_t dims[3] = {(cuuint64_t)p.M, (cuuint64_t)p.N, (cuuint64_t)p.B};
    cuuint64_t str[2] = {(cuuint64_t)p.ald * 4, (cuuint64_t)p.ald * 4 * p.N};
    cuuint32_t box[3] = {32, 32, 1};
    if ((st = encode(&P.m_stash, b.alpha, 1, 3, dims, str, box)) != ATTN_OK) return st;
  }
  {
    cuuint64_t dims[3] = {(cuuint64_t)p.Mp, (cuuint64_t)p.N, (cuuint64_t)p.B};
    cuuint64_t str[2] = {(cuuint64_t)p.Mp * 2, (cuuint64_t)p.Mp * 2 * p.N};
    cuuint32_t box[3] = {32, 32, 1};
    if ((st = encode(&P.m_abf, b.abf, 0, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B)) != ATTN_OK)
      return st;
  }
  P.src_len = b.src_len;
  P.d = p.d;
  P.mbox = mbox;
  P.qrows = qrows;
  P.store_abf = 0;   // the fused backward builds its bf16 alpha tile from the fp32 stash
  P.trace = g_attn_trace;
  return launch_attn_k(attn_fwd_kernel, P, p.B, ATF_SMEM, stream);
}
// B3: dQ = de S (bf16, into `dq`), dH_enc = alpha^T dC + de^T Q
static attn_status_t attn_fused_bwd(const Plan& p, const void* Q, const void* S, void* dq, void* dS,
                                    const Bufs& b, cudaStream_t stream) {
  static AttnBwdParams P;
  memset(&P, 0, sizeof(P));
  const int mbox = (p.M + 63) / 64 * 64, qrows = (p.N + 15) / 16 * 16;
  attn_status_t st;
  if ((st = map_rows3(&P.m_dc, b.dcbf, p.d, p.N, p.B, qrows)) != ATTN_OK) return st;
  if ((st = map_rows3(&P.m_s, S, p.d, p.M, p.B, mbox)) != ATTN_OK) return st;
  if ((st = map_rows3(&P.m_q, Q, p.d, p.N, p.B, qrows)) != ATTN_OK) return st;
  if ((st = map_rows3(&P.m_dq, dq, p.d, p.N, p.B, 32)) != ATTN_OK) return st;
  if ((st = map_rows3(&P.m_dhe, dS, p.d, p.M, p.B, 32)) != ATTN_OK) return st;
  P.alpha = b.alpha;
  P.N = p.N; P.M = p.M; P.d = p.d; P.ald = (int)p.ald; P.mbox = mbox; P.qrows = qrows;
  P.trace = g_attn_trace ? g_attn_trace + (long long)p.B * 16 : nullptr;
  return launch_attn_k(attn_bwd_kernel, P, p.B, ATB_SMEM, stream);
}

// ---------------------------------------------------------------- attention on tcgen05 (bf16)
// One small GEMM per sentence (batched problems; M <= 128 source positions).
static attn_status_t attention_forward_tc(const Plan& p, const void* H, const void* S, const Bufs& b,
                                          cudaStream_t stream, int* (*next)(void*), void* ctx_,
                                          const void* Wa) {
  const int d = p.d, N = p.N, M = p.M, Mp = p.Mp, B = p.B;
  // Eq. 2 general score: Q = H W_alpha (row form of H^T W_alpha), else Q = H
  const void* Q = H;
  if (Wa) {
    GemmDesc g = g_query(p, b, H, Wa);
    attn_status_t st = launch_tc_group<__nv_bfloat16>(&g, 1, next(ctx_), stream, PAIR_FWD);
    if (st != ATTN_OK) return st;
    Q = b.q;
  }
  if (attn_fused_ok(p)) return attn_fused_fwd(p, Q, S, b, stream);
  // F1 + Eq. 1: scores E_b = H_b S_b^T with the masked row softmax fused
  {
    GemmDesc g;
    g.batch = B; g.M = N; g.N = M; g.K = d;
    g.a0 = kmaj(Q, N, d, d, (long long)N * d);
    g.b0 = kmaj(S, M, d, d, (long long)M * d);
    g.bn = (M + 31) / 32 * 32;   // UMMA N = the source positions, not a 256-wide tile
    g.epi.kind = EPI_ATTN_SOFTMAX; g.epi.stash_f32 = b.alpha; g.epi.stash_ld = p.ald;
    g.epi.ncols_valid = M; g.out_bstride = (long long)N * Mp;
    g.epi.out = b.abf; g.epi.ldo = Mp; g.epi.ncols_store = Mp; g.epi.src_len = b.src_len;
    attn_status_t st = launch_tc_group<__nv_bfloat16>(&g, 1, next(ctx_), stream);
    if (st != ATTN_OK) return st;
  }
  // F2 (Eq. 3): C_b = alpha_b S_b   (S as MN-major B, K = source positions)
  GemmDesc g;
  g.batch = B; g.M = N; g.N = d; g.K = M;
  g.a0 = kmaj(b.abf, N, M, Mp, (long long)N * Mp);
  g.b_mn = 1; g.b0 = mnmaj(S, M, d, d, (long long)M * d);
  g.epi.kind = EPI_STORE_BF16; g.epi.out = b.ctx; g.epi.ldo = d; g.epi.ncols_valid = d;
  g.epi.ncols_store = d;
  g.out_bstride = (long long)N * d;
  return launch_tc_group<__nv_bfloat16>(&g, 1, next(ctx_), stream);
}

static attn_status_t attention_backward_tc(const Plan& p, const void* H, const void* S,
                                           void* dH, void* dS, const Bufs& b, cudaStream_t stream,
                                           int* (*next)(void*), void* ctx_, const void* Wa,
                                           float* dWa) {
  const int d = p.d, N = p.N, M = p.M, Mp = p.Mp, B = p.B;
  const void* Q = Wa ? b.q : H;
  if (attn_fused_ok(p)) {
    // dot score: dQ into b.dq2, added to dz W_c[:, :d] by the caller's second
    // projection-backward launch; general score: dQ into b.dq, then
    // dH_dec = dH_part + dQ W_alpha^T and dW_alpha = H^T dQ
    attn_status_t st = attn_fused_bwd(p, Q, S, Wa ? b.dq : b.dq2, dS, b, stream);
    if (st != ATTN_OK || !Wa) return st;
    GemmDesc ga[2] = {g_query_bwd_dh(p, b, Wa, dH, EPI_ADD_BF16), g_query_bwd_dw(p, b, H, dWa)};
    return launch_tc_group<__nv_bfloat16>(ga, 2, next(ctx_), stream, PAIR_PBWD);
  }
  // dalpha_b = dC_b S_b^T with the softmax backward fused: de (bf16)
  {
    GemmDesc g;
    g.batch = B; g.M = N; g.N = M; g.K = d;
    g.a0 = kmaj(b.dcbf, N, d, d, (long long)N * d);
    g.b0 = kmaj(S, M, d, d, (long long)M * d);
    g.bn = (M + 31) / 32 * 32;
    g.epi.kind = EPI_ATTN_SOFTMAX_BWD; g.epi.stash_f32 = b.alpha; g.epi.stash_ld = p.ald;
    g.epi.ncols_valid = M; g.out_bstride = (long long)N * Mp;
    g.epi.out = b.debf; g.epi.ldo = Mp; g.epi.ncols_store = Mp;
    attn_status_t st = launch_tc_group<__nv_bfloat16>(&g, 1, next(ctx_), stream);
    if (st != ATTN_OK) return st;
  }
  GemmDesc gs[2];
  // dQ_b = de_b S_b; dot score: dH_dec_b = dH_part_b + dQ_b (fused add),
  // general score: dQ stored, dH_dec = dH_part + dQ W_alpha^T below
  {
    GemmDesc& g = gs[0];
    g.batch = B; g.M = N; g.N = d; g.K = M;
    g.a0 = kmaj(b.debf, N, M, Mp, (long long)N * Mp);
    g.b_mn = 1; g.b0 = mnmaj(S, M, d, d, (long long)M * d);
    g.epi.ldo = d; g.epi.ncols_valid = d; g.epi.ncols_store = d;
    if (Wa) {
      g.epi.kind = EPI_STORE_BF16; g.epi.out = b.dq;
    } else {
      g.epi.kind = EPI_ADD_BF16; g.epi.out = dH; g.epi.addend = b.dhpart; g.epi.add_ld = d;
    }
    g.out_bstride = (long long)N * d;
  }
  // dH_enc_b = alpha_b^T dC_b + de_b^T H_b: two K segments over the decoder rows
  {
    GemmDesc& g = gs[1];
    g.batch = B; g.M = M; g.N = d; g.K = 2 * N;
    g.a_mn = 1;
    g.a0 = mnmaj(b.abf, N, Mp, Mp, (long long)N * Mp);
    g.a1 = mnmaj(b.debf, N, Mp, Mp, (long long)N * Mp);
    g.kseg = (N + TC_BK - 1) / TC_BK;
    g.b_mn = 1; g.b_seg = 1;
    g.b0 = mnmaj(b.dcbf, N, d, d, (long long)N * d);
    g.b1 = mnmaj(Q, N, d, d, (long long)N * d);
    g.epi.kind = EPI_STORE_BF16; g.epi.out = dS; g.epi.ldo = d; g.epi.ncols_valid = d;
    g.epi.ncols_store = d;
    g.out_bstride = (long long)M * d;
  }
  attn_status_t st = launch_tc_group<__nv_bfloat16>(gs, 2, next(ctx_), stream);
  if (st != ATTN_OK || !Wa) return st;
  // general score: dH_dec = dH_part + dQ W_alpha^T;  dW_alpha = H^T dQ
  GemmDesc ga[2] = {g_query_bwd_dh(p, b, Wa, dH, EPI_ADD_BF16), g_query_bwd_dw(p, b, H, dWa)};
  return launch_tc_group<__nv_bfloat16>(ga, 2, next(ctx_), stream, PAIR_PBWD);
}

// F4 + F5 + B1 as one launch (vocab.cuh): tensor maps, dispatch blocks,
// counters.  Counter layout in `ctr` (zeroed by the caller): [0] tile
// counter, [1] g5count (LSE CTA-portions), then g0done [nrb], lsedone [nrb], rowdone
// [nchunks][nrb], coldone [nchunks][2][ncolf], consumed [nchunks][2], g2done
// [nchunks], dhcdone [nrb][ndt], g2part [nchunks][n2max], and blockpart (double [nrb * CTAS]) at the
// end, 8-byte aligned (vb_ctr_layout).
struct VbLayout {
  int TM, nrb, ndt, ncolf;
  size_t g0done, lsedone, rowdone, coldone, consumed, g2done, dhcdone, g2part, blockpart, total;
  int n2max;
};
static VbLayout vb_ctr_layout(const Plan& p, bool pair) {
  VbLayout L;
  L.TM = pair ? 256 : 128;
  L.nrb = (int)((p.T + L.TM - 1) / L.TM);
  L.ndt = (p.d + VB_BN - 1) / VB_BN;
  L.ncolf = p.Vc / VB_BN;
  const size_t nch = p.nchunks;
  L.g0done = 2;
  L.lsedone = L.g0done + L.nrb;
  L.rowdone = L.lsedone + L.nrb;
  L.coldone = L.rowdone + nch * L.nrb;
  L.consumed = L.coldone + 2 * nch * L.ncolf;          // [nchunks][row half][ncolf]
  L.g2done = L.consumed + 2 * nch;                     // consumed: [nchunks][row half]
  L.dhcdone = L.g2done + nch;
  L.n2max = (int)((p.Vc + L.TM - 1) / L.TM) * L.ndt;   // G2 tiles of a chunk (narrow: upper bound)
  L.g2part = L.dhcdone + (size_t)L.nrb * L.ndt;
  L.blockpart = (L.g2part + nch * L.n2max + 1) & ~(size_t)1;   // in unsigned units
  L.total = L.blockpart + 2 * (size_t)L.nrb * (pair ? 2 : 1);
  return L;
}
// unsigned words of the counter region, for the larger (single-CTA) layout
static size_t vb_ctr_words(const Plan& p) { return vb_ctr_layout(p, false).total; }

struct VbArgs {
  const void* hc; const void* W_out; void* dl; float* dhc; float* dW_out;
  float2* part; int part_ld; float* tgt_logit; float* lse; float* nll; float* rowscale;
  float* loss; float loss_scale; const int* tgt; const int* tgt_len; const void* bias;
  float* db_part; unsigned* ctr;
  bool fwd;   // F4 + F5 in this launch (else lse / rowscale / tgt_logit are inputs)
};

template <bool kPair>
static attn_status_t launch_vocab_k(const Plan& p, const VbArgs& a, int ctas, cudaStream_t stream) {
  using Cfg = VbCfg<kPair>;
  attn_status_t st;
  if ((st = ensure_smem_attr(vocab_kernel<kPair>, VB_SMEM_BYTES)) != ATTN_OK) return st;
  static VbParams P;   // large (blk_start): filled per call under the lock
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  memset(&P, 0, sizeof(P));
  const long long T = p.T, d = p.d, V = p.V, Vc = p.Vc, NB = p.nbuf;
  const cuuint32_t brows = Cfg::B_ROWS;
  {   // H_c [T, d]: K-major A of G0 / G1
    cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)T, 1};
    cuuint64_t str[2] = {(cuuint64_t)(d * 2), (cuuint64_t)(T * d * 2)};
    cuuint32_t box[3] = {64, 128, 1};
    if ((st = encode(&P.m_hc_k, a.hc, 0, 3, dims, str, box)) != ATTN_OK) return st;
  }
  {   // W_out [V, d]: K-major B of G0 / G1
    cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)V, 1};
    cuuint64_t str[2] = {(cuuint64_t)(d * 2), (cuuint64_t)(V * d * 2)};
    cuuint32_t box[3] = {64, brows, 1};
    if ((st = encode(&P.m_wo_k, a.W_out, 0, 3, dims, str, box)) != ATTN_OK) return st;
  }
  {   // dL [NB][T][Vc]: K-major A of G3
    cuuint64_t dims[3] = {(cuuint64_t)Vc, (cuuint64_t)T, (cuuint64_t)NB};
    cuuint64_t str[2] = {(cuuint64_t)(Vc * 2), (cuuint64_t)(T * Vc * 2)};
    cuuint32_t box[3] = {64, 128, 1};
    if ((st = encode(&P.m_dl_k, a.dl, 0, 3, dims, str, box)) != ATTN_OK) return st;
  }
  {   // W_out as [K = V][N = d] MN-major: 64-column atoms 128 bytes apart
    cuuint64_t dims[4] = {64, (cuuint64_t)V, (cuuint64_t)(d / 64), 1};
    cuuint64_t str[3] = {(cuuint64_t)(d * 2), 128, (cuuint64_t)(V * d * 2)};
    cuuint32_t box[4] = {64, 64, brows / 64, 1};
    if ((st = encode(&P.m_wo_mn, a.W_out, 0, 4, dims, str, box)) != ATTN_OK) return st;
  }
  {   // dL as [K = T][M = Vc] MN-major per buffer
    cuuint64_t dims[4] = {64, (cuuint64_t)T, (cuuint64_t)(Vc / 64), (cuuint64_t)NB};
    cuuint64_t str[3] = {(cuuint64_t)(Vc * 2), 128, (cuuint64_t)(T * Vc * 2)};
    cuuint32_t box[4] = {64, 64, 2, 1};
    if ((st = encode(&P.m_dl_mn, a.dl, 0, 4, dims, str, box)) != ATTN_OK) return st;
  }
  {   // H_c as [K = T][N = d] MN-major
    cuuint64_t dims[4] = {64, (cuuint64_t)T, (cuuint64_t)(d / 64), 1};
    cuuint64_t str[3] = {(cuuint64_t)(d * 2), 128, (cuuint64_t)(T * d * 2)};
    cuuint32_t box[4] = {64, 64, brows / 64, 1};
    if ((st = encode(&P.m_hc_mn, a.hc, 0, 4, dims, str, box)) != ATTN_OK) return st;
  }
  {   // dL store: bf16 boxes of 32 rows x 64 columns
    cuuint64_t dims[3] = {(cuuint64_t)Vc, (cuuint64_t)T, (cuuint64_t)NB};
    cuuint64_t str[2] = {(cuuint64_t)(Vc * 2), (cuuint64_t)(T * Vc * 2)};
    cuuint32_t box[3] = {64, 32, 1};
    if ((st = encode(&P.m_dl_st, a.dl, 0, 3, dims, str, box)) != ATTN_OK) return st;
  }
  {   // dW_out fp32 [V, d] and dHc fp32 [T, d]: boxes of 32 x 32
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)V};
    cuuint64_t str[1] = {(cuuint64_t)(d * 4)};
    cuuint32_t box[2] = {32, 32};
    if ((st = encode(&P.m_dw_st, a.dW_out, 1, 2, dims, str, box)) != ATTN_OK) return st;
    cuuint64_t dims2[2] = {(cuuint64_t)d, (cuuint64_t)T};
    if ((st = encode(&P.m_dhc_st, a.dhc, 1, 2, dims2, str, box)) != ATTN_OK) return st;
  }
  const VbLayout L = vb_ctr_layout(p, kPair);
  P.T = (int)T; P.d = (int)d; P.V = (int)V; P.Vc = (int)Vc; P.nchunks = p.nchunks;
  P.nbuf = (int)NB;
  P.N = p.N;
  P.nrb = L.nrb;
  P.ndt = L.ndt;
  P.ncolf = L.ncolf;
  P.wide = (kPair && g_opt_vb_wide && d % 512 == 0) ? 1 : 0;
  P.ndw = P.wide ? L.ndt / 2 : L.ndt;
  P.ntn = (int)((V + VB_BN - 1) / VB_BN);
  P.fwd_tiles = a.fwd ? P.nrb * P.ntn : 0;
  P.last_g2_first = g_opt_vb_g2first;
  // order 1 with one buffer would wait on later tiles; order 2 reuses the
  // buffer per row half, whose consumers are dispatched in the previous block
  P.order = (NB >= 2 || g_opt_vb_order == 2) ? g_opt_vb_order : 0;
  P.nh = (P.order == 2 && g_opt_vb_g2split && P.nrb >= 2) ? 2 : 1;
  P.h0 = P.nh == 2 ? (P.nrb + 1) / 2 : P.nrb;
  P.lag = g_opt_vb_lag;
  // vb_claim: -1 = late for order 2 only, 0 = early, 1 = late (two k-blocks
  // before the end), k >= 2 = k k-blocks before the end
  P.claim_late = g_opt_vb_claim < 0 ? (P.order == 2 ? 2 : 0)
                                    : g_opt_vb_claim == 1 ? 2 : g_opt_vb_claim;
  P.g1wide = (kPair && g_opt_vb_g1wide) ? 1 : 0;
  const int g1w = P.g1wide ? 2 * VB_BN : VB_BN;   // G1 tile columns
  P.n2max = L.n2max;
  P.trace = g_vb_trace;
  P.debug = g_vb_debug;
  P.l2hints = g_opt_vb_l2;
  // backward dispatch blocks: 0 = G1(0); c + 1 = G1(c + 1), G3(c), G2(c)
  auto vcc = [&](int c) { return (int)std::min(Vc, V - (long long)c * Vc); };
  int t = 0;
  if (P.order == 2) {   // block c = chunk c: G1(c), G3(c), nh x G2(c)
    for (int c = 0; c < p.nchunks; ++c) {
      P.blk_start[c] = t;
      t += P.nrb * ((vcc(c) + g1w - 1) / g1w) + P.nrb * P.ndw +
           P.nh * ((vcc(c) + Cfg::TM - 1) / Cfg::TM) * P.ndw;
    }
    P.blk_start[p.nchunks] = t;
  } else {
    P.blk_start[0] = 0;
    t += P.nrb * ((vcc(0) + g1w - 1) / g1w);
    for (int c = 0; c < p.nchunks; ++c) {
      P.blk_start[c + 1] = t;
      t += P.nrb * P.ndw + ((vcc(c) + Cfg::TM - 1) / Cfg::TM) * P.ndw;
      if (c + 1 < p.nchunks) t += P.nrb * ((vcc(c + 1) + g1w - 1) / g1w);
    }
    P.blk_start[p.nchunks + 1] = t;
  }
  P.total_tiles = P.fwd_tiles + t;
  unsigned* ctr = a.ctr;
  P.tile_counter = (int*)ctr;
  P.g5count = ctr + 1;
  P.g0done = ctr + L.g0done;
  P.lsedone = ctr + L.lsedone;
  P.rowdone = ctr + L.rowdone;
  P.coldone = ctr + L.coldone;
  P.consumed = ctr + L.consumed;
  P.g2done = ctr + L.g2done;
  P.dhcdone = ctr + L.dhcdone;
  P.g2part = ctr + L.g2part;
  P.blockpart = reinterpret_cast<double*>(ctr + L.blockpart);
  P.part = a.part; P.tgt_logit = a.tgt_logit; P.lse = a.lse; P.nll = a.nll;
  P.rowscale = a.rowscale; P.loss = a.loss; P.loss_scale = a.loss_scale; P.tgt = a.tgt;
  P.tgt_len = a.tgt_len; P.bias = a.bias; P.db_part = a.db_part;
  int units = (ctas > 0 ? ctas : dev_info().sms) / Cfg::CTAS;
  units = std::max(1, std::min(units, P.total_tiles));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(units * Cfg::CTAS);
  cfg.blockDim = dim3(VB_THREADS);
  cfg.dynamicSmemBytes = VB_SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (kPair) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (g_opt_pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, vocab_kernel<kPair>, P));
  ++g_launches;
  return ATTN_OK;
}

static attn_status_t launch_vocab(const Plan& p, const VbArgs& a, int ctas, cudaStream_t stream) {
  return g_opt_vb_pair ? launch_vocab_k<true>(p, a, ctas, stream)
                       : launch_vocab_k<false>(p, a, ctas, stream);
}

struct CounterCtx {
  const Bufs* b;
  int idx;
};
static int* next_counter_fn(void* c) {
  CounterCtx* cc = (CounterCtx*)c;
  return (int*)(cc->b->counters + 1 + (cc->idx++));
}

template <typename T>
static attn_status_t run_stage(const Plan& p, const T* H, const T* S, const int32_t* tgt_ids,
                               const T* W_c, const T* W_out, const T* Wa, const T* b_out,
                               float loss_scale, float* loss, T* dH, T* dS, float* dW_c,
                               float* dW_out, float* dWa, float* db_out, const Bufs& b,
                               attn_comm_t* comm, cudaStream_t stream) {
  attn_status_t st;
  const bool tc = p.bf16;
  CounterCtx cctx{&b, 0};
  // once gradients are being allreduced (after the first dW_out chunk), the
  // persistent GEMMs leave the SMs NCCL's kernels are capped to
  int reserve = 0;
  auto gemm = [&](const GemmDesc* gs, int n, int pair_bit) -> attn_status_t {
    if (tc)
      return launch_tc_group<__nv_bfloat16>(gs, n, next_counter_fn(&cctx), stream, pair_bit,
                                            reserve > 0 ? dev_info().sms - reserve : 0);
    return launch_simt_group(gs, n, stream);
  };
  const int d = p.d;
  const long long TT = p.T;
  CUDA_TRY(cudaMemsetAsync(b.counters, 0, sizeof(unsigned int) * kNumCounters, stream));
  g_prof.n = 0;
  g_launches = 0;
  prof_mark("start", stream);

  // ---- F1, F2 (Eqs. 1-3); Eq. 2 general score: Q = H W_alpha first
  if (tc) {
    st = attention_forward_tc(p, H, S, b, stream, next_counter_fn, &cctx, Wa);
  } else {
    if (Wa) {
      GemmDesc g = g_query(p, b, H, Wa);
      if ((st = gemm(&g, 1, 0)) != ATTN_OK) return st;
    }
    st = attention_forward<T>(p, Wa ? (const T*)b.q : H, S, b.src_len, b.alpha, (T*)b.ctx, stream);
  }
  if (st != ATTN_OK) return st;
  prof_mark("attn_fwd", stream);

  // ---- F3 (Eq. 4)
  {
    GemmDesc g = g_proj(p, H, b.ctx, W_c, b.hc);
    if ((st = gemm(&g, 1, PAIR_FWD)) != ATTN_OK) return st;
  }
  prof_mark("proj_tanh", stream, true);
  CommRun cr;
  if (comm) {
    if ((st = comm_begin(comm, stream, &cr)) != ATTN_OK) return st;
  }
  // ---- F4 + F5 + B1, bf16: ONE persistent launch (vocab.cuh): the logits
  // tiles' (max, sum exp) partials, lse / NLL / loss, and the backward with
  // the logits recomputed per V-chunk -- the logits never reach HBM (their bf16
  // gradient dL passes through an L2-sized chunk scratch)
  if (p.vb) {
    if (!g_opt_vb_fwd) {
      // F4 on the single-CTA engine (logits discarded, per-tile (max, sum
      // exp) kept), then Eq. 6
      GemmDesc g = g_vocab_fwd(p, b, W_out, tgt_ids, b_out);
      if ((st = gemm(&g, 1, PAIR_FWD)) != ATTN_OK) return st;
      prof_mark("vocab_fwd", stream, true);
      const int blocks = (int)((TT + 7) / 8);
      st = launch_pdl(lse_reduce_kernel, dim3(blocks), dim3(256), stream, (const float2*)b.part,
                      p.part_ld, (const float*)b.tgt_logit, (const int*)b.tgt_len, (int)TT, p.N,
                      loss_scale, b.lse, b.nll, b.rowscale, b.blockpart, b.counters, loss);
      if (st != ATTN_OK) return st;
      prof_mark("lse_reduce", stream, true);
    }
    CUDA_TRY(cudaMemsetAsync(b.vbctr, 0, sizeof(unsigned) * p.n_vbctr, stream));
    int ctas = 0;
    if (comm) {
      // allreduce dW_out in groups of ~32 MB of chunks, each as soon as the
      // launch has stored those rows (a one-thread wait kernel on the comm
      // stream watches the counters); the launch leaves NCCL's SMs free
      if ((st = comm_fork(comm, &cr, stream)) != ATTN_OK) return st;
      const VbLayout L = vb_ctr_layout(p, g_opt_vb_pair != 0);
      const unsigned* g2done = b.vbctr + L.g2done;
      const long long chunk_bytes = 4ll * p.Vc * d;
      const int per = (int)std::max(1ll, (32ll << 20) / chunk_bytes);
      for (int c0 = 0; c0 < p.nchunks; c0 += per) {
        const int c1 = std::min(p.nchunks, c0 + per);
        vb_wait_g2_kernel<<<1, 32, 0, comm_stream(comm)>>>(
            g2done, c0, c1, p.Vc, p.V, L.ndt, VB_EPI_WARPS * (g_opt_vb_pair ? 2 : 1), L.TM);
        CUDA_TRY(cudaGetLastError());
        ++g_launches;
        const long long r0 = (long long)c0 * p.Vc, r1 = std::min((long long)p.V, (long long)c1 * p.Vc);
        if ((st = comm_allreduce_forked(comm, &cr, dW_out + r0 * d, (size_t)((r1 - r0) * d))) !=
            ATTN_OK)
          return st;
      }
      reserve = comm_max_ctas(comm);
      if (reserve > 0) ctas = (dev_info().sms - reserve) & ~1;
    }
    VbArgs va;
    va.hc = b.hc; va.W_out = W_out; va.dl = b.dl[0]; va.dhc = b.dhc; va.dW_out = dW_out;
    va.part = b.part; va.part_ld = p.part_ld; va.tgt_logit = b.tgt_logit; va.lse = b.lse;
    va.nll = b.nll; va.rowscale = b.rowscale; va.loss = loss; va.loss_scale = loss_scale;
    va.tgt = tgt_ids; va.tgt_len = b.tgt_len; va.bias = b_out; va.db_part = db_out ? b.dbpart : nullptr;
    va.ctr = b.vbctr;
    va.fwd = g_opt_vb_fwd != 0;
    if ((st = launch_vocab(p, va, ctas, stream)) != ATTN_OK) return st;
    if (db_out) {   // F_c bias: db_out = the launch's per-32-row column sums, added in order
      st = launch_pdl(db_final_kernel, dim3((unsigned)((p.V + 255) / 256)), dim3(256), stream,
                      (const float*)b.dbpart, (int)((TT + 31) / 32), p.V, db_out);
      if (st != ATTN_OK) return st;
    }
    prof_mark(g_opt_vb_fwd ? "vocab" : "vocab_bwd", stream, true);
  } else {
  // ---- F4 (Eq. 5): logits discarded, per-tile (max, sumexp) kept
  {
    GemmDesc g = g_vocab_fwd(p, b, W_out, tgt_ids, b_out);
    if ((st = gemm(&g, 1, PAIR_FWD)) != ATTN_OK) return st;
  }
  prof_mark("vocab_fwd", stream, true);
  // ---- Eq. 6: lse, token NLL, row scale, loss
  {
    const int blocks = (int)((TT + 7) / 8);
    st = launch_pdl(lse_reduce_kernel, dim3(blocks), dim3(256), stream, (const float2*)b.part,
                    p.part_ld, (const float*)b.tgt_logit, (const int*)b.tgt_len, (int)TT, p.N,
                    loss_scale, b.lse, b.nll, b.rowscale, b.blockpart, b.counters, loss);
    if (st != ATTN_OK) return st;
  }
  prof_mark("lse_reduce", stream, true);

  // ---- B1: V-chunked vocab backward.  Launch c runs dW_out[c] and dHc += ...
  // for chunk c together with the dlogits of chunk c+1 (double-buffered).
  // With stored logits, an elementwise kernel makes dlogits_c from the
  // forward's fp16 logits before launch c (no recompute on the tensor cores).
  {
    // db_out: column sums of each dlogits chunk -- by the stored-logits
    // ablation's dlogits kernels (db_mode 2) or column-sum kernels (0)
    const int db_mode = g_opt_db_gemm >= 0 ? g_opt_db_gemm : (p.store_logits ? 2 : 0);
    const bool db_ew = db_out && p.store_logits && db_mode == 2;
    int ew_parts0 = 0, ew_parts = 0;   // db_ew: row groups of chunk 0 / the later chunks
    // dlogits of chunk c from the stored logits (on `s`, `blocks` blocks)
    auto dlogits_ew = [&](int c, cudaStream_t s, int blocks) -> attn_status_t {
      const int c0 = c * p.Vc, vcc = std::min(p.Vc, p.V - c0);
      if (db_ew) {   // + column sums: column slabs x row groups, ~`blocks` blocks
        // (the row-group count depends on the full chunk width only, so every
        // chunk after the first has the same number of partial rows)
        const int slabs = (vcc + 8 * kEwThreads - 1) / (8 * kEwThreads);
        const int full_slabs = (std::min(p.Vc, p.V) + 8 * kEwThreads - 1) / (8 * kEwThreads);
        const int groups = (int)std::min<long long>(
            TT, std::max(1, std::min(kEwParts, blocks / full_slabs)));
        (c == 0 ? ew_parts0 : ew_parts) = groups;
        return launch_pdl(dlogits_colsum_kernel, dim3((unsigned)groups, (unsigned)slabs),
                          dim3(kEwThreads), s, (const __half*)b.logits, p.Vld, c0, vcc, (int)TT,
                          (const float*)b.lse, (const float*)b.rowscale, tgt_ids,
                          (const float*)b.tgt_logit, (__nv_bfloat16*)b.dl[c & 1], (long long)p.Vc,
                          b.dbpart, (long long)p.V,
                          (c == 0 || !g_opt_pdl || g_opt_store_logits == 2) ? 1 : 0);
      }
      return launch_pdl(dlogits_from_logits_kernel,
                        dim3((unsigned)std::min<long long>(TT, blocks)), dim3(kEwThreads), s,
                        (const __half*)b.logits, p.Vld, c0, vcc, (int)TT, (const float*)b.lse,
                        (const float*)b.rowscale, tgt_ids, (const float*)b.tgt_logit,
                        (__nv_bfloat16*)b.dl[c & 1], (long long)p.Vc,
                        (c == 0 || !g_opt_pdl || g_opt_store_logits == 2) ? 1 : 0);
    };
    const int sms = dev_info().sms;
    if (p.store_logits) {
      if ((st = dlogits_ew(0, stream, 4 * sms)) != ATTN_OK) return st;
    } else {   // fp32 path: chunk 0's dlogits on the CUDA-core engine
      GemmDesc g0 = g_dlogits(p, b, W_out, tgt_ids, 0, b_out);
      if ((st = gemm(&g0, 1, 0)) != ATTN_OK) return st;
    }
    for (int c = 0; c < p.nchunks; ++c) {
      // chunks >= 1 start beside the previous launch: exactly one block per
      // SM (a finished block waits there for that launch, so a second wave
      // would only start after it)
      if (p.store_logits && c > 0 && !g_debug_skip_ew &&
          (st = dlogits_ew(c, stream, g_opt_store_logits == 1 && g_opt_pdl ? sms : 4 * sms)) !=
              ATTN_OK)
        return st;
      GemmDesc gs[4];
      int n = 0;
      gs[n++] = g_dwout(p, b, dW_out, c);   // K = T: the long tiles first
      gs[n++] = g_dhc(p, b, W_out, c);
      if (c + 1 < p.nchunks && !p.store_logits)
        gs[n++] = g_dlogits(p, b, W_out, tgt_ids, c + 1, b_out);
      if ((st = gemm(gs, n, PAIR_VBWD)) != ATTN_OK) return st;
      if (db_out && !db_ew) {
        // F_c bias: db_out[chunk c] = column sums of dlogits_c (still intact:
        // the next launch is the one that overwrites its buffer)
        const int c0 = c * p.Vc, vcc = std::min(p.Vc, p.V - c0);
        const int splits = (int)std::min<long long>(16, std::max<long long>(1, TT / 256));
        const int rps = (int)((TT + splits - 1) / splits);
        float* part = b.dbpart;
        colsum_part_kernel<T><<<dim3((vcc + 255) / 256, splits), 256, 0, stream>>>(
            (const T*)b.dl[c & 1], p.Vc, (int)TT, rps, vcc, part);
        colsum_final_kernel<<<(vcc + 255) / 256, 256, 0, stream>>>(part, splits, vcc, db_out + c0);
        CUDA_TRY(cudaGetLastError());
        g_launches += 2;
      }
      if (comm) {
        const int c0 = c * p.Vc;
        const int vcc = std::min(p.Vc, p.V - c0);
        if ((st = comm_enqueue_allreduce(comm, &cr, stream, dW_out + (size_t)c0 * d,
                                         (size_t)vcc * d)) != ATTN_OK)
          return st;
        reserve = comm_max_ctas(comm);
      }
    }
    if (db_ew) {   // db_out = the dlogits kernels' row-group partials, added in order
      st = launch_pdl(ew_colsum_final_kernel, dim3((unsigned)((p.V + 255) / 256)), dim3(256), stream,
                      (const float*)b.dbpart, ew_parts0, std::min(p.Vc, p.V),
                      p.nchunks > 1 ? ew_parts : ew_parts0, p.V, db_out);
      if (st != ATTN_OK) return st;
    }
  }
  }   // fp32 path / stored-logits ablation
  // dot score with the fused attention kernels: B2 as {dC, dW_c split-K in
  // two halves} before the attention backward and {dH_dec = dz W_c[:, :d] +
  // dQ} after it (the 64 long dW_c tiles balance against the dC tiles; dQ
  // travels as bf16 instead of an fp32 dH_part)
  const bool b2split = tc && !Wa && attn_fused_ok(p);
  // tanh backward of Eq. 4: dz = dHc (1 - H_c^2)  (and, split B2: dW_c = 0)
  {
    const long long n = TT * d;
    st = launch_pdl(dz_kernel<T>, dim3((int)std::min<long long>((n + 255) / 256, 148ll * 16)),
                    dim3(256), stream, (const float*)b.dhc, (const T*)b.hc, (T*)b.dz, n,
                    reinterpret_cast<float4*>(dW_c), b2split ? (long long)d * 2 * d / 4 : 0ll);
    if (st != ATTN_OK) return st;
  }
  prof_mark(p.vb ? "dz" : "vocab_bwd", stream, true);
  // ---- B2: dW_c = dz^T [H | C];  dH_part = dz W_c[:, :d];  dC = dz W_c[:, d:]
  {
    GemmDesc gs[3];
    int n = 0;
    if (b2split && p.T >= 256) {
      gs[n++] = g_dwc_half(p, b, H, dW_c, 0);
      gs[n++] = g_dwc_half(p, b, H, dW_c, 1);
      gs[n++] = g_dzwc(p, b, W_c, d, d, EPI_STORE_BF16, b.dcbf, d);
    } else if (b2split) {
      gs[n++] = g_dwc_half(p, b, H, dW_c, -1);
      gs[n++] = g_dzwc(p, b, W_c, d, d, EPI_STORE_BF16, b.dcbf, d);
    } else {
      gs[n++] = g_dwc(p, b, H, dW_c);
    }
    if (b2split) {
    } else if (tc) {
      gs[n++] = g_dzwc(p, b, W_c, 0, d, EPI_STORE_F32, b.dhpart, d);
      gs[n++] = g_dzwc(p, b, W_c, d, d, EPI_STORE_BF16, b.dcbf, d);
    } else {
      gs[n++] = g_dzwc(p, b, W_c, 0, 2 * d, EPI_STORE_F32, b.dhc2, 2ll * d);
    }
    if ((st = gemm(gs, n, PAIR_PBWD)) != ATTN_OK) return st;
    if (comm) {
      if ((st = comm_enqueue_allreduce(comm, &cr, stream, dW_c, (size_t)d * 2 * d)) != ATTN_OK) return st;
    }
  }
  prof_mark("proj_bwd", stream);
  // ---- B3: attention backward
  if (tc) {
    st = attention_backward_tc(p, H, S, dH, dS, b, stream, next_counter_fn, &cctx, Wa, dWa);
  } else {
    st = attention_backward<T>(p, Wa ? (const T*)b.q : H, S, b.alpha, b.dalpha, b.dhc2, dH, dS,
                               Wa ? (T*)b.dq : nullptr, stream);
    if (st == ATTN_OK && Wa) {
      // dH_dec = dH_part + dQ W_alpha^T (accumulated onto a copy of dH_part);
      // dW_alpha = H^T dQ
      CUDA_TRY(cudaMemcpy2DAsync(dH, sizeof(T) * d, b.dhc2, sizeof(float) * 2 * d, sizeof(T) * d,
                                 (size_t)TT, cudaMemcpyDeviceToDevice, stream));
      GemmDesc ga[2] = {g_query_bwd_dh(p, b, Wa, dH, EPI_ACCUM_F32), g_query_bwd_dw(p, b, H, dWa)};
      st = gemm(ga, 2, 0);
    }
  }
  if (st != ATTN_OK) return st;
  if (b2split) {   // dH_dec = dz W_c[:, :d] + dQ (bf16 addend)
    GemmDesc g = g_dzwc(p, b, W_c, 0, d, EPI_ADD_BF16, dH, d);
    g.epi.addend = reinterpret_cast<const float*>(b.dq2);
    g.epi.addend_bf16 = 1;
    g.epi.add_ld = d;
    if ((st = gemm(&g, 1, PAIR_PBWD)) != ATTN_OK) return st;
  }
  prof_mark("attn_bwd", stream);
  if (comm && dWa) {
    if ((st = comm_enqueue_allreduce(comm, &cr, stream, dWa, (size_t)d * d)) != ATTN_OK) return st;
  }
  if (comm && db_out) {
    if ((st = comm_enqueue_allreduce(comm, &cr, stream, db_out, (size_t)p.V)) != ATTN_OK) return st;
  }
  if (comm) {
    if ((st = comm_enqueue_allreduce(comm, &cr, stream, loss, 1)) != ATTN_OK) return st;
    if ((st = comm_end(comm, &cr, stream)) != ATTN_OK) return st;
  }
  return ATTN_OK;
}

// Has this device already run the call path given by the shape, the optional
// operands and the options (see the lazy-loading note in attn_softmax_fwd_bwd_ex)?
// Marks it as run.
static bool path_warmed(const Plan& p, bool wa, bool bias) {
  static std::mutex mu;
  static std::set<std::pair<int, uint64_t>> seen;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  uint64_t h = 1469598103934665603ull;   // FNV-1a over the path's determinants
  auto mix = [&](long long v) { h = (h ^ (uint64_t)v) * 1099511628211ull; };
  for (long long v : {(long long)p.B, (long long)p.N, (long long)p.M, (long long)p.d,
                      (long long)p.V, (long long)p.bf16, (long long)wa, (long long)bias,
                      (long long)g_opt_vb_pair, (long long)g_opt_vb_fwd,
                      (long long)g_opt_store_logits, (long long)g_opt_attn_fused,
                      (long long)g_opt_vb_wide, (long long)g_opt_wide, (long long)g_opt_db_gemm,
                      (long long)g_opt_proj_bn, (long long)g_opt_vb_order,
                      (long long)g_opt_vb_g1wide, (long long)g_opt_mn3d})
    mix(v);
  std::lock_guard<std::mutex> lk(mu);
  return !seen.insert({dev, h}).second;
}

extern "C" attn_status_t attn_softmax_fwd_bwd_ex(
    const attn_shape_t* s, const void* H_dec, const void* H_enc, const int32_t* src_lens_host,
    const int32_t* tgt_lens_host, const int32_t* tgt_ids, const void* W_c, const void* W_out,
    const void* W_alpha, const void* b_out, float loss_scale, float* loss, void* dH_dec,
    void* dH_enc, float* dW_c, float* dW_out, float* dW_alpha, float* db_out, void* workspace,
    size_t workspace_bytes, attn_comm_t* comm, void* stream_) {
  attnsm::NvtxRange nvtx_range_("attn_softmax_fwd_bwd_ex");
  OPT_LOCK;
  attn_status_t st = validate(s, H_dec, H_enc, src_lens_host, tgt_lens_host, tgt_ids, W_c, W_out,
                              W_alpha, loss, dH_dec, dH_enc, dW_c, dW_out, dW_alpha,
                              workspace_bytes, workspace);
  if (st != ATTN_OK) return st;
  if ((b_out == nullptr) != (db_out == nullptr))
    return fail(ATTN_ERR_INVALID_ARG,
                "b_out and db_out go together: both NULL (no F_c bias, DESIGN.md R6) or both set; "
                "got b_out=%p db_out=%p", b_out, (const void*)db_out);
  cudaStream_t stream = (cudaStream_t)stream_;
  const Plan p = make_plan(s);
  const Bufs b = carve(p, workspace);
  // lengths: host -> workspace (the harness's arrays are small and pageable)
  if ((st = upload_lens(b.src_len, src_lens_host, tgt_lens_host, p.B, stream)) != ATTN_OK) return st;
  // With a communicator, spinning wait kernels on the comm stream (they
  // release each dW_out chunk group's allreduce) are resident while the main
  // stream launches the rest of the step.  Under CUDA's lazy module loading
  // the first launch of a kernel may have to wait for the device to go idle,
  // which the spinning kernel prevents: a deadlock (measured: bench.py
  // --force-comm hung when its first call carried the communicator).  So the
  // first call of each path (shape, operands, options) on a device runs once
  // without the communicator, which loads every kernel the path launches.
  // (not while the stream is being captured into a CUDA graph: nothing runs
  // during capture, and instantiation loads the graph's kernels)
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CUDA_TRY(cudaStreamIsCapturing(stream, &cap));
  if (comm && cap == cudaStreamCaptureStatusNone &&
      !path_warmed(p, W_alpha != nullptr, b_out != nullptr)) {
    st = p.bf16 ? run_stage<__nv_bfloat16>(p, (const __nv_bfloat16*)H_dec, (const __nv_bfloat16*)H_enc,
                                           tgt_ids, (const __nv_bfloat16*)W_c,
                                           (const __nv_bfloat16*)W_out, (const __nv_bfloat16*)W_alpha,
                                           (const __nv_bfloat16*)b_out, loss_scale, loss,
                                           (__nv_bfloat16*)dH_dec, (__nv_bfloat16*)dH_enc, dW_c,
                                           dW_out, dW_alpha, db_out, b, nullptr, stream)
                : run_stage<float>(p, (const float*)H_dec, (const float*)H_enc, tgt_ids,
                                   (const float*)W_c, (const float*)W_out, (const float*)W_alpha,
                                   (const float*)b_out, loss_scale, loss, (float*)dH_dec,
                                   (float*)dH_enc, dW_c, dW_out, dW_alpha, db_out, b, nullptr, stream);
    if (st != ATTN_OK) return st;
  }
  if (p.bf16)
    st = run_stage<__nv_bfloat16>(p, (const __nv_bfloat16*)H_dec, (const __nv_bfloat16*)H_enc,
                                  tgt_ids, (const __nv_bfloat16*)W_c,
                                  (const __nv_bfloat16*)W_out, (const __nv_bfloat16*)W_alpha,
                                  (const __nv_bfloat16*)b_out, loss_scale, loss,
                                  (__nv_bfloat16*)dH_dec, (__nv_bfloat16*)dH_enc, dW_c, dW_out,
                                  dW_alpha, db_out, b, comm, stream);
  else
    st = run_stage<float>(p, (const float*)H_dec, (const float*)H_enc, tgt_ids, (const float*)W_c,
                          (const float*)W_out, (const float*)W_alpha, (const float*)b_out,
                          loss_scale, loss, (float*)dH_dec, (float*)dH_enc, dW_c, dW_out,
                          dW_alpha, db_out, b, comm, stream);
  g_launches += (2 * p.B + 511) / 512;   // the length upload kernels
  return st;
}

extern "C" attn_status_t attn_softmax_fwd_bwd(
    const attn_shape_t* s, const void* H_dec, const void* H_enc, const int32_t* src_lens_host,
    const int32_t* tgt_lens_host, const int32_t* tgt_ids, const void* W_c, const void* W_out,
    const void* W_alpha, float loss_scale, float* loss, void* dH_dec, void* dH_enc, float* dW_c,
    float* dW_out, float* dW_alpha, void* workspace, size_t workspace_bytes, attn_comm_t* comm,
    void* stream_) {
  attnsm::NvtxRange nvtx_range_("attn_softmax_fwd_bwd");
  return attn_softmax_fwd_bwd_ex(s, H_dec, H_enc, src_lens_host, tgt_lens_host, tgt_ids, W_c,
                                 W_out, W_alpha, nullptr, loss_scale, loss, dH_dec, dH_enc, dW_c,
                                 dW_out, dW_alpha, nullptr, workspace, workspace_bytes, comm,
                                 stream_);
}

// ------------------------------------------------------------------ host-buffer variant
extern "C" size_t attn_softmax_host_staging_size(const attn_shape_t* s) {
  if (check_shape(s) != ATTN_OK) return 0;
  const size_t elt = s->dtype == ATTN_BF16 ? 2 : 4;
  const size_t T = (size_t)s->batch * s->tgt_len;
  return align_up(elt * T * s->hidden) + align_up(elt * (size_t)s->batch * s->src_len * s->hidden) +
         align_up(sizeof(int32_t) * T) + align_up(sizeof(float));
}

extern "C" attn_status_t attn_softmax_fwd_bwd_host(
    const attn_shape_t* s, const void* H_dec_host, const void* H_enc_host,
    const int32_t* src_lens_host, const int32_t* tgt_lens_host, const int32_t* tgt_ids_host,
    const void* W_c, const void* W_out, float loss_scale, float* loss_host, void* dH_dec,
    void* dH_enc, float* dW_c, float* dW_out, void* staging, size_t staging_bytes,
    void* workspace, size_t workspace_bytes, attn_comm_t* comm, void* stream_) {
  attnsm::NvtxRange nvtx_range_("attn_softmax_fwd_bwd_host");
  attn_status_t st = check_shape(s);
  if (st != ATTN_OK) return st;
  if (!H_dec_host || !H_enc_host || !tgt_ids_host || !loss_host || !staging)
    return fail(ATTN_ERR_INVALID_ARG, "host-variant buffer is NULL");
  const size_t need = attn_softmax_host_staging_size(s);
  if (staging_bytes < need)
    return fail(ATTN_ERR_WORKSPACE, "staging_bytes = %zu < required %zu", staging_bytes, need);
  cudaStream_t stream = (cudaStream_t)stream_;
  const size_t elt = s->dtype == ATTN_BF16 ? 2 : 4;
  const size_t T = (size_t)s->batch * s->tgt_len;
  const size_t bh = elt * T * s->hidden, be = elt * (size_t)s->batch * s->src_len * s->hidden;
  char* st0 = (char*)staging;
  void* dHd = st0;
  void* dHe = st0 + align_up(bh);
  int32_t* dIds = (int32_t*)(st0 + align_up(bh) + align_up(be));
  float* dLoss = (float*)((char*)dIds + align_up(sizeof(int32_t) * T));
  CUDA_TRY(cudaMemcpyAsync(dHd, H_dec_host, bh, cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaMemcpyAsync(dHe, H_enc_host, be, cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaMemcpyAsync(dIds, tgt_ids_host, sizeof(int32_t) * T, cudaMemcpyHostToDevice, stream));
  st = attn_softmax_fwd_bwd(s, dHd, dHe, src_lens_host, tgt_lens_host, dIds, W_c, W_out, nullptr,
                            loss_scale, dLoss, dH_dec, dH_enc, dW_c, dW_out, nullptr, workspace,
                            workspace_bytes, comm, stream_);
  if (st != ATTN_OK) return st;
  CUDA_TRY(cudaMemcpyAsync(loss_host, dLoss, sizeof(float), cudaMemcpyDeviceToHost, stream));
  return ATTN_OK;
}

// ------------------------------------------------------------------ pipelined host variant
// Library-owned copy stream and per-staging-buffer "ready" events.
struct StagingSlot {
  const void* ptr = nullptr;
  cudaEvent_t ready = nullptr;
  int dev = -1;        // the device the event belongs to
};
static std::mutex g_stage_mu;
static StagingSlot g_slots[8];
static int g_slot_next = 0;
// the H2D copy stream and its ordering event, one per device (created on first use)
constexpr int kMaxDevices = 64;
static cudaStream_t g_copy_stream[kMaxDevices] = {};
static cudaEvent_t g_free_ev[kMaxDevices] = {};

static attn_status_t staging_slot(const void* ptr, int dev, cudaEvent_t* ev) {
  std::lock_guard<std::mutex> lk(g_stage_mu);
  for (auto& sl : g_slots)
    if (sl.ptr == ptr && sl.dev == dev) { *ev = sl.ready; return ATTN_OK; }
  StagingSlot& sl = g_slots[g_slot_next++ % 8];
  if (sl.ready && sl.dev != dev) {   // an event of another device: replace it
    CUDA_TRY(cudaEventDestroy(sl.ready));
    sl.ready = nullptr;
  }
  if (!sl.ready) CUDA_TRY(cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming));
  sl.ptr = ptr;
  sl.dev = dev;
  *ev = sl.ready;
  return ATTN_OK;
}

struct StagingViews {
  void* H_dec; void* H_enc; int32_t* ids; float* loss;
};
static StagingViews staging_views(const attn_shape_t* s, const void* staging) {
  const size_t elt = s->dtype == ATTN_BF16 ? 2 : 4;
  const size_t T = (size_t)s->batch * s->tgt_len;
  const size_t bh = elt * T * s->hidden, be = elt * (size_t)s->batch * s->src_len * s->hidden;
  char* p = (char*)staging;
  StagingViews v;
  v.H_dec = p;
  v.H_enc = p + align_up(bh);
  v.ids = (int32_t*)(p + align_up(bh) + align_up(be));
  v.loss = (float*)((char*)v.ids + align_up(sizeof(int32_t) * T));
  return v;
}

extern "C" attn_status_t attn_softmax_prefetch_host(const attn_shape_t* s, const void* H_dec_host,
                                                    const void* H_enc_host,
                                                    const int32_t* tgt_ids_host, void* staging,
                                                    size_t staging_bytes, void* stream_) {
  attn_status_t st = check_shape(s);
  if (st != ATTN_OK) return st;
  if (!H_dec_host || !H_enc_host || !tgt_ids_host || !staging)
    return fail(ATTN_ERR_INVALID_ARG, "prefetch: NULL argument");
  if (staging_bytes < attn_softmax_host_staging_size(s))
    return fail(ATTN_ERR_WORKSPACE, "staging_bytes = %zu < required %zu", staging_bytes,
                attn_softmax_host_staging_size(s));
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (dev >= kMaxDevices) return fail(ATTN_ERR_UNSUPPORTED, "prefetch: device %d >= %d", dev, kMaxDevices);
  cudaStream_t copy_stream;
  cudaEvent_t free_ev;
  {
    std::lock_guard<std::mutex> lk(g_stage_mu);
    if (!g_copy_stream[dev]) {
      CUDA_TRY(cudaStreamCreateWithFlags(&g_copy_stream[dev], cudaStreamNonBlocking));
      CUDA_TRY(cudaEventCreateWithFlags(&g_free_ev[dev], cudaEventDisableTiming));
    }
    copy_stream = g_copy_stream[dev];
    free_ev = g_free_ev[dev];
  }
  cudaEvent_t ready;
  if ((st = staging_slot(staging, dev, &ready)) != ATTN_OK) return st;
  // the staging buffer is free once everything enqueued on `stream` so far is done
  CUDA_TRY(cudaEventRecord(free_ev, (cudaStream_t)stream_));
  CUDA_TRY(cudaStreamWaitEvent(copy_stream, free_ev, 0));
  const size_t elt = s->dtype == ATTN_BF16 ? 2 : 4;
  const size_t T = (size_t)s->batch * s->tgt_len;
  StagingViews v = staging_views(s, staging);
  CUDA_TRY(cudaMemcpyAsync(v.H_dec, H_dec_host, elt * T * s->hidden, cudaMemcpyHostToDevice,
                           copy_stream));
  CUDA_TRY(cudaMemcpyAsync(v.H_enc, H_enc_host, elt * (size_t)s->batch * s->src_len * s->hidden,
                           cudaMemcpyHostToDevice, copy_stream));
  CUDA_TRY(cudaMemcpyAsync(v.ids, tgt_ids_host, sizeof(int32_t) * T, cudaMemcpyHostToDevice,
                           copy_stream));
  CUDA_TRY(cudaEventRecord(ready, copy_stream));
  return ATTN_OK;
}

extern "C" attn_status_t attn_softmax_fwd_bwd_staged(
    const attn_shape_t* s, const void* staging, size_t staging_bytes, const int32_t* src_lens_host,
    const int32_t* tgt_lens_host, const void* W_c, const void* W_out, float loss_scale,
    float* loss_host, void* dH_dec, void* dH_enc, float* dW_c, float* dW_out, void* workspace,
    size_t workspace_bytes, attn_comm_t* comm, void* stream_) {
  attnsm::NvtxRange nvtx_range_("attn_softmax_fwd_bwd_staged");
  attn_status_t st = check_shape(s);
  if (st != ATTN_OK) return st;
  if (!staging || !loss_host) return fail(ATTN_ERR_INVALID_ARG, "staged: NULL argument");
  if (staging_bytes < attn_softmax_host_staging_size(s))
    return fail(ATTN_ERR_WORKSPACE, "staging_bytes = %zu < required %zu", staging_bytes,
                attn_softmax_host_staging_size(s));
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  cudaEvent_t ready;
  if ((st = staging_slot(staging, dev, &ready)) != ATTN_OK) return st;
  cudaStream_t stream = (cudaStream_t)stream_;
  CUDA_TRY(cudaStreamWaitEvent(stream, ready, 0));
  StagingViews v = staging_views(s, staging);
  st = attn_softmax_fwd_bwd(s, v.H_dec, v.H_enc, src_lens_host, tgt_lens_host, v.ids, W_c, W_out,
                            nullptr, loss_scale, v.loss, dH_dec, dH_enc, dW_c, dW_out, nullptr,
                            workspace, workspace_bytes, comm, stream_);
  if (st != ATTN_OK) return st;
  CUDA_TRY(cudaMemcpyAsync(loss_host, v.loss, sizeof(float), cudaMemcpyDeviceToHost, stream));
  return ATTN_OK;
}

// ------------------------------------------------------------------ id check
extern "C" attn_status_t attn_softmax_check_ids(const attn_shape_t* s, const int32_t* tgt_lens_host,
                                                const int32_t* tgt_ids, void* stream_) {
  attn_status_t st = check_shape(s);
  if (st != ATTN_OK) return st;
  if (!tgt_lens_host || !tgt_ids) return fail(ATTN_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t stream = (cudaStream_t)stream_;
  const int T = s->batch * s->tgt_len;
  int* dev = nullptr;
  CUDA_TRY(cudaMallocAsync(&dev, sizeof(int) * (1 + s->batch), stream));
  CUDA_TRY(cudaMemsetAsync(dev, 0, sizeof(int), stream));
  CUDA_TRY(cudaMemcpyAsync(dev + 1, tgt_lens_host, sizeof(int) * s->batch, cudaMemcpyHostToDevice, stream));
  check_ids_kernel<<<(T + 255) / 256, 256, 0, stream>>>(tgt_ids, dev + 1, T, s->tgt_len, s->vocab, dev);
  int bad = 0;
  CUDA_TRY(cudaMemcpyAsync(&bad, dev, sizeof(int), cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaFreeAsync(dev, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  if (bad) return fail(ATTN_ERR_TOKEN_RANGE, "a valid target id is outside [0, V = %d)", s->vocab);
  return ATTN_OK;
}

// ------------------------------------------------------------------ decoding step (NEXT-4)
// Forward-only Eqs. 1-5 for the N live hypotheses of each of B sentences (the
// rows of one sentence share its encoder states), and per row the lse and the
// k best tokens of log P: the vocab GEMM's epilogue keeps per-tile (max,
// sumexp) and top-8 lists (logits are never stored), decode_final_kernel
// merges them.
static size_t decode_topk_bytes(const Plan& p) { return align_up(sizeof(uint32_t) * 8 * p.T * p.part_ld); }

extern "C" size_t attn_softmax_decode_workspace_size(const attn_shape_t* s) {
  OPT_LOCK;
  if (check_shape(s) != ATTN_OK || s->dtype != ATTN_BF16) return 0;
  const Plan p = make_plan(s);
  return p.total + decode_topk_bytes(p);
}

// ---------------------------------------------------------------- input feeding (NEXT-3 IF)
// Internal entry for lstm.cu's input-feeding decoder (HybridNMTIF, PAPER.md:
// 157): one decoder step of the attention for B sentences -- alpha and C of
// q = h (N = 1) over S, then Htilde = tanh(W_c [h; C]) (Eqs. 1-4) written to
// `out` with row stride ld_out (elements) -- on the same kernels as the stage.
size_t attn_internal_step_ws(int B, int M, int d) {
  attn_shape_t s{B, 1, M, d, 64, ATTN_BF16};
  return make_plan(&s).total;
}
attn_status_t attn_internal_step_attention(int B, int M, int d, const void* h, const void* S,
                                           const int* src_len_dev, const void* W_c, void* out,
                                           long long ld_out, void* ws, cudaStream_t stream) {
  OPT_LOCK;
  attn_shape_t s{B, 1, M, d, 64, ATTN_BF16};
  const Plan p = make_plan(&s);
  Bufs b = carve(p, ws);
  b.src_len = const_cast<int*>(src_len_dev);   // lengths already on the device
  CUDA_TRY(cudaMemsetAsync(b.counters, 0, sizeof(unsigned int) * kNumCounters, stream));
  CounterCtx cctx{&b, 0};
  attn_status_t st = attention_forward_tc(p, h, S, b, stream, next_counter_fn, &cctx, nullptr);
  if (st != ATTN_OK) return st;
  GemmDesc g = g_proj(p, h, b.ctx, W_c, out);
  g.epi.ldo = ld_out;
  return launch_tc_group<__nv_bfloat16>(&g, 1, next_counter_fn(&cctx), stream, PAIR_FWD);
}

// Internal entry for lstm.cu's backward (NEXT-3 training): C[M][N] fp32 =
// A^T [B0 | B1] with A [K][M], B0 [K][n0], B1 [K][N - n0] row-major bf16 (both
// operands MN-major): dW_l = dz^T [x | h_prev] over all B T rows.  `counter`
// is a zeroed int of the caller's workspace.
static GemmDesc atb_desc(int M, int N, int K, const void* A, const void* B0, int n0, const void* B1,
                         float* C) {
  GemmDesc g;
  g.M = M; g.N = N; g.K = K;
  g.a_mn = 1; g.a0 = mnmaj(A, K, M, M);
  g.b_mn = 1; g.b0 = mnmaj(B0, K, n0, n0);
  g.b1 = mnmaj(B1, K, N - n0, N - n0); g.b_nsplit = n0;
  g.epi.kind = EPI_STORE_F32; g.epi.out = C; g.epi.ldo = N;
  g.epi.ncols_valid = N; g.epi.ncols_store = N;
  return g;
}
attn_status_t attn_internal_gemm_atb(int M, int N, int K, const void* A, const void* B0, int n0,
                                     const void* B1, float* C, int* counter, cudaStream_t stream) {
  OPT_LOCK;
  GemmDesc g = atb_desc(M, N, K, A, B0, n0, B1, C);
  return launch_tc_group<__nv_bfloat16>(&g, 1, counter, stream, 0);
}
// up to kMaxProblems such products in ONE launch (the layers of an LSTM side:
// one tile list, so the layers' tiles fill the machine together)
attn_status_t attn_internal_gemm_atb_group(int n, const int* M, const int* N, const int* K,
                                           const void* const* A, const void* const* B0,
                                           const int* n0, const void* const* B1, float* const* C,
                                           int* counter, cudaStream_t stream) {
  OPT_LOCK;
  if (n < 1 || n > kMaxProblems)
    return fail(ATTN_ERR_INVALID_ARG, "grouped GEMM: %d problems (1..%d)", n, kMaxProblems);
  GemmDesc g[kMaxProblems];
  for (int i = 0; i < n; ++i) g[i] = atb_desc(M[i], N[i], K[i], A[i], B0[i], n0[i], B1[i], C[i]);
  return launch_tc_group<__nv_bfloat16>(g, n, counter, stream, 0);
}

extern "C" attn_status_t attn_softmax_decode_step(
    const attn_shape_t* s, const void* H_dec, const void* H_enc, const int32_t* src_lens_host,
    const void* W_c, const void* W_out, const void* W_alpha, const void* b_out, int k,
    int32_t* topk_ids, float* topk_logp, float* lse, void* workspace, size_t workspace_bytes,
    void* stream_) {
  attnsm::NvtxRange nvtx_range_("attn_softmax_decode_step");
  OPT_LOCK;
  attn_status_t st = check_shape(s);
  if (st != ATTN_OK) return st;
  if (s->dtype != ATTN_BF16)
    return fail(ATTN_ERR_UNSUPPORTED, "decode step: bf16 only (tcgen05 top-k epilogue)");
  if (k < 1 || k > 8 || k > s->vocab)
    return fail(ATTN_ERR_INVALID_ARG, "decode step: k = %d outside [1, min(8, V = %d)]", k, s->vocab);
  const void* req[] = {H_dec, H_enc, src_lens_host, W_c, W_out, topk_ids, topk_logp, workspace};
  const char* nm[] = {"H_dec", "H_enc", "src_lens_host", "W_c", "W_out", "topk_ids", "topk_logp",
                      "workspace"};
  for (int i = 0; i < 8; ++i)
    if (!req[i]) return fail(ATTN_ERR_INVALID_ARG, "decode step: %s is NULL", nm[i]);
  for (int b = 0; b < s->batch; ++b)
    if (src_lens_host[b] < 1 || src_lens_host[b] > s->src_len)
      return fail(src_lens_host[b] < 1 ? ATTN_ERR_EMPTY_SOURCE : ATTN_ERR_SHAPE,
                  "decode step: src_lens_host[%d] = %d outside [1, M = %d]", b, src_lens_host[b],
                  s->src_len);
  const void* al[] = {H_dec, H_enc, W_c, W_out, W_alpha, workspace};
  for (const void* a : al)
    if (misaligned(a)) return fail(ATTN_ERR_UNSUPPORTED, "decode step: 16-byte aligned pointers needed");
  const Plan p = make_plan(s);
  if (workspace_bytes < p.total + decode_topk_bytes(p))
    return fail(ATTN_ERR_WORKSPACE, "workspace_bytes = %zu < required %zu", workspace_bytes,
                p.total + decode_topk_bytes(p));
  cudaStream_t stream = (cudaStream_t)stream_;
  const Bufs b = carve(p, workspace);
  uint32_t* topk = (uint32_t*)((char*)workspace + p.total);
  if ((st = upload_lens(b.src_len, src_lens_host, nullptr, p.B, stream)) != ATTN_OK) return st;
  CUDA_TRY(cudaMemsetAsync(b.counters, 0, sizeof(unsigned int) * kNumCounters, stream));
  g_launches = 0;
  CounterCtx cctx{&b, 0};
  // F1, F2 (and F0 for the general score)
  if ((st = attention_forward_tc(p, H_dec, H_enc, b, stream, next_counter_fn, &cctx, W_alpha)) !=
      ATTN_OK)
    return st;
  // F3 (Eq. 4): few rows -- narrower tiles so more SMs take part
  {
    GemmDesc g = g_proj(p, H_dec, b.ctx, W_c, b.hc);
    if ((p.T + 127) / 128 * ((p.d + 255) / 256) < 74) g.bn = 64;
    if ((st = launch_tc_group<__nv_bfloat16>(&g, 1, next_counter_fn(&cctx), stream, PAIR_FWD)) !=
        ATTN_OK)
      return st;
  }
  // F4 (Eq. 5) with the top-k epilogue
  {
    GemmDesc g = g_vocab_fwd(p, b, W_out, nullptr, b_out);
    g.epi.kind = EPI_TOPK;
    g.epi.topk = topk;
    g.epi.tgt_logit = nullptr;
    if ((st = launch_tc_group_k<__nv_bfloat16, 1, true>(&g, 1, next_counter_fn(&cctx), stream, 0)) !=
        ATTN_OK)
      return st;
  }
  st = launch_pdl(decode_final_kernel, dim3((unsigned)p.T), dim3(DF_THREADS), stream,
                  (const float2*)b.part, (const uint32_t*)topk, p.part_ld, (int)p.T, k, (int*)topk_ids,
                  topk_logp, lse);
  return st;
}

// ------------------------------------------------------------------ debug GEMM
extern "C" attn_status_t attn_debug_gemm_bf16(int M, int N, int K, const void* A, int a_mn,
                                              const void* B, int b_mn, float* C, void* stream_) {
  OPT_LOCK;
  if (M <= 0 || N <= 0 || K <= 0 || !A || !B || !C)
    return fail(ATTN_ERR_INVALID_ARG, "debug_gemm: bad arguments");
  GemmDesc g;
  g.M = M; g.N = N; g.K = K;
  g.a_mn = a_mn; g.a0 = a_mn ? mnmaj(A, K, M, M) : kmaj(A, M, K, K);
  g.b_mn = b_mn; g.b0 = b_mn ? mnmaj(B, K, N, N) : kmaj(B, N, K, K);
  g.epi.kind = EPI_STORE_F32; g.epi.out = C; g.epi.ldo = N; g.epi.ncols_valid = N; g.epi.ncols_store = N;
  if (g_debug_epi == 1) g.epi.kind = EPI_NONE;
  if (g_debug_epi == 2 || g_debug_epi == 3) {
    // bf16 output written into the (larger) fp32 buffer C as [M, N] bf16
    g.epi.kind = g_debug_epi == 2 ? EPI_STORE_BF16 : EPI_TANH;
  }
  // one persistent device counter per process (debug entry only); the memset
  // is stream-ordered so the call can be captured in a CUDA graph
  static int* counter = nullptr;
  if (!counter) CUDA_TRY(cudaMalloc(&counter, sizeof(int)));
  cudaStream_t stream = (cudaStream_t)stream_;
  CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(int), stream));
  attn_status_t st = launch_tc_group<__nv_bfloat16>(&g, 1, counter, stream, PAIR_DEBUG);
  return st;
}
