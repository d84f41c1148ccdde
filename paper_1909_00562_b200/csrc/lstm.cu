// lstm.cu -- NEXT-3: the model-parallel half of Fig. 3 of
// arXiv 1909.00562, the stacked-LSTM encoder and decoder that produce the
// hidden states S = H_enc and H = H_dec of every step.
//
// The proposed model has no input feeding, so layer-step
// (l, t) depends only on (l, t-1) and (l-1, t): the "green arrow" wavefront
// (PAPER.md:97, :117).  The paper places layers on different GPUs and lets
// each start a step as soon as its left and lower neighbours are done; here
// the wavefront is ONE persistent cooperative kernel per side (encoder, then
// decoder) in which the SMs are split into L groups of G CTAs, group l owning
// layer l (the paper's GPUs become SM groups of one B200; the same schedule
// across GPUs would replace the flag polling below by NVLink peer flags):
//
//   CTA (l, g), g < G, owns hidden units [g U, (g+1) U), U = hd / G, i.e. the
//   4U gate rows of W_l = [W_ih | W_hh] packed gate-interleaved (row 4u + q
//   = gate q of unit u, q in i, f, g, o).  For each step t it waits until
//   every CTA of (l-1, t) and of (l, t-1) has published (global counters,
//   release / acquire at gpu scope), streams [x_t | h_{t-1}] (128 batch rows,
//   TMA from the sequences written by the neighbours) and its W rows through
//   a TMA ring into one 128 x 4U tcgen05 MMA (fp32 in TMEM, two accumulators
//   so step t+1's input part overlaps step t's cell update), and the 8 epilogue
//   warps -- one thread per batch row and half of the CTA's units -- apply the
//   LSTM cell to the accumulator row (c in fp32 global state, h written bf16 into the layer's
//   [B][T][hd] output, which is the next layer's input and, for the top
//   layer, H_enc / H_dec itself).
//
// LSTM cell (PyTorch gate order, reading N1 in DESIGN.md; oracle
// oracle/lstm_oracle.py): gates = W_ih x_t + W_hh h_{t-1} + b,
//   c_t = sigma(f) c_{t-1} + sigma(i) tanh(g),  h_t = sigma(o) tanh(c_t).
// The decoder's layer l starts from the encoder's layer-l state at source
// step src_len[b] - 1 (reading N3), captured by the encoder's epilogue.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/attn_softmax.h"
#include "ptx.cuh"

attn_status_t attn_set_error(attn_status_t code, const char* msg);

namespace attnsm {

constexpr int LS_THREADS = 320;   // warps 0-7 cell epilogue, warp 8 TMA producer + TMEM, warp 9 MMA
constexpr int LS_RING = 192 * 1024;
constexpr int LS_MAXST = 8;
constexpr int LS_SMEM = LS_RING + 1024 + 512;
constexpr int LS_MAXL = 8;

struct LsLayer {
  CUtensorMap m_x;          // input sequence [B][T][in] bf16, box {64, 1, 128}
  CUtensorMap m_h;          // this layer's output sequence [B][T][hd], box {64, 1, 128}
  CUtensorMap m_h0;         // initial h [B][hd] bf16, box {64, 128} (decoder)
  CUtensorMap m_w;          // packed W [4hd][in + hd] bf16, box {64, ntile}
  const float* bias;        // packed b [4hd] fp32
  __nv_bfloat16* h_out;     // [B][T][hd]
  float* c;                 // running cell state [B][hd]
  const float* c0;          // initial c [B][hd] (decoder) or NULL (zero)
  __nv_bfloat16* h_cap;     // [B][hd]: h at step cap[b] (encoder) or NULL
  float* c_cap;             // [B][hd]: c at step cap[b]
  int in;                   // input width (embedding size for layer 0, else hd)
};

struct alignas(64) LsParams {
  LsLayer layer[LS_MAXL];
  int L, B, T, hd, G, ntile;
  int has_init;             // h0 / c0 given (decoder)
  const int* cap;           // [B] capture step, or NULL
  unsigned* done;           // [L][T]: CTAs of (l, t) that published h_t
};

// tanh.approx.f32 (one MUFU op, ~2^-11 relative error, below the bf16
// rounding of h); sigma(x) = (1 + tanh(x / 2)) / 2
__device__ __forceinline__ float ls_tanh(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ls_sigmoid(float x) { return fmaf(0.5f, ls_tanh(0.5f * x), 0.5f); }

__device__ __forceinline__ void ls_wait_geq(const unsigned* p, unsigned target) {
  if (ld_acquire_gpu(p) >= target) return;
  while (ld_acquire_gpu(p) < target) __nanosleep(32);
}

__global__ void __launch_bounds__(LS_THREADS, 1) lstm_wavefront_kernel(const __grid_constant__ LsParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + LS_RING);
  uint64_t* full = bars;                 // [LS_MAXST]
  uint64_t* empty = full + LS_MAXST;     // [LS_MAXST]
  uint64_t* tfull = empty + LS_MAXST;    // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();
  const int l = blockIdx.x / P.G, g = blockIdx.x % P.G;
  const LsLayer& Ly = P.layer[l];
  const int kin = Ly.in / 64, khd = P.hd / 64;
  const uint32_t bbytes = (uint32_t)P.ntile * 128;
  const uint32_t stage = 16384 + bbytes;
  const int nst = min(LS_MAXST, (int)(LS_RING / stage));
  const uint32_t tcols = P.ntile <= 16 ? 32 : (P.ntile <= 64 ? 128 : (P.ntile <= 128 ? 256 : 512));

  if (warp == 8) {
    if (lane == 0) {
      for (int i = 0; i < LS_MAXST; ++i) {
        mbar_init(&full[i], 1);
        mbar_init(&empty[i], 1);
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(&tfull[i], 1);
        mbar_init(&tempty[i], 8);
      }
      fence_barrier_init();
      tma_prefetch_desc(&Ly.m_x);
      tma_prefetch_desc(&Ly.m_h);
      tma_prefetch_desc(&Ly.m_w);
    }
    __syncwarp();
    tmem_alloc(tmem_slot, tcols);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 8) {
    // ---------------- TMA producer: the step's [x_t | h_{t-1}] and W k-blocks
    int s = 0;
    uint32_t ph = 0;
    // Per step the input part (x_t, ready once layer l-1 has published step t,
    // usually long before) goes first and the recurrent part (h_{t-1}) last,
    // and each stage's W block is requested before waiting for the flag its A
    // block needs: only the h_{t-1} loads sit on the recurrence's critical path.
    for (int t = 0; t < P.T; ++t) {
      const int nk = kin + ((t > 0 || P.has_init) ? khd : 0);
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        if (lane == 0) {
          uint8_t* sa = ring + s * stage;
          mbar_arrive_expect_tx(&full[s], stage);
          tma_load_2d(sa + 16384, &Ly.m_w, &full[s], kb * 64, g * P.ntile);
          if (kb == 0 && l > 0) {
            ls_wait_geq(P.done + (size_t)(l - 1) * P.T + t, (unsigned)P.G);
            fence_proxy_async_global();
          }
          if (kb == kin && t > 0) {
            ls_wait_geq(P.done + (size_t)l * P.T + t - 1, (unsigned)P.G);
            fence_proxy_async_global();
          }
          if (kb < kin) tma_load_3d(sa, &Ly.m_x, &full[s], kb * 64, t, 0);
          else if (t > 0) tma_load_3d(sa, &Ly.m_h, &full[s], (kb - kin) * 64, t - 1, 0);
          else tma_load_2d(sa, &Ly.m_h0, &full[s], (kb - kin) * 64, 0);
        }
        __syncwarp();
        if (++s == nst) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 9) {
    // ---------------- MMA issuer: gates[128 rows, 4U] = [x_t | h_{t-1}] W_slice^T
    int s = 0;
    uint32_t ph = 0;
    const uint32_t idesc = umma_idesc_bf16(128, P.ntile, 0, 0);
    for (int t = 0; t < P.T; ++t) {
      const int acc = t & 1, use = t >> 1;
      if (use > 0) mbar_wait(&tempty[acc], (use - 1) & 1);
      tc_fence_after();
      const int nk = kin + ((t > 0 || P.has_init) ? khd : 0);
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = smem_u32(ring + s * stage);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tmem_base + acc * P.ntile, umma_sdesc(sa + k * 32, 16, 1024),
                      umma_sdesc(sa + 16384 + k * 32, 16, 1024), idesc, (kb | k) ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == nst) { s = 0; ph ^= 1; }
      }
      if (elect_one()) umma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else {
    // ---------------- LSTM cell (warps 0-7): warp w takes batch rows 32 (w % 4)..
    // (its TMEM lane quarter) and half w / 4 of the CTA's units; thread = row
    const uint32_t q = warp & 3, hh = warp >> 2;
    const int r = (int)(q * 32 + lane);
    const bool row_ok = r < P.B;
    const int U = P.ntile / 4;
    const int nc = P.ntile / 64;              // 32-column chunks (8 units) per warp
    const int u_base = g * U + (int)hh * (U / 2);
    const int cap = (P.cap && row_ok) ? P.cap[r] : -1;
    const uint32_t tq = tmem_base + ((q * 32u) << 16) + hh * (P.ntile / 2);
    const size_t crow = (size_t)(row_ok ? r : 0) * P.hd;
    for (int t = 0; t < P.T; ++t) {
      const int acc = t & 1, use = t >> 1;
      // c_{t-1} of this row's units, read before the accumulator wait
      float cp[2][8];
      for (int cc = 0; cc < nc; ++cc) {
        const int u0 = u_base + cc * 8;
        if (t > 0 || Ly.c0) {
          const float4* src = reinterpret_cast<const float4*>((t > 0 ? Ly.c : Ly.c0) + crow + u0);
          const float4 a = src[0], b = src[1];
          cp[cc][0] = a.x; cp[cc][1] = a.y; cp[cc][2] = a.z; cp[cc][3] = a.w;
          cp[cc][4] = b.x; cp[cc][5] = b.y; cp[cc][6] = b.z; cp[cc][7] = b.w;
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) cp[cc][k] = 0.f;
        }
      }
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
      for (int cc = 0; cc < nc; ++cc) {   // 8 units per 32 accumulator columns
        float v[32];
        tmem_ld32(tq + acc * P.ntile + cc * 32, v);
        const int u0 = u_base + cc * 8;
        const float4* b4 = reinterpret_cast<const float4*>(Ly.bias + 4 * u0);
        float hc[8], cn[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float4 bb = __ldg(b4 + k);
          const float gi = ls_sigmoid(v[4 * k] + bb.x);
          const float gf = ls_sigmoid(v[4 * k + 1] + bb.y);
          const float gg = ls_tanh(v[4 * k + 2] + bb.z);
          const float go = ls_sigmoid(v[4 * k + 3] + bb.w);
          cn[k] = fmaf(gf, cp[cc][k], gi * gg);
          hc[k] = go * ls_tanh(cn[k]);
        }
        if (row_ok) {
          float4* cdst = reinterpret_cast<float4*>(Ly.c + (size_t)r * P.hd + u0);
          const float4 c_lo = make_float4(cn[0], cn[1], cn[2], cn[3]);
          const float4 c_hi = make_float4(cn[4], cn[5], cn[6], cn[7]);
          cdst[0] = c_lo;
          cdst[1] = c_hi;
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            __nv_bfloat162 h2 = __floats2bfloat162_rn(hc[2 * e], hc[2 * e + 1]);
            w[e] = *reinterpret_cast<uint32_t*>(&h2);
          }
          const uint4 hv = make_uint4(w[0], w[1], w[2], w[3]);
          *reinterpret_cast<uint4*>(Ly.h_out + ((size_t)r * P.T + t) * P.hd + u0) = hv;
          if (t == cap) {
            *reinterpret_cast<uint4*>(Ly.h_cap + (size_t)r * P.hd + u0) = hv;
            float4* cc4 = reinterpret_cast<float4*>(Ly.c_cap + (size_t)r * P.hd + u0);
            cc4[0] = c_lo;
            cc4[1] = c_hi;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      // publish (l, t): every epilogue thread's h / c stores, then one release
      named_bar_sync(1, 256);
      if (threadIdx.x == 0) {
        __threadfence();
        red_release_gpu_add(P.done + (size_t)l * P.T + t, 1u);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 8) tmem_dealloc(tmem_base, tcols);
}

// layer packing: packed row 4u + q = [W_ih[q hd + u] | W_hh[q hd + u]], b likewise (fp32)
__global__ void lstm_pack_kernel(const __nv_bfloat16* __restrict__ W_ih, const __nv_bfloat16* __restrict__ W_hh,
                                 const __nv_bfloat16* __restrict__ b, int in, int hd,
                                 __nv_bfloat16* __restrict__ Wp, float* __restrict__ bp) {
  const int p = blockIdx.x;             // packed row
  const int u = p >> 2, q = p & 3;
  const int src = q * hd + u;
  const int K = in + hd;
  for (int k = threadIdx.x; k < K; k += blockDim.x)
    Wp[(size_t)p * K + k] = k < in ? W_ih[(size_t)src * in + k] : W_hh[(size_t)src * hd + (k - in)];
  if (threadIdx.x == 0) bp[p] = __bfloat162float(b[src]);
}

// X[b][t][:] = E[ids[b][t]][:]  (16-byte vectors; e % 8 == 0)
__global__ void embed_kernel(const int* __restrict__ ids, const __nv_bfloat16* __restrict__ E, int e,
                             long long rows, __nv_bfloat16* __restrict__ X) {
  const int v8 = e / 8;
  const long long n = rows * v8;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long row = i / v8;
    const int k = (int)(i % v8);
    reinterpret_cast<uint4*>(X)[row * v8 + k] =
        __ldg(reinterpret_cast<const uint4*>(E) + (long long)ids[row] * v8 + k);
  }
}

// input feeding (HybridNMTIF): X[b][:] = [E[ids[b][t]] | Htilde[b][t-1]] (0 at t = 0)
__global__ void if_input_kernel(const int* __restrict__ ids, int N, int t,
                                const __nv_bfloat16* __restrict__ E, int e,
                                const __nv_bfloat16* __restrict__ Hc, int hd, int B,
                                __nv_bfloat16* __restrict__ X) {
  const int w8 = (e + hd) / 8;
  const long long n = (long long)B * w8;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(i / w8), k = (int)(i % w8);
    uint4 v;
    if (k < e / 8) {
      v = __ldg(reinterpret_cast<const uint4*>(E) + (long long)ids[(long long)b * N + t] * (e / 8) + k);
    } else if (t > 0) {
      v = reinterpret_cast<const uint4*>(Hc + ((long long)b * N + t - 1) * hd)[k - e / 8];
    } else {
      v = make_uint4(0u, 0u, 0u, 0u);
    }
    reinterpret_cast<uint4*>(X)[i] = v;
  }
}

}  // namespace attnsm

// internal entry of attn_softmax.cu: one step of Eqs. 1-4 for the IF decoder
size_t attn_internal_step_ws(int B, int M, int d);
attn_status_t attn_internal_step_attention(int B, int M, int d, const void* h, const void* S,
                                           const int* src_len_dev, const void* W_c, void* out,
                                           long long ld_out, void* ws, cudaStream_t stream);

using namespace attnsm;

namespace {

attn_status_t lfail(attn_status_t code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return attn_set_error(code, buf);
}
#define LS_CUDA(expr)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess) return lfail(ATTN_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

typedef CUresult (*PFN_encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                               CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                               CUtensorMapFloatOOBfill);
PFN_encode encoder_fn() {
  static PFN_encode fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encode>(p);
  });
  return fn;
}
// bf16 tensor map, 128-byte swizzle, zero fill out of bounds
attn_status_t map_bf16(CUtensorMap* m, const void* ptr, int rank, const cuuint64_t* dims,
                       const cuuint64_t* strides, const cuuint32_t* box) {
  PFN_encode enc = encoder_fn();
  if (!enc) return lfail(ATTN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), dims, strides, box,
                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return lfail(ATTN_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return ATTN_OK;
}
// [B][T][w] sequence, box {64, 1, 128}
attn_status_t map_seq(CUtensorMap* m, const void* p, int w, int T, int B) {
  cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)T, (cuuint64_t)B};
  cuuint64_t str[2] = {(cuuint64_t)w * 2, (cuuint64_t)w * 2 * T};
  cuuint32_t box[3] = {64, 1, 128};
  return map_bf16(m, p, 3, dims, str, box);
}
attn_status_t map_mat(CUtensorMap* m, const void* p, int cols, int rows, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  return map_bf16(m, p, 2, dims, str, box);
}

size_t al(size_t x) { return (x + 255) / 256 * 256; }

struct LsPlan {
  size_t xs, xt, inter, c, hcap, ccap, lens, done_enc, done_dec, total;
  int U, G, ntile;
};

attn_status_t check_lstm(const attn_lstm_shape_t* s) {
  if (!s) return lfail(ATTN_ERR_INVALID_ARG, "lstm shape is NULL");
  if (s->batch < 1 || s->batch > 128)
    return lfail(ATTN_ERR_UNSUPPORTED, "lstm: batch %d outside [1, 128] (one 128-row MMA tile per step)", s->batch);
  if (s->src_len < 1 || s->tgt_len < 1) return lfail(ATTN_ERR_SHAPE, "lstm: src_len / tgt_len must be >= 1");
  if (s->layers < 1 || s->layers > LS_MAXL) return lfail(ATTN_ERR_UNSUPPORTED, "lstm: layers must be in [1, %d]", LS_MAXL);
  if (s->emb % 64 || s->hidden % 64 || s->emb < 64 || s->hidden < 64)
    return lfail(ATTN_ERR_UNSUPPORTED, "lstm: emb (%d) and hidden (%d) must be multiples of 64", s->emb, s->hidden);
  if (s->vocab_src < 1 || s->vocab_tgt < 1) return lfail(ATTN_ERR_SHAPE, "lstm: vocabularies must be non-empty");
  return ATTN_OK;
}

LsPlan plan_lstm(const attn_lstm_shape_t* s) {
  LsPlan p;
  const int B = s->batch, M = s->src_len, N = s->tgt_len, e = s->emb, hd = s->hidden, L = s->layers;
  const int Tm = std::max(M, N);
  // units per CTA: the largest of 32 / 16 whose L x (hd / U) CTAs fit the SMs
  // (fixed 148 so the plan does not depend on the device)
  p.U = (L * (hd / 32) <= 148) ? 32 : 16;
  p.G = hd / p.U;
  p.ntile = 4 * p.U;
  size_t o = 0;
  auto take = [&](size_t b) { size_t r = o; o += al(b); return r; };
  p.xs = take((size_t)B * M * e * 2);
  p.xt = take((size_t)B * N * e * 2);
  p.inter = take((size_t)std::max(L - 1, 1) * B * Tm * hd * 2);
  p.c = take((size_t)L * B * hd * 4);
  p.hcap = take((size_t)L * B * hd * 2);
  p.ccap = take((size_t)L * B * hd * 4);
  p.lens = take((size_t)B * 4);
  p.done_enc = take((size_t)L * M * 4);
  p.done_dec = take((size_t)L * N * 4);
  p.total = o;
  return p;
}

}  // namespace

extern "C" size_t attn_lstm_workspace_size(const attn_lstm_shape_t* s) {
  if (check_lstm(s) != ATTN_OK) return 0;
  return plan_lstm(s).total;
}

extern "C" size_t attn_lstm_packed_bytes(int in, int hidden) {
  return (size_t)4 * hidden * (in + hidden) * 2;
}

extern "C" attn_status_t attn_lstm_pack_layer(int in, int hidden, const void* W_ih, const void* W_hh,
                                              const void* b, void* W_packed, float* b_packed,
                                              void* stream) {
  if (in < 1 || hidden < 1) return lfail(ATTN_ERR_SHAPE, "lstm_pack: in / hidden must be >= 1");
  if (!W_ih || !W_hh || !b || !W_packed || !b_packed) return lfail(ATTN_ERR_INVALID_ARG, "lstm_pack: NULL buffer");
  lstm_pack_kernel<<<4 * hidden, 256, 0, (cudaStream_t)stream>>>(
      static_cast<const __nv_bfloat16*>(W_ih), static_cast<const __nv_bfloat16*>(W_hh),
      static_cast<const __nv_bfloat16*>(b), in, hidden, static_cast<__nv_bfloat16*>(W_packed), b_packed);
  LS_CUDA(cudaGetLastError());
  return ATTN_OK;
}

namespace {

// One cooperative launch of the wavefront kernel: L layers over T steps.
// Per layer: its output sequence hout [B][T][hd], running c state, optional
// initial (h0 bf16 [B][hd], c0 fp32 [B][hd]) and capture buffers.
struct RunCfg {
  int B, T, hd, L, G, ntile, in0;
  const void* X0;                 // layer-0 input [B][T][in0]
  const void* const* W;           // packed layers
  const float* const* b;
  void* hout[LS_MAXL];
  float* c[LS_MAXL];
  const void* h0[LS_MAXL];        // NULL: zero initial state (then c0 must be NULL too)
  const float* c0[LS_MAXL];
  void* hcap[LS_MAXL];            // capture at cap_dev[b] (or NULL)
  float* ccap[LS_MAXL];
  const int* cap_dev;
  unsigned* done;                 // [L][T], zeroed here
};

attn_status_t run_layers(const RunCfg& R, cudaStream_t st) {
  static LsParams P;   // large: filled under a lock
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  memset(&P, 0, sizeof(P));
  const int B = R.B, T = R.T, hd = R.hd, L = R.L;
  attn_status_t r;
  for (int l = 0; l < L; ++l) {
    LsLayer& Ly = P.layer[l];
    Ly.in = l == 0 ? R.in0 : hd;
    const void* xin = l == 0 ? R.X0 : R.hout[l - 1];
    if ((r = map_seq(&Ly.m_x, xin, Ly.in, T, B)) != ATTN_OK) return r;
    if ((r = map_seq(&Ly.m_h, R.hout[l], hd, T, B)) != ATTN_OK) return r;
    // (a dummy but valid map when there is no initial h: never loaded)
    if ((r = map_mat(&Ly.m_h0, R.h0[0] ? R.h0[l] : R.hout[l], hd, B, 128)) != ATTN_OK) return r;
    if ((r = map_mat(&Ly.m_w, R.W[l], Ly.in + hd, 4 * hd, R.ntile)) != ATTN_OK) return r;
    Ly.bias = R.b[l];
    Ly.h_out = static_cast<__nv_bfloat16*>(R.hout[l]);
    Ly.c = R.c[l];
    Ly.c0 = R.c0[l];
    Ly.h_cap = static_cast<__nv_bfloat16*>(R.hcap[l]);
    Ly.c_cap = R.ccap[l];
  }
  P.L = L; P.B = B; P.T = T; P.hd = hd; P.G = R.G; P.ntile = R.ntile;
  P.has_init = R.h0[0] ? 1 : 0;
  P.cap = R.cap_dev;
  P.done = R.done;
  LS_CUDA(cudaMemsetAsync(R.done, 0, sizeof(unsigned) * (size_t)L * T, st));
  static std::vector<int> attr_set;   // devices with the smem attribute set
  int dev = 0;
  LS_CUDA(cudaGetDevice(&dev));
  if (std::find(attr_set.begin(), attr_set.end(), dev) == attr_set.end()) {
    LS_CUDA(cudaFuncSetAttribute(lstm_wavefront_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, LS_SMEM));
    attr_set.push_back(dev);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(L * R.G);
  cfg.blockDim = dim3(LS_THREADS);
  cfg.dynamicSmemBytes = LS_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;   // every CTA resident: the step flags cannot deadlock
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  LS_CUDA(cudaLaunchKernelEx(&cfg, lstm_wavefront_kernel, P));
  return ATTN_OK;
}

// one side (encoder or decoder): L layers over T steps as one cooperative launch
attn_status_t run_side(const attn_lstm_shape_t* s, const LsPlan& p, int T, const void* X0,
                       const void* const* W, const float* const* b, void* H_top, char* ws,
                       bool decoder, const int* cap_dev, unsigned* done, cudaStream_t st) {
  RunCfg R;
  memset(&R, 0, sizeof(R));
  const int B = s->batch, hd = s->hidden, L = s->layers;
  R.B = B; R.T = T; R.hd = hd; R.L = L; R.G = p.G; R.ntile = p.ntile; R.in0 = s->emb;
  R.X0 = X0; R.W = W; R.b = b; R.cap_dev = decoder ? nullptr : cap_dev; R.done = done;
  __nv_bfloat16* inter = reinterpret_cast<__nv_bfloat16*>(ws + p.inter);
  for (int l = 0; l < L; ++l) {
    R.hout[l] = l == L - 1 ? H_top : (void*)(inter + (size_t)l * B * T * hd);
    R.c[l] = reinterpret_cast<float*>(ws + p.c) + (size_t)l * B * hd;
    __nv_bfloat16* hcap = reinterpret_cast<__nv_bfloat16*>(ws + p.hcap) + (size_t)l * B * hd;
    float* ccap = reinterpret_cast<float*>(ws + p.ccap) + (size_t)l * B * hd;
    R.h0[l] = decoder ? hcap : nullptr;
    R.c0[l] = decoder ? ccap : nullptr;
    R.hcap[l] = decoder ? nullptr : hcap;
    R.ccap[l] = decoder ? nullptr : ccap;
  }
  return run_layers(R, st);
}

}  // namespace

extern "C" attn_status_t attn_encoder_decoder_fwd(
    const attn_lstm_shape_t* s, const int32_t* src_ids, const int32_t* tgt_ids,
    const int32_t* src_lens_host, const void* E_src, const void* E_tgt,
    const void* const* enc_W, const float* const* enc_b, const void* const* dec_W,
    const float* const* dec_b, void* H_enc, void* H_dec, void* workspace, size_t workspace_bytes,
    void* stream) {
  attn_status_t r = check_lstm(s);
  if (r != ATTN_OK) return r;
  if (!src_ids || !tgt_ids || !src_lens_host || !E_src || !E_tgt || !enc_W || !enc_b || !dec_W ||
      !dec_b || !H_enc || !H_dec || !workspace)
    return lfail(ATTN_ERR_INVALID_ARG, "encoder_decoder_fwd: NULL argument");
  for (int l = 0; l < s->layers; ++l)
    if (!enc_W[l] || !enc_b[l] || !dec_W[l] || !dec_b[l])
      return lfail(ATTN_ERR_INVALID_ARG, "encoder_decoder_fwd: layer %d weights are NULL", l);
  for (int i = 0; i < s->batch; ++i)
    if (src_lens_host[i] < 1 || src_lens_host[i] > s->src_len)
      return lfail(ATTN_ERR_SHAPE, "src_lens_host[%d] = %d outside [1, M = %d]", i, src_lens_host[i], s->src_len);
  const LsPlan p = plan_lstm(s);
  if (workspace_bytes < p.total)
    return lfail(ATTN_ERR_WORKSPACE, "workspace_bytes = %zu < required %zu", workspace_bytes, p.total);
  int dev = 0, sms = 0;
  LS_CUDA(cudaGetDevice(&dev));
  LS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (s->layers * p.G > sms)
    return lfail(ATTN_ERR_UNSUPPORTED, "lstm: %d layers x %d CTAs exceed the %d SMs", s->layers, p.G, sms);
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = static_cast<char*>(workspace);
  const int B = s->batch, M = s->src_len, N = s->tgt_len, e = s->emb;
  // capture step src_len - 1 per sentence (host lengths -> device, stream-ordered)
  std::vector<int> cap(B);
  for (int i = 0; i < B; ++i) cap[i] = src_lens_host[i] - 1;
  int* cap_dev = reinterpret_cast<int*>(ws + p.lens);
  LS_CUDA(cudaMemcpyAsync(cap_dev, cap.data(), sizeof(int) * B, cudaMemcpyHostToDevice, st));
  // embeddings
  __nv_bfloat16* Xs = reinterpret_cast<__nv_bfloat16*>(ws + p.xs);
  __nv_bfloat16* Xt = reinterpret_cast<__nv_bfloat16*>(ws + p.xt);
  embed_kernel<<<sms * 4, 256, 0, st>>>(src_ids, static_cast<const __nv_bfloat16*>(E_src), e,
                                        (long long)B * M, Xs);
  LS_CUDA(cudaGetLastError());
  embed_kernel<<<sms * 4, 256, 0, st>>>(tgt_ids, static_cast<const __nv_bfloat16*>(E_tgt), e,
                                        (long long)B * N, Xt);
  LS_CUDA(cudaGetLastError());
  if ((r = run_side(s, p, M, Xs, enc_W, enc_b, H_enc, ws, false, cap_dev,
                    reinterpret_cast<unsigned*>(ws + p.done_enc), st)) != ATTN_OK)
    return r;
  return run_side(s, p, N, Xt, dec_W, dec_b, H_dec, ws, true, nullptr,
                  reinterpret_cast<unsigned*>(ws + p.done_dec), st);
}

// ---------------------------------------------------------------- input feeding
namespace {
struct IfPlan {
  size_t x, h, c, srclen, done, attn, total;
};
IfPlan plan_if(const attn_lstm_shape_t* s, const LsPlan& base) {
  IfPlan q;
  const int B = s->batch, hd = s->hidden, L = s->layers;
  size_t o = base.total;
  auto take = [&](size_t b) { size_t r = o; o += al(b); return r; };
  q.x = take((size_t)B * (s->emb + hd) * 2);
  q.h = take((size_t)2 * L * B * hd * 2);
  q.c = take((size_t)2 * L * B * hd * 4);
  q.srclen = take((size_t)B * 4);
  q.done = take((size_t)L * 4);
  q.attn = take(attn_internal_step_ws(B, s->src_len, hd));
  q.total = o;
  return q;
}
}  // namespace

extern "C" size_t attn_lstm_if_workspace_size(const attn_lstm_shape_t* s) {
  if (check_lstm(s) != ATTN_OK) return 0;
  const LsPlan p = plan_lstm(s);
  return plan_if(s, p).total;
}

extern "C" attn_status_t attn_encoder_decoder_if_fwd(
    const attn_lstm_shape_t* s, const int32_t* src_ids, const int32_t* tgt_ids,
    const int32_t* src_lens_host, const void* E_src, const void* E_tgt,
    const void* const* enc_W, const float* const* enc_b, const void* const* dec_W,
    const float* const* dec_b, const void* W_c, void* H_enc, void* H_dec, void* Htilde,
    void* workspace, size_t workspace_bytes, void* stream) {
  attn_status_t r = check_lstm(s);
  if (r != ATTN_OK) return r;
  if (!src_ids || !tgt_ids || !src_lens_host || !E_src || !E_tgt || !enc_W || !enc_b || !dec_W ||
      !dec_b || !W_c || !H_enc || !H_dec || !Htilde || !workspace)
    return lfail(ATTN_ERR_INVALID_ARG, "encoder_decoder_if_fwd: NULL argument");
  for (int l = 0; l < s->layers; ++l)
    if (!enc_W[l] || !enc_b[l] || !dec_W[l] || !dec_b[l])
      return lfail(ATTN_ERR_INVALID_ARG, "encoder_decoder_if_fwd: layer %d weights are NULL", l);
  if (s->src_len > 128)
    return lfail(ATTN_ERR_UNSUPPORTED, "encoder_decoder_if_fwd: M = %d > 128 (fused attention step)", s->src_len);
  for (int i = 0; i < s->batch; ++i)
    if (src_lens_host[i] < 1 || src_lens_host[i] > s->src_len)
      return lfail(ATTN_ERR_SHAPE, "src_lens_host[%d] = %d outside [1, M = %d]", i, src_lens_host[i], s->src_len);
  const LsPlan p = plan_lstm(s);
  const IfPlan q = plan_if(s, p);
  if (workspace_bytes < q.total)
    return lfail(ATTN_ERR_WORKSPACE, "workspace_bytes = %zu < required %zu", workspace_bytes, q.total);
  int dev = 0, sms = 0;
  LS_CUDA(cudaGetDevice(&dev));
  LS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (s->layers * p.G > sms)
    return lfail(ATTN_ERR_UNSUPPORTED, "lstm: %d layers x %d CTAs exceed the %d SMs", s->layers, p.G, sms);
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = static_cast<char*>(workspace);
  const int B = s->batch, M = s->src_len, N = s->tgt_len, e = s->emb, hd = s->hidden, L = s->layers;
  // encoder (wavefront over all source steps), capturing the state at src_len - 1
  std::vector<int> cap(B), sl(B);
  for (int i = 0; i < B; ++i) {
    cap[i] = src_lens_host[i] - 1;
    sl[i] = src_lens_host[i];
  }
  int* cap_dev = reinterpret_cast<int*>(ws + p.lens);
  int* sl_dev = reinterpret_cast<int*>(ws + q.srclen);
  LS_CUDA(cudaMemcpyAsync(cap_dev, cap.data(), sizeof(int) * B, cudaMemcpyHostToDevice, st));
  LS_CUDA(cudaMemcpyAsync(sl_dev, sl.data(), sizeof(int) * B, cudaMemcpyHostToDevice, st));
  __nv_bfloat16* Xs = reinterpret_cast<__nv_bfloat16*>(ws + p.xs);
  embed_kernel<<<sms * 4, 256, 0, st>>>(src_ids, static_cast<const __nv_bfloat16*>(E_src), e,
                                        (long long)B * M, Xs);
  LS_CUDA(cudaGetLastError());
  if ((r = run_side(s, p, M, Xs, enc_W, enc_b, H_enc, ws, false, cap_dev,
                    reinterpret_cast<unsigned*>(ws + p.done_enc), st)) != ATTN_OK)
    return r;
  // decoder with input feeding: step t needs Htilde_{t-1} = tanh(W_c [h_{t-1}; C_{t-1}])
  // (PAPER.md:75, :99), so the steps run one after another: per step one
  // wavefront launch over the L layers (T = 1), then Eqs. 1-4 for that step
  __nv_bfloat16* X = reinterpret_cast<__nv_bfloat16*>(ws + q.x);
  __nv_bfloat16* hbuf = reinterpret_cast<__nv_bfloat16*>(ws + q.h);
  float* cbuf = reinterpret_cast<float*>(ws + q.c);
  __nv_bfloat16* hcap = reinterpret_cast<__nv_bfloat16*>(ws + p.hcap);
  float* ccap = reinterpret_cast<float*>(ws + p.ccap);
  const size_t lay = (size_t)B * hd;
  for (int t = 0; t < N; ++t) {
    const int cur = t & 1, prv = cur ^ 1;
    if_input_kernel<<<sms, 256, 0, st>>>(tgt_ids, N, t, static_cast<const __nv_bfloat16*>(E_tgt), e,
                                         static_cast<const __nv_bfloat16*>(Htilde), hd, B, X);
    LS_CUDA(cudaGetLastError());
    RunCfg R;
    memset(&R, 0, sizeof(R));
    R.B = B; R.T = 1; R.hd = hd; R.L = L; R.G = p.G; R.ntile = p.ntile; R.in0 = e + hd;
    R.X0 = X; R.W = dec_W; R.b = dec_b; R.done = reinterpret_cast<unsigned*>(ws + q.done);
    for (int l = 0; l < L; ++l) {
      R.hout[l] = hbuf + ((size_t)cur * L + l) * lay;
      R.c[l] = cbuf + ((size_t)cur * L + l) * lay;
      R.h0[l] = t == 0 ? (const void*)(hcap + l * lay) : (const void*)(hbuf + ((size_t)prv * L + l) * lay);
      R.c0[l] = t == 0 ? (const float*)(ccap + l * lay) : (const float*)(cbuf + ((size_t)prv * L + l) * lay);
    }
    if ((r = run_layers(R, st)) != ATTN_OK) return r;
    const void* htop = R.hout[L - 1];
    LS_CUDA(cudaMemcpy2DAsync(static_cast<char*>(H_dec) + (size_t)t * hd * 2, (size_t)N * hd * 2, htop,
                              (size_t)hd * 2, (size_t)hd * 2, B, cudaMemcpyDeviceToDevice, st));
    if ((r = attn_internal_step_attention(B, M, hd, htop, H_enc, sl_dev, W_c,
                                          static_cast<char*>(Htilde) + (size_t)t * hd * 2,
                                          (long long)N * hd, ws + q.attn, st)) != ATTN_OK)
      return r;
  }
  return ATTN_OK;
}
