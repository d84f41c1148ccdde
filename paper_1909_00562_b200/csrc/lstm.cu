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
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/attn_softmax.h"
#include "nvtx.cuh"
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
  __nv_bfloat16* gates_seq; // training: [B][T][4hd] post-activation i, f, g, o (packed order) or NULL
  float* c_seq;             // training: [B][T][hd] c_t
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
  // (an unbounded spin on purpose: the bounded spin_wait_geq of ptx.cuh made
  // the wavefront kernels 5-8% slower -- their per-step flag waits are short
  // and on the recurrence's critical path)
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
        float hc[8], cn[8], ga[32];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float4 bb = __ldg(b4 + k);
          const float gi = ls_sigmoid(v[4 * k] + bb.x);
          const float gf = ls_sigmoid(v[4 * k + 1] + bb.y);
          const float gg = ls_tanh(v[4 * k + 2] + bb.z);
          const float go = ls_sigmoid(v[4 * k + 3] + bb.w);
          ga[4 * k] = gi; ga[4 * k + 1] = gf; ga[4 * k + 2] = gg; ga[4 * k + 3] = go;
          cn[k] = fmaf(gf, cp[cc][k], gi * gg);
          hc[k] = go * ls_tanh(cn[k]);
        }
        if (row_ok && Ly.gates_seq) {
          // training: the cell's activations (packed gate order) and c_t for the backward
          uint4* gdst = reinterpret_cast<uint4*>(Ly.gates_seq + ((size_t)r * P.T + t) * 4 * P.hd + 4 * u0);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              __nv_bfloat162 h2 = __floats2bfloat162_rn(ga[8 * q4 + 2 * e], ga[8 * q4 + 2 * e + 1]);
              w[e] = *reinterpret_cast<uint32_t*>(&h2);
            }
            gdst[q4] = make_uint4(w[0], w[1], w[2], w[3]);
          }
          float4* cs = reinterpret_cast<float4*>(Ly.c_seq + ((size_t)r * P.T + t) * P.hd + u0);
          cs[0] = make_float4(cn[0], cn[1], cn[2], cn[3]);
          cs[1] = make_float4(cn[4], cn[5], cn[6], cn[7]);
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

// ============================================================== backward (NEXT-3 training)
// The reverse wavefront ("the alternation ... on the backward
// process goes in a similar but opposite direction"): layer-step (l, t)
// needs (l+1, t) (the gradient w.r.t. its output h_t, from the layer above)
// and (l, t+1) (W_hh^T dz of the later step and the cell-state carry), so
// the top layer starts at t = T-1 and the others follow.  One cooperative
// launch per side, CTA (l, g) again owning units [32 g, 32 g + 32) of layer
// l.  Per step:
//   E  (8 epilogue warps, thread = batch row, 16 units each): the cell's
//      backward from the saved activations (i, f, g, o bf16, c fp32) --
//      dc = dc_next + dh o (1 - tanh^2 c_t), dz = [dc g i(1-i), dc c_{t-1}
//      f(1-f), dc i (1-g^2), dh tanh(c_t) o(1-o)], dc_next = dc f -- dz
//      written bf16 (packed gate order) into dG_l [B][T][4hd]; publish.
//   G  once every CTA of the layer has published step t: the CTA's 64-column
//      slices of [dx_t | dh_{t-1}] = dz_t W_l (M = B rows, K = 4hd, N = 64;
//      dz K-major, W_l as the MN-major B), fp32 into dx_out [B][T][in] (the
//      layer below's upstream gradient, or the embeddings') and dh_rec
//      [2][B][hd]; publish.
// dW_l = sum_t dz_t^T [x_t | h_{t-1}] and db_l are one large GEMM / column
// sum after the kernel (attn_encoder_decoder_bwd).
struct LbLayer {
  CUtensorMap m_dg;            // dG_l [B][T][4hd] bf16, box {64, 1, 128}
  CUtensorMap m_w;             // W_l packed [4hd][in + hd] bf16, box {64 cols, 64 rows} (MN-major B)
  __nv_bfloat16* dg;           // dG_l
  const __nv_bfloat16* gates;  // saved activations [B][T][4hd]
  const float* c_seq;          // saved c_t [B][T][hd]
  const float* c0;             // initial c [B][hd] or NULL (zero)
  const __nv_bfloat16* dh_top; // top layer: dL/dh_t [B][T][hd] bf16 (the stage's dH_enc / dH_dec)
  const float* dx_above;       // other layers: layer l+1's dx_out [B][T][hd]
  float* dx_out;               // dL/dx_t of this layer's input [B][T][in] fp32
  float* dh_rec;               // [2][B][hd] fp32: (W_hh^T dz_{t+1}) for step t
  float* dh0_out;              // [B][hd] gradient w.r.t. the initial state (decoder) or NULL
  float* dc0_out;
  const float* inj_dh;         // encoder: the decoder's initial-state gradient of this layer, added at
  const float* inj_dc;         //   t = cap[b] (or NULL)
  int in;
};
struct alignas(64) LbParams {
  LbLayer layer[LS_MAXL];
  int L, B, T, hd, G;
  int C;                       // cluster size (1, 2, 4): the CTAs of a cluster share each dz k-block
                               // (one of them loads it, TMA multicast to all)
  int Gk;                      // K split (1, 2, 4): CTA g takes the 4hd / Gk gate columns [kh 4hd / Gk, ..)
                               // of the product, kh = g / (G / Gk), over 64 Gk-column tiles, and writes
                               // partial kh of dx / dh_rec; the readers add the Gk partials in order
  long long dx_kstride;        // floats between the partials of dx_out / dx_above
  long long rec_kstride;       // floats between the partials of dh_rec
  const int* cap;              // [B] (encoder) or NULL
  unsigned* dgdone;            // [L][T] CTAs that wrote dz of (l, t)
  unsigned* outdone;           // [L][T] CTAs that stored their [dx | dh] slices of (l, t)
  long long* trace;            // debug (option "lstm_trace"): [L G][T][8] globaltimer stamps, NULL = off
};
__device__ __forceinline__ long long lb_gt() {
  long long c;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(c));
  return c;
}
#define LB_TRACE(t, i)                                                              \
  do {                                                                              \
    if (P.trace) P.trace[((long long)blockIdx.x * P.T + (t)) * 8 + (i)] = lb_gt();  \
  } while (0)

constexpr int LB_STAGE = 24 * 1024;   // dz block 16 KB + W block 8 KB
constexpr int LB_STAGES = 8;
constexpr int LB_SMEM = LB_STAGES * LB_STAGE + 1024 + 512;

__global__ void __launch_bounds__(LS_THREADS, 1) lstm_bwd_kernel(const __grid_constant__ LbParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + LB_STAGES * LB_STAGE);
  uint64_t* full = bars;
  uint64_t* empty = full + LB_STAGES;
  uint64_t* tfull = empty + LB_STAGES;   // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();
  const int l = blockIdx.x / P.G, g = blockIdx.x % P.G;
  const LbLayer& Ly = P.layer[l];
  const int hd = P.hd, T = P.T, U = hd / P.G;
  const int Gk = P.Gk, Gn = P.G / Gk, kh = g / Gn, gn = g % Gn;
  const int NT = 64 * Gk;                      // output tile width
  const int ncol = (Ly.in + hd) / NT;          // output tiles of the layer
  const int kb_n = 4 * hd / 64 / Gk;           // k-blocks (gate columns) of this CTA's K range
  const int kb0 = kh * kb_n;
  const uint32_t stage_bytes = 16384u + 8192u * (uint32_t)Gk;
  const int nst = LB_STAGES * LB_STAGE / (int)stage_bytes;
  const int C = P.C;
  const uint32_t crank = C > 1 ? cluster_ctarank() : 0;
  const uint16_t cmask = (uint16_t)((1u << C) - 1u);
  if (warp == 8) {
    if (lane == 0) {
      for (int i = 0; i < nst; ++i) {
        mbar_init(&full[i], 1);
        mbar_init(&empty[i], C);   // every CTA of the cluster reads the multicast dz block
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(&tfull[i], 1);
        mbar_init(&tempty[i], 8);
      }
      fence_barrier_init();
      tma_prefetch_desc(&Ly.m_dg);
      tma_prefetch_desc(&Ly.m_w);
    }
    __syncwarp();
    tmem_alloc(tmem_slot, 2 * NT);
  }
  tc_fence_before();
  if (C > 1) cluster_sync();   // the peers' barriers exist before any multicast
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 8) {
    // ---------------- TMA producer: per step, this CTA's tiles x its k-blocks
    int s = 0;
    uint32_t ph = 0;
    for (int t = T - 1; t >= 0; --t) {
      bool first = true;
      for (int ct = gn; ct < ncol; ct += Gn) {
        for (int kk = 0; kk < kb_n; ++kk) {
          const int kb = kb0 + kk;
          if (C > 1) mbar_wait_cluster(&empty[s], ph ^ 1);
          else mbar_wait(&empty[s], ph ^ 1);
          if (lane == 0) {
            uint8_t* st = ring + s * stage_bytes;
            mbar_arrive_expect_tx(&full[s], stage_bytes);
            for (int a = 0; a < Gk; ++a)
              tma_load_2d(st + 16384 + 8192 * a, &Ly.m_w, &full[s], ct * NT + 64 * a, kb * 64);
            if (kk % C == (int)crank) {   // this CTA's share of the cluster's dz blocks
              if (first) {   // dz of step t: every CTA of the layer has written its units
                ls_wait_geq(P.dgdone + (size_t)l * T + t, (unsigned)P.G);
                fence_proxy_async_global();
                first = false;
                LB_TRACE(t, 2);
              }
              if (C > 1) tma_load_3d_mc(st, &Ly.m_dg, &full[s], kb * 64, t, 0, cmask);
              else tma_load_3d(st, &Ly.m_dg, &full[s], kb * 64, t, 0);
            }
          }
          __syncwarp();
          if (++s == nst) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 9) {
    // ---------------- MMA issuer: out[128, NT] = dz_t[:, K range] (K-major) x W_l[K range, tile] (MN-major)
    int s = 0;
    uint32_t ph = 0;
    int n = 0;
    const uint32_t idesc = umma_idesc_bf16(128, NT, 0, 1);
    for (int t = T - 1; t >= 0; --t) {
      for (int ct = gn; ct < ncol; ct += Gn, ++n) {
        const int acc = n & 1, use = n >> 1;
        if (use > 0) mbar_wait(&tempty[acc], (use - 1) & 1);
        tc_fence_after();
        for (int kb = 0; kb < kb_n; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          if (kb == 0 && lane == 0) LB_TRACE(t, 3);
          if (elect_one()) {
            const uint32_t sa = smem_u32(ring + s * stage_bytes);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16(tmem_base + acc * NT, umma_sdesc(sa + k * 32, 16, 1024),
                        umma_sdesc(sa + 16384 + k * 2048, 8192, 1024), idesc, (kb | k) ? 1u : 0u);
            if (C > 1) umma_commit_mc(&empty[s], cmask);   // frees the stage in every peer
            else umma_commit(&empty[s]);
          }
          __syncwarp();
          if (++s == nst) { s = 0; ph ^= 1; }
        }
        if (elect_one()) umma_commit(&tfull[acc]);
        __syncwarp();
        if (lane == 0) LB_TRACE(t, 4);
      }
    }
  } else {
    // ---------------- cell backward (E) and the slices' epilogue (G), warps 0-7
    const uint32_t q = warp & 3, hh = warp >> 2;
    const int r = (int)(q * 32 + lane);
    const bool row_ok = r < P.B;
    const int rr = row_ok ? r : 0;
    const int u_base = g * U + (int)hh * (U / 2);   // 16 units per thread (U = 32)
    const int nu = U / 2;
    const int cap = (P.cap && row_ok) ? P.cap[r] : -1;
    float dcc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) dcc[k] = 0.f;
    int n = 0;
    // the saved activations of step t (i, f, g, o, c_t, c_{t-1}) do not depend on
    // the wavefront: they are loaded for step t - 1 while step t's GEMM runs
    uint4 pg[2][4];
    float4 pc[2][2], pp[2][2];
    auto prefetch = [&](int t) {
      if (!row_ok || t < 0) return;
#pragma unroll
      for (int i2 = 0; i2 < 2; ++i2) {
        if (i2 * 8 >= nu) break;
        const int u0 = u_base + i2 * 8;
        const uint4* g4 = reinterpret_cast<const uint4*>(Ly.gates + ((size_t)r * T + t) * 4 * hd + 4 * u0);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) pg[i2][q4] = g4[q4];
        const float4* c4 = reinterpret_cast<const float4*>(Ly.c_seq + ((size_t)r * T + t) * hd + u0);
        pc[i2][0] = c4[0];
        pc[i2][1] = c4[1];
        if (t > 0) {
          const float4* p4 = reinterpret_cast<const float4*>(Ly.c_seq + ((size_t)r * T + t - 1) * hd + u0);
          pp[i2][0] = p4[0];
          pp[i2][1] = p4[1];
        } else if (Ly.c0) {
          const float4* p4 = reinterpret_cast<const float4*>(Ly.c0 + (size_t)r * hd + u0);
          pp[i2][0] = p4[0];
          pp[i2][1] = p4[1];
        } else {
          pp[i2][0] = pp[i2][1] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    };
    prefetch(T - 1);
    for (int t = T - 1; t >= 0; --t) {
      // ---- E: wait for the gradient w.r.t. h_t (layer above) and W_hh^T dz_{t+1} (own layer)
      if (threadIdx.x == 0) {
        if (l < P.L - 1) ls_wait_geq(P.outdone + (size_t)(l + 1) * T + t, (unsigned)P.G);
        if (t < T - 1) ls_wait_geq(P.outdone + (size_t)l * T + t + 1, (unsigned)P.G);
        __threadfence();
      }
      named_bar_sync(1, 256);
      if (threadIdx.x == 0) LB_TRACE(t, 0);
      if (row_ok) {
        // dL/dh_t of this row's units: every load first (the dz stores below
        // could alias them for the compiler), added in a fixed order:
        // (dh_top | 0 + dx_above partials) + dh_rec partials
        const int ni2 = nu > 8 ? 2 : 1;
        float dhs[2][8];
#pragma unroll
        for (int i2 = 0; i2 < 2; ++i2)
#pragma unroll
          for (int k = 0; k < 8; ++k) dhs[i2][k] = 0.f;
        auto add8 = [](float (&d)[8], const float4& a, const float4& b) {
          d[0] += a.x; d[1] += a.y; d[2] += a.z; d[3] += a.w; d[4] += b.x; d[5] += b.y; d[6] += b.z; d[7] += b.w;
        };
        if (Ly.dh_top) {
#pragma unroll
          for (int i2 = 0; i2 < 2; ++i2) {
            if (i2 >= ni2) break;
            const uint4 hv = *reinterpret_cast<const uint4*>(Ly.dh_top + ((size_t)r * T + t) * hd + u_base + 8 * i2);
            const uint32_t w4[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[e]));
              dhs[i2][2 * e] = f2.x;
              dhs[i2][2 * e + 1] = f2.y;
            }
          }
        } else {
#pragma unroll
          for (int pk = 0; pk < 4; ++pk) {   // the Gk partials, in order
            if (pk >= Gk) break;
#pragma unroll
            for (int i2 = 0; i2 < 2; ++i2) {
              if (i2 >= ni2) break;
              const float4* a4 = reinterpret_cast<const float4*>(Ly.dx_above + pk * P.dx_kstride +
                                                                 ((size_t)r * T + t) * hd + u_base + 8 * i2);
              add8(dhs[i2], __ldcg(a4), __ldcg(a4 + 1));
            }
          }
        }
        if (t < T - 1) {
#pragma unroll
          for (int pk = 0; pk < 4; ++pk) {
            if (pk >= Gk) break;
#pragma unroll
            for (int i2 = 0; i2 < 2; ++i2) {
              if (i2 >= ni2) break;
              const float4* a4 = reinterpret_cast<const float4*>(Ly.dh_rec + pk * P.rec_kstride +
                                                                 ((size_t)((t + 1) & 1) * P.B + r) * hd + u_base + 8 * i2);
              add8(dhs[i2], __ldcg(a4), __ldcg(a4 + 1));
            }
          }
        }
#pragma unroll
        for (int i2 = 0; i2 < 2; ++i2) {
          const int k0 = i2 * 8;
          if (k0 >= nu) break;
          const int u0 = u_base + k0;
          float dh[8], cp[8], ct[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) dh[k] = dhs[i2][k];
          if (t == cap && Ly.inj_dh) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              dh[k] += Ly.inj_dh[(size_t)r * hd + u0 + k];
              dcc[k0 + k] += Ly.inj_dc[(size_t)r * hd + u0 + k];
            }
          }
          {
            const float4 a = pc[i2][0], b = pc[i2][1];
            ct[0] = a.x; ct[1] = a.y; ct[2] = a.z; ct[3] = a.w; ct[4] = b.x; ct[5] = b.y; ct[6] = b.z; ct[7] = b.w;
            const float4 c = pp[i2][0], d = pp[i2][1];
            cp[0] = c.x; cp[1] = c.y; cp[2] = c.z; cp[3] = c.w; cp[4] = d.x; cp[5] = d.y; cp[6] = d.z; cp[7] = d.w;
          }
          // saved activations of these 8 units: 32 bf16 in packed order (4u + q)
          float ga[32];
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const uint4 gv = pg[i2][q4];
            const uint32_t w4[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[e]));
              ga[8 * q4 + 2 * e] = f2.x;
              ga[8 * q4 + 2 * e + 1] = f2.y;
            }
          }
          float dz[32];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float gi = ga[4 * k], gf = ga[4 * k + 1], gg = ga[4 * k + 2], go = ga[4 * k + 3];
            const float tc = tanhf(ct[k]);
            const float dc = dcc[k0 + k] + dh[k] * go * (1.f - tc * tc);
            dz[4 * k] = dc * gg * gi * (1.f - gi);
            dz[4 * k + 1] = dc * cp[k] * gf * (1.f - gf);
            dz[4 * k + 2] = dc * gi * (1.f - gg * gg);
            dz[4 * k + 3] = dh[k] * tc * go * (1.f - go);
            dcc[k0 + k] = dc * gf;
          }
          uint4* zd = reinterpret_cast<uint4*>(Ly.dg + ((size_t)r * T + t) * 4 * hd + 4 * u0);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              __nv_bfloat162 h2 = __floats2bfloat162_rn(dz[8 * q4 + 2 * e], dz[8 * q4 + 2 * e + 1]);
              w[e] = *reinterpret_cast<uint32_t*>(&h2);
            }
            zd[q4] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
      named_bar_sync(1, 256);
      if (threadIdx.x == 0) {
        LB_TRACE(t, 1);
        __threadfence();
        red_release_gpu_add(P.dgdone + (size_t)l * T + t, 1u);
      }
      prefetch(t - 1);
      // ---- G epilogue: this CTA's tiles of [dx_t | dh_{t-1}] (fp32, partial kh)
      for (int ct = gn; ct < ncol; ct += Gn, ++n) {
        const int acc = n & 1, use = n >> 1;
        mbar_wait(&tfull[acc], use & 1);
        tc_fence_after();
        if (threadIdx.x == 0) LB_TRACE(t, 5);
        for (int j = 0; j < Gk; ++j) {   // NT / 2 columns per warp, 32 at a time
          float v[32];
          tmem_ld32(tmem_base + ((q * 32u) << 16) + acc * NT + hh * (NT / 2) + 32 * j, v);
          const int col = ct * NT + (int)hh * (NT / 2) + 32 * j;
          if (row_ok) {
            float* dst = col < Ly.in
                             ? Ly.dx_out + kh * P.dx_kstride + ((size_t)r * T + t) * Ly.in + col
                             : Ly.dh_rec + kh * P.rec_kstride + ((size_t)(t & 1) * P.B + r) * hd + (col - Ly.in);
            float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
            for (int e = 0; e < 8; ++e) d4[e] = make_float4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
      named_bar_sync(1, 256);
      if (threadIdx.x == 0) {
        __threadfence();
        red_release_gpu_add(P.outdone + (size_t)l * T + t, 1u);
        LB_TRACE(t, 6);
      }
    }
    // initial-state gradients: dh_{-1} = the h part of step 0's product (all CTAs), dc carry
    if (Ly.dh0_out) {
      if (threadIdx.x == 0) {
        ls_wait_geq(P.outdone + (size_t)l * T, (unsigned)P.G);
        __threadfence();
      }
      named_bar_sync(1, 256);
      if (row_ok)
        for (int k = 0; k < nu; ++k) {
          float v = 0.f;
          for (int pk = 0; pk < Gk; ++pk) v += __ldcg(Ly.dh_rec + pk * P.rec_kstride + (size_t)r * hd + u_base + k);
          Ly.dh0_out[(size_t)r * hd + u_base + k] = v;
          Ly.dc0_out[(size_t)r * hd + u_base + k] = dcc[k];
        }
    }
    (void)rr;
  }
  tc_fence_before();
  if (C > 1) cluster_sync();   // no CTA leaves while a peer may still multicast into it
  else __syncthreads();
  tc_fence_after();
  if (warp == 8) tmem_dealloc(tmem_base, 2 * NT);
}

// dX0 rows scattered into the embedding gradient: dE[ids[b][t]] += dX0[b][t]
// (fp32 atomics: the summation order over repeated ids is not fixed)
// (dX holds nk K-split partials, kstride floats apart, added in order)
__global__ void embed_grad_kernel(const int* __restrict__ ids, const float* __restrict__ dX, int nk,
                                  long long kstride, int e, long long rows, float* __restrict__ dE) {
  const long long n = rows * e;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long row = i / e;
    float v = dX[i];
    for (int k = 1; k < nk; ++k) v += dX[k * kstride + i];
    atomicAdd(dE + (long long)ids[row] * e + (i % e), v);
  }
}
// Hprev[b][t] = t > 0 ? H[b][t-1] : h0[b] (zero when h0 is NULL), bf16, 16-byte vectors
__global__ void shift_h_kernel(const __nv_bfloat16* __restrict__ H, const __nv_bfloat16* __restrict__ h0,
                               int B, int T, int hd, __nv_bfloat16* __restrict__ Hp) {
  const int v8 = hd / 8;
  const long long n = (long long)B * T * v8;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long row = i / v8;
    const int k = (int)(i % v8);
    const int b = (int)(row / T), t = (int)(row % T);
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (t > 0) v = reinterpret_cast<const uint4*>(H)[(row - 1) * v8 + k];
    else if (h0) v = reinterpret_cast<const uint4*>(h0)[(long long)b * v8 + k];
    reinterpret_cast<uint4*>(Hp)[i] = v;
  }
}
// db[j] = sum over rows of dG[row][j], deterministic in two passes: block
// (x, y) sums rows [128 y, 128 y + 128) of columns [256 x, 256 x + 256) in
// order into part[y][j]; then part is summed over y in order.
constexpr int LB_CS_ROWS = 128;
__global__ void lstm_db_part_kernel(const __nv_bfloat16* __restrict__ dG, long long rows, int cols,
                                   float* __restrict__ part) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  const long long r0 = (long long)blockIdx.y * LB_CS_ROWS;
  const long long r1 = r0 + LB_CS_ROWS < rows ? r0 + LB_CS_ROWS : rows;
  float s = 0.f;
  for (long long r = r0; r < r1; ++r) s += __bfloat162float(dG[r * cols + j]);
  part[(long long)blockIdx.y * cols + j] = s;
}
__global__ void lstm_db_final_kernel(const float* __restrict__ part, int nparts, int cols, float* __restrict__ db) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  float s = 0.f;
  for (int y = 0; y < nparts; ++y) s += part[(long long)y * cols + j];
  db[j] = s;
}

// option "lstm_trace" (attn_softmax_set_option): stamps of the last backward launch
long long* g_lstm_trace = nullptr;

}  // namespace attnsm

// internal entry of attn_softmax.cu: C = A^T [B0 | B1] on the tcgen05 engine (dW of the backward)
attn_status_t attn_internal_gemm_atb(int M, int N, int K, const void* A, const void* B0, int n0,
                                     const void* B1, float* C, int* counter, cudaStream_t stream);
attn_status_t attn_internal_gemm_atb_group(int n, const int* M, const int* N, const int* K,
                                           const void* const* A, const void* const* B0,
                                           const int* n0, const void* const* B1, float* const* C,
                                           int* counter, cudaStream_t stream);
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
  void* gates_seq[LS_MAXL];       // training saves (or NULL)
  float* c_seq[LS_MAXL];
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
    Ly.gates_seq = static_cast<__nv_bfloat16*>(R.gates_seq[l]);
    Ly.c_seq = R.c_seq[l];
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
  attnsm::NvtxRange nvtx_range_("attn_encoder_decoder_fwd");
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
  attnsm::NvtxRange nvtx_range_("attn_encoder_decoder_if_fwd");
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

// ---------------------------------------------------------------- training (forward saves + backward)
namespace {
struct TrPlan {
  size_t inter_enc, inter_dec, gates_enc, gates_dec, cseq_enc, cseq_dec;   // forward saves
  size_t dg, dxo, dhrec, dh0, dc0, hprev, flags, counter, dbpart, total;
};
TrPlan plan_train(const attn_lstm_shape_t* s, const LsPlan& base) {
  TrPlan q;
  const size_t B = s->batch, M = s->src_len, N = s->tgt_len, hd = s->hidden, L = s->layers;
  const size_t Tm = std::max(M, N), w0 = std::max<size_t>(s->emb, hd);
  size_t o = base.total;
  auto take = [&](size_t b) { size_t r = o; o += al(b); return r; };
  q.inter_enc = take(std::max<size_t>(L - 1, 1) * B * M * hd * 2);
  q.inter_dec = take(std::max<size_t>(L - 1, 1) * B * N * hd * 2);
  q.gates_enc = take(L * B * M * 4 * hd * 2);
  q.gates_dec = take(L * B * N * 4 * hd * 2);
  q.cseq_enc = take(L * B * M * hd * 4);
  q.cseq_dec = take(L * B * N * hd * 4);
  q.dg = take(L * B * Tm * 4 * hd * 2);
  q.dxo = take(4 * L * B * Tm * w0 * 4);     // [Gk <= 4][L][B][Tm][w0]
  q.dhrec = take(4 * L * 2 * B * hd * 4);    // [Gk <= 4][L][2][B][hd]
  q.dh0 = take(L * B * hd * 4);
  q.dc0 = take(L * B * hd * 4);
  q.hprev = take(L * B * Tm * hd * 2);   // one [B][T][hd] h_prev per layer (grouped dW GEMM)
  q.flags = take(2 * L * Tm * 4);
  q.counter = take(256);
  q.dbpart = take(((B * Tm + 127) / 128) * 4 * hd * 4);
  q.total = o;
  return q;
}

// forward of one side with the training saves (separate intermediates per side)
attn_status_t run_side_train(const attn_lstm_shape_t* s, const LsPlan& p, const TrPlan& q, bool decoder,
                             const void* X0, const void* const* W, const float* const* b, void* H_top,
                             char* ws, const int* cap_dev, cudaStream_t st) {
  RunCfg R;
  memset(&R, 0, sizeof(R));
  const int B = s->batch, hd = s->hidden, L = s->layers, T = decoder ? s->tgt_len : s->src_len;
  R.B = B; R.T = T; R.hd = hd; R.L = L; R.G = p.G; R.ntile = p.ntile; R.in0 = s->emb;
  R.X0 = X0; R.W = W; R.b = b; R.cap_dev = decoder ? nullptr : cap_dev;
  R.done = reinterpret_cast<unsigned*>(ws + (decoder ? p.done_dec : p.done_enc));
  __nv_bfloat16* inter = reinterpret_cast<__nv_bfloat16*>(ws + (decoder ? q.inter_dec : q.inter_enc));
  __nv_bfloat16* gates = reinterpret_cast<__nv_bfloat16*>(ws + (decoder ? q.gates_dec : q.gates_enc));
  float* cseq = reinterpret_cast<float*>(ws + (decoder ? q.cseq_dec : q.cseq_enc));
  for (int l = 0; l < L; ++l) {
    R.hout[l] = l == L - 1 ? H_top : (void*)(inter + (size_t)l * B * T * hd);
    R.c[l] = reinterpret_cast<float*>(ws + p.c) + (size_t)l * B * hd;
    __nv_bfloat16* hcap = reinterpret_cast<__nv_bfloat16*>(ws + p.hcap) + (size_t)l * B * hd;
    float* ccap = reinterpret_cast<float*>(ws + p.ccap) + (size_t)l * B * hd;
    R.h0[l] = decoder ? hcap : nullptr;
    R.c0[l] = decoder ? ccap : nullptr;
    R.hcap[l] = decoder ? nullptr : hcap;
    R.ccap[l] = decoder ? nullptr : ccap;
    R.gates_seq[l] = gates + (size_t)l * B * T * 4 * hd;
    R.c_seq[l] = cseq + (size_t)l * B * T * hd;
  }
  return run_layers(R, st);
}

attn_status_t check_common(const attn_lstm_shape_t* s, const int32_t* src_lens_host, size_t need,
                           size_t have, const LsPlan& p) {
  for (int i = 0; i < s->batch; ++i)
    if (src_lens_host[i] < 1 || src_lens_host[i] > s->src_len)
      return lfail(ATTN_ERR_SHAPE, "src_lens_host[%d] = %d outside [1, M = %d]", i, src_lens_host[i], s->src_len);
  if (have < need) return lfail(ATTN_ERR_WORKSPACE, "workspace_bytes = %zu < required %zu", have, need);
  int dev = 0, sms = 0;
  LS_CUDA(cudaGetDevice(&dev));
  LS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (s->layers * p.G > sms)
    return lfail(ATTN_ERR_UNSUPPORTED, "lstm: %d layers x %d CTAs exceed the %d SMs", s->layers, p.G, sms);
  return ATTN_OK;
}

// K split of the backward wavefront's product: ATTN_LSTM_KSPLIT = 1, 2 or 4 (default 2)
static int lb_ksplit() {
  static const int k = [] {
    const char* e = getenv("ATTN_LSTM_KSPLIT");
    const int v = e ? atoi(e) : 2;
    return (v == 1 || v == 2 || v == 4) ? v : 2;
  }();
  return k;
}

// cluster size of the backward wavefront (dz multicast): ATTN_LSTM_CLUSTER = 1, 2 or 4 (default 2)
static int lb_cluster_size() {
  static const int c = [] {
    const char* e = getenv("ATTN_LSTM_CLUSTER");
    const int v = e ? atoi(e) : 2;
    return (v == 1 || v == 2 || v == 4) ? v : 2;
  }();
  return c;
}

// the reverse wavefront of one side
attn_status_t run_bwd_side(const attn_lstm_shape_t* s, const LsPlan& p, const TrPlan& q, bool decoder,
                           const void* const* W, const void* dH_top, char* ws, const int* cap_dev,
                           cudaStream_t st, int* gk_out) {
  static LbParams P;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  memset(&P, 0, sizeof(P));
  const int B = s->batch, hd = s->hidden, L = s->layers, T = decoder ? s->tgt_len : s->src_len;
  const size_t w0 = std::max(s->emb, hd);
  attn_status_t r;
  __nv_bfloat16* dg = reinterpret_cast<__nv_bfloat16*>(ws + q.dg);
  float* dxo = reinterpret_cast<float*>(ws + q.dxo);
  float* dhrec = reinterpret_cast<float*>(ws + q.dhrec);
  __nv_bfloat16* gates = reinterpret_cast<__nv_bfloat16*>(ws + (decoder ? q.gates_dec : q.gates_enc));
  float* cseq = reinterpret_cast<float*>(ws + (decoder ? q.cseq_dec : q.cseq_enc));
  float* ccap = reinterpret_cast<float*>(ws + p.ccap);
  float* dh0 = reinterpret_cast<float*>(ws + q.dh0);
  float* dc0 = reinterpret_cast<float*>(ws + q.dc0);
  for (int l = 0; l < L; ++l) {
    LbLayer& Ly = P.layer[l];
    Ly.in = l == 0 ? s->emb : hd;
    Ly.dg = dg + (size_t)l * B * T * 4 * hd;
    {
      cuuint64_t dims[3] = {(cuuint64_t)(4 * hd), (cuuint64_t)T, (cuuint64_t)B};
      cuuint64_t str[2] = {(cuuint64_t)(4 * hd) * 2, (cuuint64_t)(4 * hd) * 2 * T};
      cuuint32_t box[3] = {64, 1, 128};
      if ((r = map_bf16(&Ly.m_dg, Ly.dg, 3, dims, str, box)) != ATTN_OK) return r;
    }
    if ((r = map_mat(&Ly.m_w, W[l], Ly.in + hd, 4 * hd, 64)) != ATTN_OK) return r;
    Ly.gates = gates + (size_t)l * B * T * 4 * hd;
    Ly.c_seq = cseq + (size_t)l * B * T * hd;
    Ly.c0 = decoder ? ccap + (size_t)l * B * hd : nullptr;
    Ly.dh_top = l == L - 1 ? static_cast<const __nv_bfloat16*>(dH_top) : nullptr;
    Ly.dx_above = l == L - 1 ? nullptr : dxo + (size_t)(l + 1) * B * T * w0;
    Ly.dx_out = dxo + (size_t)l * B * T * w0;
    Ly.dh_rec = dhrec + (size_t)l * 2 * B * hd;
    Ly.dh0_out = decoder ? dh0 + (size_t)l * B * hd : nullptr;
    Ly.dc0_out = decoder ? dc0 + (size_t)l * B * hd : nullptr;
    Ly.inj_dh = decoder ? nullptr : dh0 + (size_t)l * B * hd;
    Ly.inj_dc = decoder ? nullptr : dc0 + (size_t)l * B * hd;
  }
  P.L = L; P.B = B; P.T = T; P.hd = hd; P.G = p.G;
  // K split: the largest Gk <= the option with G % Gk == 0 and every layer's output
  // width a multiple of the 64 Gk-column tile
  P.Gk = 1;
  for (int k = lb_ksplit(); k > 1; k /= 2)
    if (p.G % k == 0 && (s->emb + hd) % (64 * k) == 0 && (2 * hd) % (64 * k) == 0 && (hd / 16) % k == 0) {
      P.Gk = k;
      break;
    }
  P.dx_kstride = (long long)L * B * std::max(s->src_len, s->tgt_len) * (long long)w0;
  P.rec_kstride = (long long)L * 2 * B * hd;
  *gk_out = P.Gk;
  P.cap = decoder ? nullptr : cap_dev;
  unsigned* flags = reinterpret_cast<unsigned*>(ws + q.flags);
  P.dgdone = flags;
  P.outdone = flags + (size_t)L * T;
  P.trace = g_lstm_trace;
  LS_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned) * 2 * (size_t)L * T, st));
  static std::vector<int> attr_set;
  int dev = 0;
  LS_CUDA(cudaGetDevice(&dev));
  if (std::find(attr_set.begin(), attr_set.end(), dev) == attr_set.end()) {
    LS_CUDA(cudaFuncSetAttribute(lstm_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, LB_SMEM));
    attr_set.push_back(dev);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(L * p.G);
  cfg.blockDim = dim3(LS_THREADS);
  cfg.dynamicSmemBytes = LB_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // clusters of C CTAs of one layer share each dz k-block (TMA multicast): C
  // divides G, every CTA of a cluster owns the same number of 64-column slices,
  // and all L G / C clusters are co-resident (the flags are spin-waited on)
  int C = lb_cluster_size();
  const int Gn = p.G / P.Gk;
  for (; C > 1; C /= 2) {
    bool ok = Gn % C == 0;
    for (int l = 0; ok && l < L; ++l) {
      const int ncol = ((l == 0 ? s->emb : hd) + hd) / (64 * P.Gk);
      auto cnt = [&](int gn) { return gn < ncol ? (ncol - 1 - gn) / Gn + 1 : 0; };
      for (int gn = 0; ok && gn < Gn; ++gn) ok = cnt(gn) == cnt(gn - gn % C);
    }
    if (!ok) continue;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = C;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.numAttrs = 2;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, lstm_bwd_kernel, &cfg) == cudaSuccess &&
        nclusters >= L * p.G / C)
      break;
    (void)cudaGetLastError();
    cfg.numAttrs = 1;
  }
  P.C = C > 1 ? C : 1;
  cfg.numAttrs = P.C > 1 ? 2 : 1;
  LS_CUDA(cudaLaunchKernelEx(&cfg, lstm_bwd_kernel, P));
  return ATTN_OK;
}

// dW_l = dz^T [x | h_prev], db_l = column sums of dz, for every layer of one side
attn_status_t side_weight_grads(const attn_lstm_shape_t* s, const LsPlan& p, const TrPlan& q, bool decoder,
                                const void* X0, const void* H_top, float* const* dW, float* const* db,
                                char* ws, int sms, cudaStream_t st) {
  const int B = s->batch, hd = s->hidden, L = s->layers, T = decoder ? s->tgt_len : s->src_len;
  const long long rows = (long long)B * T;
  __nv_bfloat16* dg = reinterpret_cast<__nv_bfloat16*>(ws + q.dg);
  __nv_bfloat16* inter = reinterpret_cast<__nv_bfloat16*>(ws + (decoder ? q.inter_dec : q.inter_enc));
  __nv_bfloat16* hprev = reinterpret_cast<__nv_bfloat16*>(ws + q.hprev);
  const __nv_bfloat16* hcap = reinterpret_cast<const __nv_bfloat16*>(ws + p.hcap);
  int* counter = reinterpret_cast<int*>(ws + q.counter);
  attn_status_t r;
  // h_prev of every layer, then the layers' dW = dz^T [x | h_prev] products in
  // grouped launches of up to 4 (one tile list: 4 x 256 tiles at Table 1 sizes
  // instead of 256 per launch, 1.73 waves on 148 SMs)
  for (int l = 0; l < L; ++l) {
    const void* Hl = l == L - 1 ? H_top : (const void*)(inter + (size_t)l * B * T * hd);
    shift_h_kernel<<<sms * 4, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(Hl),
                                            decoder ? hcap + (size_t)l * B * hd : nullptr, B, T, hd,
                                            hprev + (size_t)l * B * T * hd);
    LS_CUDA(cudaGetLastError());
  }
  for (int l0 = 0; l0 < L; l0 += 4) {
    const int n = std::min(4, L - l0);
    int Mv[4], Nv[4], Kv[4], n0v[4];
    const void* Av[4]; const void* B0v[4]; const void* B1v[4]; float* Cv[4];
    for (int i = 0; i < n; ++i) {
      const int l = l0 + i;
      const int in = l == 0 ? s->emb : hd;
      Mv[i] = 4 * hd; Nv[i] = in + hd; Kv[i] = (int)rows; n0v[i] = in;
      Av[i] = dg + (size_t)l * B * T * 4 * hd;
      B0v[i] = l == 0 ? X0 : (const void*)(inter + (size_t)(l - 1) * B * T * hd);
      B1v[i] = hprev + (size_t)l * B * T * hd;
      Cv[i] = dW[l];
    }
    LS_CUDA(cudaMemsetAsync(counter, 0, sizeof(int), st));
    if ((r = attn_internal_gemm_atb_group(n, Mv, Nv, Kv, Av, B0v, n0v, B1v, Cv, counter, st)) != ATTN_OK)
      return r;
  }
  for (int l = 0; l < L; ++l) {
    const __nv_bfloat16* dgl = dg + (size_t)l * B * T * 4 * hd;
    float* part = reinterpret_cast<float*>(ws + q.dbpart);
    const int nparts = (int)((rows + LB_CS_ROWS - 1) / LB_CS_ROWS);
    lstm_db_part_kernel<<<dim3((4 * hd + 255) / 256, nparts), 256, 0, st>>>(dgl, rows, 4 * hd, part);
    LS_CUDA(cudaGetLastError());
    lstm_db_final_kernel<<<(4 * hd + 255) / 256, 256, 0, st>>>(part, nparts, 4 * hd, db[l]);
    LS_CUDA(cudaGetLastError());
  }
  return ATTN_OK;
}
}  // namespace

extern "C" size_t attn_lstm_train_workspace_size(const attn_lstm_shape_t* s) {
  if (check_lstm(s) != ATTN_OK) return 0;
  const LsPlan p = plan_lstm(s);
  return plan_train(s, p).total;
}

extern "C" attn_status_t attn_encoder_decoder_fwd_train(
    const attn_lstm_shape_t* s, const int32_t* src_ids, const int32_t* tgt_ids,
    const int32_t* src_lens_host, const void* E_src, const void* E_tgt,
    const void* const* enc_W, const float* const* enc_b, const void* const* dec_W,
    const float* const* dec_b, void* H_enc, void* H_dec, void* workspace, size_t workspace_bytes,
    void* stream) {
  attnsm::NvtxRange nvtx_range_("attn_encoder_decoder_fwd_train");
  attn_status_t r = check_lstm(s);
  if (r != ATTN_OK) return r;
  if (!src_ids || !tgt_ids || !src_lens_host || !E_src || !E_tgt || !enc_W || !enc_b || !dec_W ||
      !dec_b || !H_enc || !H_dec || !workspace)
    return lfail(ATTN_ERR_INVALID_ARG, "encoder_decoder_fwd_train: NULL argument");
  const LsPlan p = plan_lstm(s);
  const TrPlan q = plan_train(s, p);
  if ((r = check_common(s, src_lens_host, q.total, workspace_bytes, p)) != ATTN_OK) return r;
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = static_cast<char*>(workspace);
  const int B = s->batch, M = s->src_len, N = s->tgt_len, e = s->emb;
  int sms = 0, dev = 0;
  LS_CUDA(cudaGetDevice(&dev));
  LS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  std::vector<int> cap(B);
  for (int i = 0; i < B; ++i) cap[i] = src_lens_host[i] - 1;
  int* cap_dev = reinterpret_cast<int*>(ws + p.lens);
  LS_CUDA(cudaMemcpyAsync(cap_dev, cap.data(), sizeof(int) * B, cudaMemcpyHostToDevice, st));
  __nv_bfloat16* Xs = reinterpret_cast<__nv_bfloat16*>(ws + p.xs);
  __nv_bfloat16* Xt = reinterpret_cast<__nv_bfloat16*>(ws + p.xt);
  embed_kernel<<<sms * 4, 256, 0, st>>>(src_ids, static_cast<const __nv_bfloat16*>(E_src), e, (long long)B * M, Xs);
  LS_CUDA(cudaGetLastError());
  embed_kernel<<<sms * 4, 256, 0, st>>>(tgt_ids, static_cast<const __nv_bfloat16*>(E_tgt), e, (long long)B * N, Xt);
  LS_CUDA(cudaGetLastError());
  if ((r = run_side_train(s, p, q, false, Xs, enc_W, enc_b, H_enc, ws, cap_dev, st)) != ATTN_OK) return r;
  return run_side_train(s, p, q, true, Xt, dec_W, dec_b, H_dec, ws, cap_dev, st);
}

extern "C" attn_status_t attn_encoder_decoder_bwd(
    const attn_lstm_shape_t* s, const int32_t* src_ids, const int32_t* tgt_ids,
    const int32_t* src_lens_host, const void* const* enc_W, const void* const* dec_W,
    const void* H_enc, const void* H_dec, const void* dH_enc, const void* dH_dec,
    float* const* dW_enc, float* const* db_enc, float* const* dW_dec, float* const* db_dec,
    float* dE_src, float* dE_tgt, void* workspace, size_t workspace_bytes, void* stream) {
  attnsm::NvtxRange nvtx_range_("attn_encoder_decoder_bwd");
  attn_status_t r = check_lstm(s);
  if (r != ATTN_OK) return r;
  if (!src_ids || !tgt_ids || !src_lens_host || !enc_W || !dec_W || !H_enc || !H_dec || !dH_enc ||
      !dH_dec || !dW_enc || !db_enc || !dW_dec || !db_dec || !dE_src || !dE_tgt || !workspace)
    return lfail(ATTN_ERR_INVALID_ARG, "encoder_decoder_bwd: NULL argument");
  for (int l = 0; l < s->layers; ++l)
    if (!enc_W[l] || !dec_W[l] || !dW_enc[l] || !db_enc[l] || !dW_dec[l] || !db_dec[l])
      return lfail(ATTN_ERR_INVALID_ARG, "encoder_decoder_bwd: layer %d buffer is NULL", l);
  const LsPlan p = plan_lstm(s);
  const TrPlan q = plan_train(s, p);
  if ((r = check_common(s, src_lens_host, q.total, workspace_bytes, p)) != ATTN_OK) return r;
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = static_cast<char*>(workspace);
  const int B = s->batch, M = s->src_len, N = s->tgt_len, e = s->emb;
  int sms = 0, dev = 0;
  LS_CUDA(cudaGetDevice(&dev));
  LS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  std::vector<int> cap(B);
  for (int i = 0; i < B; ++i) cap[i] = src_lens_host[i] - 1;
  int* cap_dev = reinterpret_cast<int*>(ws + p.lens);
  LS_CUDA(cudaMemcpyAsync(cap_dev, cap.data(), sizeof(int) * B, cudaMemcpyHostToDevice, st));
  float* dxo = reinterpret_cast<float*>(ws + q.dxo);
  LS_CUDA(cudaMemsetAsync(dE_src, 0, sizeof(float) * (size_t)s->vocab_src * e, st));
  LS_CUDA(cudaMemsetAsync(dE_tgt, 0, sizeof(float) * (size_t)s->vocab_tgt * e, st));
  // decoder first: its initial-state gradients reach the encoder at src_len - 1
  int gk = 1;
  if ((r = run_bwd_side(s, p, q, true, dec_W, dH_dec, ws, cap_dev, st, &gk)) != ATTN_OK) return r;
  if ((r = side_weight_grads(s, p, q, true, ws + p.xt, H_dec, dW_dec, db_dec, ws, sms, st)) != ATTN_OK) return r;
  // layer 0's dx_out is dL/dx [B][N][e]: the target embeddings' rows
  const long long dx_kstride = (long long)s->layers * B * std::max(M, N) * (long long)std::max(e, s->hidden);
  embed_grad_kernel<<<sms * 8, 256, 0, st>>>(tgt_ids, dxo, gk, dx_kstride, e, (long long)B * N, dE_tgt);
  LS_CUDA(cudaGetLastError());
  if ((r = run_bwd_side(s, p, q, false, enc_W, dH_enc, ws, cap_dev, st, &gk)) != ATTN_OK) return r;
  if ((r = side_weight_grads(s, p, q, false, ws + p.xs, H_enc, dW_enc, db_enc, ws, sms, st)) != ATTN_OK) return r;
  embed_grad_kernel<<<sms * 8, 256, 0, st>>>(src_ids, dxo, gk, dx_kstride, e, (long long)B * M, dE_src);
  LS_CUDA(cudaGetLastError());
  return ATTN_OK;
}
