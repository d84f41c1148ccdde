// small_kernels.cuh -- memory-bound kernels of the stage (both dtype paths).
//
//   softmax_fwd_kernel   Eq. 1: masked row softmax of the
//                        attention scores over j < src_len[b]; masked
//                        positions become exactly 0 (reading R8).  One warp
//                        per decoder row, warp-shuffle max / sum.
//   softmax_bwd_kernel   backward of Eq. 1: de_ij = a_ij (da_ij - sum_k a_ik da_ik)
//   lse_reduce_kernel    Eqs. 5-6: combine the per-tile (max, sumexp)
//                        partials of the vocab GEMM epilogue into lse_t, the
//                        token NLL lse_t - l_{t,y_t} on valid rows, the row
//                        scale of the backward, and the deterministic loss sum.
//   check_ids_kernel     target-id range check (ATTN_ERR_TOKEN_RANGE)
//   decode_final_kernel  decoding step (NEXT-4): lse and the k best tokens of
//                        each row from the vocab GEMM's per-tile partials
//   dlogits_from_logits_kernel  B1 with the forward's stored fp16 logits
//   colsum_*_kernel      db_out of the F_c bias (NEXT-1): column sums of one
//                        dlogits V-chunk, two passes in a fixed order (fp32
//                        path and paired tiles; else a ones GEMM)
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

#include "epilogue.cuh"
#include "ptx.cuh"

namespace attnsm {

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// buf [B*N, M] fp32: scores in, alpha out (in place).
__global__ void __launch_bounds__(256) softmax_fwd_kernel(float* __restrict__ buf,
                                                          const int* __restrict__ src_len,
                                                          int rows, int N, int M) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int L = src_len[row / N];
  float* e = buf + (long long)row * M;
  float mx = -INFINITY;
  for (int j = lane; j < L; j += 32) mx = fmaxf(mx, e[j]);
  mx = warp_max(mx);
  float s = 0.f;
  for (int j = lane; j < L; j += 32) s += expf(e[j] - mx);
  s = warp_sum(s);
  const float inv = 1.f / s;
  for (int j = lane; j < M; j += 32) e[j] = (j < L) ? expf(e[j] - mx) * inv : 0.f;
}

// alpha [B*N, M], da [B*N, M] (dalpha in, de out in place).
__global__ void __launch_bounds__(256) softmax_bwd_kernel(const float* __restrict__ alpha,
                                                          float* __restrict__ da, int rows,
                                                          int M) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* a = alpha + (long long)row * M;
  float* g = da + (long long)row * M;
  float D = 0.f;
  for (int j = lane; j < M; j += 32) D += a[j] * g[j];
  D = warp_sum(D);
  for (int j = lane; j < M; j += 32) g[j] = a[j] * (g[j] - D);
}

// One warp per row t = b*N + i.  part [T, part_ld] (max, sumexp).
// Block partial sums (double) go to blockpart[]; the last block to finish
// sums them in index order (deterministic) and writes *loss.
__global__ void __launch_bounds__(256) lse_reduce_kernel(
    const float2* __restrict__ part, int part_ld, const float* __restrict__ tgt_logit,
    const int* __restrict__ tgt_len, int T, int N, float loss_scale, float* __restrict__ lse_out,
    float* __restrict__ nll_out, float* __restrict__ rowscale, double* __restrict__ blockpart,
    unsigned int* __restrict__ done_counter, float* __restrict__ loss) {
  pdl_wait();   // launched as a programmatic dependent of the vocab GEMM
  __shared__ double wsum[8];
  __shared__ bool is_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;
  double contrib = 0.0;
  if (row < T) {
    const float2* pr = part + (long long)row * part_ld;
    float mx = -INFINITY;
    for (int j = lane; j < part_ld; j += 32) mx = fmaxf(mx, pr[j].x);
    mx = warp_max(mx);
    float s = 0.f;
    for (int j = lane; j < part_ld; j += 32) {
      const float2 q = pr[j];
      s += q.y * expf(q.x - mx);
    }
    s = warp_sum(s);
    const float lse = mx + logf(s);
    const bool valid = (row % N) < tgt_len[row / N];
    const float nll = valid ? lse - tgt_logit[row] : 0.f;
    if (lane == 0) {
      lse_out[row] = lse;
      nll_out[row] = nll;
      rowscale[row] = valid ? loss_scale : 0.f;
    }
    contrib = (double)nll;
  }
  if (lane == 0) wsum[warp] = contrib;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < 8; ++w) b += wsum[w];
    blockpart[blockIdx.x] = b;
    __threadfence();
    const unsigned int prev = atomicAdd(done_counter, 1u);
    is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last) {
    __threadfence();
    if (threadIdx.x < 32) {
      double acc = 0.0;
      // fixed assignment of blocks to lanes, fixed shuffle tree: deterministic
      for (int i = threadIdx.x; i < (int)gridDim.x; i += 32)
        acc += ((volatile double*)blockpart)[i];
      acc = warp_sum_d(acc);
      if (threadIdx.x == 0) {
        *loss = (float)(acc * (double)loss_scale);
        *done_counter = 0u;
      }
    }
  }
}

// Backward of Eq. 4's tanh: dz = dHc * (1 - H_c^2), written in the
// activation dtype (the operand of the W_c backward GEMMs).
template <typename T>
__global__ void __launch_bounds__(256) dz_kernel(const float* __restrict__ dhc,
                                                 const T* __restrict__ hc, T* __restrict__ dz,
                                                 long long n, float4* __restrict__ zero, long long nzero4) {
  pdl_wait();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // side job: zero `nzero4` float4 of `zero` (dW_c, summed by split-K reduce-adds)
  for (long long k = i; k < nzero4; k += stride) zero[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  if constexpr (sizeof(T) == 2) {
    // 8 elements per thread and iteration: 2 x 16 B of dHc, 16 B of H_c, 16 B of dz
    const long long n8 = n / 8;
    for (long long k = i; k < n8; k += stride) {
      const float4 a = reinterpret_cast<const float4*>(dhc)[2 * k];
      const float4 b = reinterpret_cast<const float4*>(dhc)[2 * k + 1];
      const uint4 hu = reinterpret_cast<const uint4*>(hc)[k];
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&hu);
      const float g[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 h = __bfloat1622float2(h2[e]);
        __nv_bfloat162 o = __floats2bfloat162_rn(g[2 * e] * (1.f - h.x * h.x),
                                                 g[2 * e + 1] * (1.f - h.y * h.y));
        w[e] = *reinterpret_cast<uint32_t*>(&o);
      }
      reinterpret_cast<uint4*>(dz)[k] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    for (long long k = 8 * n8 + i; k < n; k += stride) {
      const float h = to_f32(hc[k]);
      dz[k] = to_out<T>(dhc[k] * (1.f - h * h));
    }
  } else {
    for (long long k = i; k < n; k += stride) {
      const float h = to_f32(hc[k]);
      dz[k] = to_out<T>(dhc[k] * (1.f - h * h));
    }
  }
}

// db[c] = sum_t dl[t, c] for c < ncols (dl row stride ld, 16-byte aligned
// rows), in two deterministic passes.  Pass 1: block (x, y) owns columns
// [256 x, 256 x + 256) and the row split y; thread t of warp w loads 8
// consecutive columns (16 bytes of bf16 / 2 x 16 of fp32) of rows
// y*rps + w, +8, ...; the 8 warp partials are added in a fixed order into
// part[y][c].  Pass 2 adds the splits in order.
template <typename T>
__global__ void __launch_bounds__(256) colsum_part_kernel(const T* __restrict__ dl, long long ld,
                                                          int rows, int rps, int ncols,
                                                          float* __restrict__ part) {
  __shared__ float red[8][257];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c0 = blockIdx.x * 256 + lane * 8;
  const int r0 = blockIdx.y * rps, r1 = min(rows, r0 + rps);
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  if (c0 + 8 <= ncols) {
    for (int r = r0 + w; r < r1; r += 8) {
      const T* row = dl + (long long)r * ld + c0;
      if constexpr (sizeof(T) == 2) {
        const uint4 u = *reinterpret_cast<const uint4*>(row);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h[e]);
          acc[2 * e] += f.x;
          acc[2 * e + 1] += f.y;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += to_f32(row[e]);
      }
    }
  } else {
    for (int r = r0 + w; r < r1; r += 8)
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (c0 + e < ncols) acc[e] += to_f32(dl[(long long)r * ld + c0 + e]);
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) red[w][lane * 8 + e] = acc[e];
  __syncthreads();
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c < ncols) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][threadIdx.x];
    part[(long long)blockIdx.y * ncols + c] = t;
  }
}
__global__ void __launch_bounds__(256) colsum_final_kernel(const float* __restrict__ part, int splits,
                                                           int ncols, float* __restrict__ db) {
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c >= ncols) return;
  float t = 0.f;
  for (int y = 0; y < splits; ++y) t += part[(long long)y * ncols + c];
  db[c] = t;
}

// One block of 4 warps per row: lse from the (max, sumexp) partials (as
// lse_reduce) and the k <= 8 best (logit, token) pairs merged from the
// per-slot sorted top-8 lists: thread i takes slots i, i + 128, ..., merges
// their lists with branch-free bitonic top-8 merges of 64-bit keys
// (epilogue.cuh tk_*), then a butterfly across each warp's lanes and warp 0
// merges the four warps' lists.  The key order is total, so the result is
// unique; the lse sums run in a fixed order (per thread, then the lanes, then
// the warps).
constexpr int DF_THREADS = 128;
__global__ void __launch_bounds__(DF_THREADS) decode_final_kernel(const float2* __restrict__ part,
                                                                  const uint32_t* __restrict__ topk,
                                                                  int part_ld, int T, int k,
                                                                  int* __restrict__ ids,
                                                                  float* __restrict__ logp,
                                                                  float* __restrict__ lse_out) {
  pdl_wait();
  __shared__ float red[DF_THREADS / 32];
  __shared__ unsigned long long lists[DF_THREADS / 32][8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int row = blockIdx.x;
  if (row >= T) return;
  const float2* pr = part + (long long)row * part_ld;
  float mx = -INFINITY;
  for (int j = tid; j < part_ld; j += DF_THREADS) mx = fmaxf(mx, pr[j].x);
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  __syncthreads();
  float s = 0.f;
  for (int j = tid; j < part_ld; j += DF_THREADS) {
    const float2 q = pr[j];
    if (q.y > 0.f) s += q.y * __expf(q.x - mx);
  }
  s = warp_sum(s);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  const float lse = mx + logf(((red[0] + red[1]) + red[2]) + red[3]);
  // slot j covers columns [128 j, 128 j + 128): its 32-bit keys become
  // 64-bit (value, token) keys, merged across slots, lanes and warps
  unsigned long long best[8], b2[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) best[i] = 0ull;
  const uint4* tk = reinterpret_cast<const uint4*>(topk + (long long)row * part_ld * 8);
  for (int j = tid; j < part_ld; j += DF_THREADS) {
    const uint4 a = tk[(long long)j * 2], c = tk[(long long)j * 2 + 1];
    const uint32_t kk[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
#pragma unroll
    for (int i = 0; i < 8; ++i)
      b2[i] = kk[i] ? tk_key(tk32_val(kk[i]), 128 * j + tk32_local(kk[i])) : 0ull;
    tk_merge8(best, b2);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int i = 0; i < 8; ++i) b2[i] = __shfl_xor_sync(0xffffffffu, best[i], o);
    tk_merge8(best, b2);
  }
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < 8; ++i) lists[warp][i] = best[i];
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < DF_THREADS / 32; ++w) {
#pragma unroll
      for (int i = 0; i < 8; ++i) b2[i] = lists[w][i];
      tk_merge8(best, b2);
    }
    for (int i = 0; i < k; ++i) {
      ids[(long long)row * k + i] = tk_id(best[i]);
      logp[(long long)row * k + i] = tk_val(best[i]) - lse;
    }
    if (lse_out) lse_out[row] = lse;
  }
}

// Host length arrays reach the device as kernel parameters (by value): no
// host staging buffer, so the call is CUDA-graph capturable and a captured
// graph replays with the lengths it was captured with.
struct LensChunk {
  int* dst;
  int n;
  int vals[512];
};
__global__ void __launch_bounds__(512) lens_kernel(const __grid_constant__ LensChunk c) {
  if ((int)threadIdx.x < c.n) c.dst[threadIdx.x] = c.vals[threadIdx.x];
}

// B1 with stored logits (option store_logits): dlogits_c[t, v] = rs_t
// (exp(l_tv - lse_t) - [v = y_t]) for the V-chunk [c0, c0 + vcc) from the
// forward's fp16 logits, bf16 out (row stride dld); the target column uses
// the fp32 target logit (as the GEMM epilogue does); 0 on padded rows.
// Blocks stride over rows; a thread handles 8 columns (16-byte loads and
// stores), four loads in flight.  256 threads of <= 64 registers: one block
// fits beside a resident persistent GEMM CTA (registers, and the 1 KB of
// shared memory the SM reserves per block); the overlapped chunks launch
// exactly one block per SM.  (Same-box C1: 6 or 8 loads in flight, or 384
// threads, were 1-2% slower -- more concurrent traffic slows the GEMM.)  wait_first = 0 (chunks
// c >= 1, launched as programmatic dependents of launch c-1): the blocks
// start while launch c-1 still runs and do their work beside it -- every
// input is older than launch c-1 and the dlogits buffer they write was last
// read by launch c-2, complete before launch c-1 passed its own wait -- and
// only wait for launch c-1 at the end, so that launch c still starts after
// launch c-1 has finished (dHc accumulation order).
__device__ __forceinline__ uint32_t bf16x2_bits(float a, float b) {
  __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h2);
}
#ifndef ATTN_EW_THREADS
#define ATTN_EW_THREADS 256
#endif
#ifndef ATTN_EW_LOADS
#define ATTN_EW_LOADS 4
#endif
constexpr int kEwThreads = ATTN_EW_THREADS;   // see the block-size note above
constexpr int kEwLoads = ATTN_EW_LOADS;       // 16-byte loads in flight per thread
// (min 4 blocks: caps registers at 16384 / threads, what the persistent CTA leaves)
__global__ void __launch_bounds__(kEwThreads, 4) dlogits_from_logits_kernel(
    const __half* __restrict__ lg, long long lld, int c0, int vcc, int T,
    const float* __restrict__ lse, const float* __restrict__ rowscale, const int* __restrict__ tgt,
    const float* __restrict__ tgt_logit, __nv_bfloat16* __restrict__ dl, long long dld,
    int wait_first) {
  if (wait_first) pdl_wait();
  const int cols8 = (vcc + 7) / 8;
  for (int row = blockIdx.x; row < T; row += gridDim.x) {
    const float rs = rowscale[row];
    float c2 = 0.f, fix = 0.f;
    int y = -1;
    if (rs > 0.f) {
      const float ls = lse[row];
      c2 = __log2f(rs) - ls * kLog2e;
      y = tgt[row] - c0;
      fix = rs * (__expf(tgt_logit[row] - ls) - 1.f);
    }
    const __half* l = lg + (long long)row * lld + c0;
    __nv_bfloat16* o = dl + (long long)row * dld;
    for (int j0 = threadIdx.x; j0 < cols8; j0 += kEwLoads * kEwThreads) {
      uint4 u[kEwLoads];
#pragma unroll
      for (int k = 0; k < kEwLoads; ++k) {
        const int col = (j0 + k * kEwThreads) * 8;
        u[k] = (rs > 0.f && col + 8 <= vcc) ? __ldcs(reinterpret_cast<const uint4*>(l + col))
                                            : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int k = 0; k < kEwLoads; ++k) {
        const int col = (j0 + k * kEwThreads) * 8;
        if (col >= vcc) break;
        float g[8];
        if (rs > 0.f) {
          if (col + 8 <= vcc) {
            const uint32_t w[4] = {u[k].x, u[k].y, u[k].z, u[k].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[e]));
              g[2 * e] = ex2_mufu(fmaf(f.x, kLog2e, c2));
              g[2 * e + 1] = ex2_mufu(fmaf(f.y, kLog2e, c2));
            }
          } else {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              g[e] = col + e < vcc ? ex2_mufu(fmaf(__half2float(l[col + e]), kLog2e, c2)) : 0.f;
          }
          const int yl = y - col;
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (e == yl) g[e] = fix;
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) g[e] = 0.f;
        }
        if (col + 8 <= vcc) {
          *reinterpret_cast<uint4*>(o + col) =
              make_uint4(bf16x2_bits(g[0], g[1]), bf16x2_bits(g[2], g[3]),
                         bf16x2_bits(g[4], g[5]), bf16x2_bits(g[6], g[7]));
        } else {
          for (int e = 0; e < 8 && col + e < vcc; ++e) o[col + e] = __float2bfloat16_rn(g[e]);
        }
      }
    }
  }
  if (!wait_first) pdl_wait();
}

// The same dlogits plus the F_c bias's column sums (db_out): a 2D grid,
// blockIdx.y = a slab of kEwThreads x 8 columns (one 8-column group per
// thread), blockIdx.x = a row group (rows blockIdx.x, + gridDim.x, ...,
// three in flight).  Each thread sums its 8 columns' fp32 dlogits down its
// rows in a fixed order into dbpart[blockIdx.x][c0 + col] (row stride pld);
// ew_colsum_final_kernel adds the row groups in order -- deterministic, and
// no column-sum launch breaks the overlapped chain.
__global__ void __launch_bounds__(kEwThreads, 4) dlogits_colsum_kernel(
    const __half* __restrict__ lg, long long lld, int c0, int vcc, int T,
    const float* __restrict__ lse, const float* __restrict__ rowscale, const int* __restrict__ tgt,
    const float* __restrict__ tgt_logit, __nv_bfloat16* __restrict__ dl, long long dld,
    float* __restrict__ dbpart, long long pld, int wait_first) {
  if (wait_first) pdl_wait();
  constexpr int kR = 3;
  const int j = blockIdx.y * kEwThreads + threadIdx.x;
  const int col = j * 8;
  if (col < vcc) {
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    for (int row0 = blockIdx.x; row0 < T; row0 += kR * gridDim.x) {
      uint4 u[kR];
      float rs[kR], c2[kR];
#pragma unroll
      for (int k = 0; k < kR; ++k) {
        const int row = row0 + k * (int)gridDim.x;
        rs[k] = row < T ? rowscale[row] : 0.f;
        c2[k] = rs[k] > 0.f ? __log2f(rs[k]) - lse[row] * kLog2e : 0.f;
        u[k] = (rs[k] > 0.f && col + 8 <= vcc)
                   ? __ldcs(reinterpret_cast<const uint4*>(lg + (long long)row * lld + c0 + col))
                   : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int k = 0; k < kR; ++k) {
        const int row = row0 + k * (int)gridDim.x;
        if (row >= T) break;
        float g[8];
        if (rs[k] > 0.f) {
          if (col + 8 <= vcc) {
            const uint32_t w[4] = {u[k].x, u[k].y, u[k].z, u[k].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[e]));
              g[2 * e] = ex2_mufu(fmaf(f.x, kLog2e, c2[k]));
              g[2 * e + 1] = ex2_mufu(fmaf(f.y, kLog2e, c2[k]));
            }
          } else {
            const __half* l = lg + (long long)row * lld + c0;
#pragma unroll
            for (int e = 0; e < 8; ++e)
              g[e] = col + e < vcc ? ex2_mufu(fmaf(__half2float(l[col + e]), kLog2e, c2[k])) : 0.f;
          }
          const int yl = tgt[row] - c0 - col;
          if ((unsigned)yl < 8u) {
            const float fix = rs[k] * (__expf(tgt_logit[row] - lse[row]) - 1.f);
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (e == yl) g[e] = fix;
          }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) g[e] = 0.f;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += g[e];
        __nv_bfloat16* o = dl + (long long)row * dld;
        if (col + 8 <= vcc) {
          *reinterpret_cast<uint4*>(o + col) =
              make_uint4(bf16x2_bits(g[0], g[1]), bf16x2_bits(g[2], g[3]),
                         bf16x2_bits(g[4], g[5]), bf16x2_bits(g[6], g[7]));
        } else {
          for (int e = 0; e < 8 && col + e < vcc; ++e) o[col + e] = __float2bfloat16_rn(g[e]);
        }
      }
    }
    float* pp = dbpart + (long long)blockIdx.x * pld + c0 + col;
    for (int e = 0; e < 8 && col + e < vcc; ++e) pp[e] = acc[e];
  }
  if (!wait_first) pdl_wait();
}

// db_out from the dlogits kernels' row-group partials part[y][c] (row stride
// ncols): columns < first_cols have n_first partial rows, the rest n_rest;
// added in row order
__global__ void __launch_bounds__(256) ew_colsum_final_kernel(const float* __restrict__ part,
                                                              int n_first, int first_cols,
                                                              int n_rest, int ncols,
                                                              float* __restrict__ db) {
  pdl_wait();
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c >= ncols) return;
  const int n = c < first_cols ? n_first : n_rest;
  float t = 0.f;
  for (int y = 0; y < n; ++y) t += part[(long long)y * ncols + c];
  db[c] = t;
}


__global__ void check_ids_kernel(const int* __restrict__ ids, const int* __restrict__ tgt_len,
                                 int T, int N, int V, int* __restrict__ bad) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  if ((t % N) < tgt_len[t / N]) {
    const int y = ids[t];
    if (y < 0 || y >= V) atomicExch(bad, 1);
  }
}

}  // namespace attnsm
