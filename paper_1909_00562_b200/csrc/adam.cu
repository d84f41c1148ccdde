// adam.cu -- NEXT-2: the optimizer step that follows the
// gradient exchange of the data-parallel stage.  Adam (Kingma & Ba 2015,
// Algorithm 1) with the paper's setting (beta1 0.9,
// beta2 0.999, eps 1e-8, lr 1e-3), on fp32 master weights and moments, with an
// optional bf16 copy of the updated weights for the next step's GEMMs.
//
//   attn_adam_step          replicated update of n parameters
//   attn_adam_step_sharded  reduce-scatter of the summed gradient (NCCL, fp32),
//                           update of this rank's contiguous shard, all-gather
//                           of the bf16 weights: 4 + 2 bytes per parameter on
//                           the wire instead of the 8 of allreduce + replicated
//                           update, and 1/R of the optimizer state per GPU.
//
// The update is HBM-bound: 16 bytes read (w, m, v, g) and 12 + 2 written per
// parameter, float4-vectorised, grid sized to the SM count.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>

#include "../../include/attn_softmax.h"
#include "nvtx.cuh"
#include "comm.h"

attn_status_t attn_set_error(attn_status_t code, const char* msg);

namespace {

attn_status_t fail(attn_status_t code, const char* msg) { return attn_set_error(code, msg); }

struct AdamK {
  float lr, b1, omb1, b2, omb2, eps, inv_bc1, inv_bc2;   // omb = 1 - beta (from double)
};

__device__ __forceinline__ void adam1(float& w, float& m, float& v, float g, const AdamK& k) {
  m = k.b1 * m + k.omb1 * g;
  v = k.b2 * v + k.omb2 * g * g;
  const float mhat = m * k.inv_bc1;
  const float vhat = v * k.inv_bc2;
  w = w - k.lr * mhat / (sqrtf(vhat) + k.eps);
}

__global__ void __launch_bounds__(256) adam_kernel(float* __restrict__ w, float* __restrict__ m,
                                                   float* __restrict__ v,
                                                   const float* __restrict__ g,
                                                   __nv_bfloat16* __restrict__ wb, long long n,
                                                   AdamK k) {
  const long long n4 = n / 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  float4* w4 = reinterpret_cast<float4*>(w);
  float4* m4 = reinterpret_cast<float4*>(m);
  float4* v4 = reinterpret_cast<float4*>(v);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 a = w4[i], b = m4[i], c = v4[i];
    const float4 d = g4[i];
    adam1(a.x, b.x, c.x, d.x, k);
    adam1(a.y, b.y, c.y, d.y, k);
    adam1(a.z, b.z, c.z, d.z, k);
    adam1(a.w, b.w, c.w, d.w, k);
    w4[i] = a;
    m4[i] = b;
    v4[i] = c;
    if (wb) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(a.x, a.y), hi = __floats2bfloat162_rn(a.z, a.w);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&lo);
      u.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(wb)[i] = u;
    }
  }
  // tail (n % 4 elements)
  const long long t = 4 * n4 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) {
    float a = w[t], b = m[t], c = v[t];
    adam1(a, b, c, g[t], k);
    w[t] = a;
    m[t] = b;
    v[t] = c;
    if (wb) wb[t] = __float2bfloat16_rn(a);
  }
}

bool misaligned(const void* p) { return p && (reinterpret_cast<uintptr_t>(p) & 15); }

attn_status_t check(const attn_adam_t* h) {
  if (!h) return fail(ATTN_ERR_INVALID_ARG, "adam: hyper-parameters are NULL");
  if (h->step < 1) return fail(ATTN_ERR_INVALID_ARG, "adam: step must be >= 1 (Kingma & Ba Alg. 1)");
  if (!(h->beta1 >= 0.0 && h->beta1 < 1.0) || !(h->beta2 >= 0.0 && h->beta2 < 1.0) ||
      !(h->eps > 0.0) || !(h->lr >= 0.0))
    return fail(ATTN_ERR_INVALID_ARG, "adam: need 0 <= beta1, beta2 < 1, eps > 0, lr >= 0");
  return ATTN_OK;
}

AdamK consts(const attn_adam_t* h) {
  AdamK k;
  k.lr = (float)h->lr;
  k.b1 = (float)h->beta1;
  k.omb1 = (float)(1.0 - h->beta1);
  k.b2 = (float)h->beta2;
  k.omb2 = (float)(1.0 - h->beta2);
  k.eps = (float)h->eps;
  k.inv_bc1 = (float)(1.0 / (1.0 - std::pow(h->beta1, (double)h->step)));
  k.inv_bc2 = (float)(1.0 / (1.0 - std::pow(h->beta2, (double)h->step)));
  return k;
}

attn_status_t launch(float* w, float* m, float* v, const float* g, void* wb, size_t n,
                     const AdamK& k, cudaStream_t s) {
  if (n == 0) return ATTN_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long n4 = (long long)n / 4;
  long long blocks = (n4 + 255) / 256;
  if (blocks > (long long)sms * 8) blocks = (long long)sms * 8;
  if (blocks < 1) blocks = 1;
  adam_kernel<<<(int)blocks, 256, 0, s>>>(w, m, v, g, static_cast<__nv_bfloat16*>(wb),
                                          (long long)n, k);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    char buf[256];
    snprintf(buf, sizeof(buf), "adam_kernel launch: %s", cudaGetErrorString(e));
    return fail(ATTN_ERR_CUDA, buf);
  }
  return ATTN_OK;
}

}  // namespace

extern "C" attn_status_t attn_adam_step(const attn_adam_t* h, size_t n, float* w, float* m,
                                        float* v, const float* g, void* w_bf16, void* stream) {
  attnsm::NvtxRange nvtx_range_("attn_adam_step");
  attn_status_t st = check(h);
  if (st != ATTN_OK) return st;
  if (n && (!w || !m || !v || !g)) return fail(ATTN_ERR_INVALID_ARG, "adam: w / m / v / g is NULL");
  if (misaligned(w) || misaligned(m) || misaligned(v) || misaligned(g) ||
      (w_bf16 && (reinterpret_cast<uintptr_t>(w_bf16) & 7)))
    return fail(ATTN_ERR_UNSUPPORTED, "adam: fp32 buffers need 16-byte, w_bf16 8-byte alignment");
  return launch(w, m, v, g, w_bf16, n, consts(h), (cudaStream_t)stream);
}

extern "C" size_t attn_adam_shard_len(const attn_comm_t* c, size_t n) {
  const size_t R = (size_t)comm_nranks(c);
  const size_t per = (n + R - 1) / R;
  return (per + 3) / 4 * 4;
}

extern "C" attn_status_t attn_adam_step_sharded(attn_comm_t* c, const attn_adam_t* h, size_t n,
                                                float* g, float* w_shard, float* m_shard,
                                                float* v_shard, void* w_bf16, void* stream) {
  attnsm::NvtxRange nvtx_range_("attn_adam_step_sharded");
  attn_status_t st = check(h);
  if (st != ATTN_OK) return st;
  if (!c) return fail(ATTN_ERR_INVALID_ARG, "adam_sharded: comm is NULL (use attn_adam_step)");
  if (n && (!g || !w_shard || !m_shard || !v_shard || !w_bf16))
    return fail(ATTN_ERR_INVALID_ARG, "adam_sharded: a buffer is NULL");
  if (misaligned(g) || misaligned(w_shard) || misaligned(m_shard) || misaligned(v_shard) ||
      misaligned(w_bf16))
    return fail(ATTN_ERR_UNSUPPORTED, "adam_sharded: buffers need 16-byte alignment");
  if (n == 0) return ATTN_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t S = attn_adam_shard_len(c, n);
  const size_t R = (size_t)comm_nranks(c), r = (size_t)comm_rank(c);
  if (R * S > n) {   // zero the padded tail of the gradient
    cudaError_t e = cudaMemsetAsync(g + n, 0, sizeof(float) * (R * S - n), s);
    if (e != cudaSuccess) return fail(ATTN_ERR_CUDA, cudaGetErrorString(e));
  }
  if ((st = comm_reduce_scatter_f32(c, g, S, s)) != ATTN_OK) return st;
  __nv_bfloat16* wb = static_cast<__nv_bfloat16*>(w_bf16) + r * S;
  if ((st = launch(w_shard, m_shard, v_shard, g + r * S, wb, S, consts(h), s)) != ATTN_OK) return st;
  return comm_all_gather_bf16(c, w_bf16, S, s);
}
