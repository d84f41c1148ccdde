// gemm_simt.cuh -- fp32 CUDA-core GEMM engines.
//
// (1) gemm_simt_kernel: the fp32-path counterpart of gemm_tc_kernel with the
//     same problem description and the same row epilogues.  TF32 tensor cores
//     would miss the 1e-5 fp32 parity bar (SURVEY.md §7 "hard parts"), so the
//     fp32 path runs FFMA.  64x64 tiles, 256 threads, 4x4 outputs per thread.
// (2) bgemm_kernel: batched per-sentence GEMM with strided operands and an
//     optional second K segment, used by the attention steps (Eqs. 1-3 and
//     their backward) of both dtype paths: fp32 accumulation, operands fp32 or
//     bf16.
#pragma once
#include "epilogue.cuh"

namespace attnsm {

constexpr int SG_BM = 64;
constexpr int SG_BN = 64;
constexpr int SG_BK = 16;

struct SimtProblem {
  int M, N, K;
  int tiles_m, tiles_n, k_splits, k_per_split;
  int tile_begin;
  // A(m,k) = a0[m*sam + k*sak]            for k <  a_ksplit (or a1 == null)
  //        = a1[m*sam + (k-a_ksplit)*sak] for k >= a_ksplit
  const float* a0; const float* a1; long long sam, sak; int a_ksplit;
  // B(n,k) = b0[n*sbn + (k+b_koff)*sbk] for n < b_nsplit (or b1 == null), else b1 at n-b_nsplit
  const float* b0; const float* b1; long long sbn, sbk; int b_nsplit; int b_koff;
  EpiParams epi;
};

struct SimtParams {
  SimtProblem prob[4];
  int nprob;
};

__device__ __forceinline__ float simt_a(const SimtProblem& p, int m, int k) {
  if (m >= p.M || k >= p.K) return 0.f;
  if (p.a1 && k >= p.a_ksplit) return p.a1[m * p.sam + (long long)(k - p.a_ksplit) * p.sak];
  return p.a0[m * p.sam + (long long)k * p.sak];
}
__device__ __forceinline__ float simt_b(const SimtProblem& p, int n, int k) {
  if (n >= p.N || k >= p.K) return 0.f;
  const long long kk = (long long)(k + p.b_koff) * p.sbk;
  if (p.b1 && n >= p.b_nsplit) return p.b1[(long long)(n - p.b_nsplit) * p.sbn + kk];
  return p.b0[(long long)n * p.sbn + kk];
}

template <typename OutT>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const __grid_constant__ SimtParams P) {
  __shared__ float As[SG_BK][SG_BM + 4];
  __shared__ float Bs[SG_BK][SG_BN + 4];
  __shared__ float Cs[SG_BM][SG_BN + 1];
  const int t = blockIdx.x;
  int pi = 0;
  for (int i = 1; i < P.nprob; ++i)
    if (t >= P.prob[i].tile_begin) pi = i;
  const SimtProblem& p = P.prob[pi];
  int local = t - p.tile_begin;
  const int per_split = p.tiles_m * p.tiles_n;
  const int split = local / per_split;
  local -= split * per_split;
  const int m0 = (local % p.tiles_m) * SG_BM;
  const int tn = local / p.tiles_m;
  const int n0 = tn * SG_BN;
  const int kbeg = split * p.k_per_split;
  const int kend = min(p.K, kbeg + p.k_per_split);

  const int tid = threadIdx.x;
  const int ty = tid / 16, tx = tid % 16;
  float acc[4][4] = {};
  for (int k0 = kbeg; k0 < kend; k0 += SG_BK) {
    for (int i = tid; i < SG_BK * SG_BM; i += 256) {
      const int kk = i / SG_BM, mm = i % SG_BM;
      const int k = k0 + kk;
      As[kk][mm] = (k < kend) ? simt_a(p, m0 + mm, k) : 0.f;
      Bs[kk][mm] = (k < kend) ? simt_b(p, n0 + mm, k) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SG_BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) Cs[ty * 4 + i][tx * 4 + j] = acc[i][j];
  __syncthreads();
  if (tid < SG_BM) {
    const int row = m0 + tid;
    if (row < p.M) {
      RowEpilogue<OutT, false> epi(p.epi, row, split);
#pragma unroll 1
      for (int c = 0; c < SG_BN / 32; ++c) {
        if (n0 + c * 32 >= p.N) break;
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = Cs[tid][c * 32 + j];
        epi.chunk(n0 + c * 32, v);
      }
      epi.finish(tn);
    }
  }
}

// ------------------------------------------------------------------ bgemm
// out[b](m,n) = alpha_sum_k A[b](m,k) B[b](n,k)  (+ add[b](m,n))
// with two K segments: k < K0 uses (a0,b0), k >= K0 uses (a1,b1) at k-K0.
template <typename TA, typename TB>
struct BSeg {
  const TA* a; long long sab, sam, sak;
  const TB* b; long long sbb, sbn, sbk;
};

template <typename TA0, typename TB0, typename TA1, typename TB1, typename OutT>
struct BGemm {
  int batch, M, N, K0, K1;
  BSeg<TA0, TB0> s0;
  BSeg<TA1, TB1> s1;
  OutT* out; long long sob, som, son;
  const float* add; long long sadd_b, sadd_m, sadd_n;   // optional addend (fp32)
};

template <typename TA0, typename TB0, typename TA1, typename TB1, typename OutT>
__global__ void __launch_bounds__(256) bgemm_kernel(const __grid_constant__ BGemm<TA0, TB0, TA1, TB1, OutT> g) {
  __shared__ float As[SG_BK][SG_BM + 4];
  __shared__ float Bs[SG_BK][SG_BN + 4];
  const int b = blockIdx.z;
  const int m0 = blockIdx.y * SG_BM;
  const int n0 = blockIdx.x * SG_BN;
  const int tid = threadIdx.x;
  const int ty = tid / 16, tx = tid % 16;
  float acc[4][4] = {};
  const int K = g.K0 + g.K1;
  for (int k0 = 0; k0 < K; k0 += SG_BK) {
    for (int i = tid; i < SG_BK * SG_BM; i += 256) {
      // consecutive threads walk the operand's unit-stride dimension when it
      // is k (row-major [m,k]) -- loads are coalesced for both layouts used
      const int kk = i % SG_BK, mm = i / SG_BK;
      const int k = k0 + kk, m = m0 + mm, n = n0 + mm;
      float av = 0.f, bv = 0.f;
      if (k < g.K0) {
        if (m < g.M) av = to_f32(g.s0.a[b * g.s0.sab + m * g.s0.sam + (long long)k * g.s0.sak]);
        if (n < g.N) bv = to_f32(g.s0.b[b * g.s0.sbb + n * g.s0.sbn + (long long)k * g.s0.sbk]);
      } else if (k < K) {
        const int k1 = k - g.K0;
        if (m < g.M) av = to_f32(g.s1.a[b * g.s1.sab + m * g.s1.sam + (long long)k1 * g.s1.sak]);
        if (n < g.N) bv = to_f32(g.s1.b[b * g.s1.sbb + n * g.s1.sbn + (long long)k1 * g.s1.sbk]);
      }
      As[kk][mm] = av;
      Bs[kk][mm] = bv;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SG_BK; ++kk) {
      float a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= g.N) continue;
      float v = acc[i][j];
      if (g.add) v += g.add[b * g.sadd_b + m * g.sadd_m + n * g.sadd_n];
      g.out[b * g.sob + m * g.som + n * g.son] = to_out<OutT>(v);
    }
  }
}

}  // namespace attnsm
