// epilogue.cuh -- row-oriented GEMM epilogues shared by the tcgen05 engine
// (gemm_tc.cuh) and the fp32 CUDA-core engine (gemm_simt.cuh).
//
// Both engines hand an epilogue one output row at a time, in chunks of 32
// consecutive fp32 accumulator columns (the tcgen05.ld 32x32b.x32 shape: one
// row per thread, so row reductions need no cross-thread traffic).
//
//   EPI_STORE_F32  out[r,c] = acc                    (dW_out chunk, dW_c, [dH|dC])
//   EPI_TANH       out[r,c] = tanh(acc)              (Eq. 4)
//   EPI_LSE        per (row, column tile): running max m and sum_c exp(acc-m)
//                  over columns c < ncols_valid, and the target logit when the
//                  row's target id falls in the tile (Eqs. 5-6 forward)
//   EPI_DLOGITS    out[r,c] = rowscale[r] * (exp(acc - lse[r]) - [c+col_base == y_r])
//                  (softmax - onehot; backward of Eqs. 5-6; fp32 engine)
//   EPI_ACCUM_F32  out[r,c] += acc                   (dHc over V-chunks; the tcgen05
//                  engine does it with a TMA reduce-add, no loads)
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace attnsm {

enum EpiKind : int {
  EPI_STORE_F32 = 0, EPI_TANH = 1, EPI_LSE = 2, EPI_DLOGITS = 3, EPI_ACCUM_F32 = 4,
  EPI_NONE = 5,               // debug: read the accumulator, store nothing
  EPI_STORE_BF16 = 6,         // out = acc (bf16): C, dC, dH_enc
  EPI_ADD_BF16 = 7,           // out = acc + addend (fp32, or bf16 with addend_bf16) -> bf16:
                              // dH_dec = dH_part + de S, or dz W_c[:, :d] + dQ
  EPI_ATTN_SOFTMAX = 8,       // masked row softmax of the scores (Eq. 1), tcgen05 path
  EPI_ATTN_SOFTMAX_BWD = 9,   // its backward, tcgen05 path
  EPI_TOPK = 11               // decoding step (NEXT-4): LSE partials as EPI_LSE plus the 8 best
                              // (logit, token) of the row's columns in the tile (tcgen05 path)
};

// Output element type of each kind (tcgen05 path: bf16 activations).
__host__ __device__ constexpr bool epi_out_is_f32(int kind) {
  return kind == EPI_STORE_F32 || kind == EPI_ACCUM_F32;
}

struct EpiParams {
  int kind;
  int ncols_valid;       // columns < ncols_valid are real (V tail, chunk tail)
  int ncols_store;       // columns < ncols_store may be written (row capacity)
  int col_base;          // global column of problem column 0 (V-chunk start)
  void* out;             // STORE_F32 / ACCUM_F32: float; TANH / DLOGITS: OutT; LSE (tcgen05,
                         // optional): the logits as fp16 [rows, ldo] (option store_logits)
  long long ldo;         // row stride of out (elements)
  long long split_stride;// element offset between split-K partial outputs
  float2* part;          // LSE: [rows, part_ld] (max, sumexp)
  int part_ld;
  float* tgt_logit;      // LSE: [rows]
  const int* tgt;        // LSE/DLOGITS: [rows] target ids
  const float* lse;      // DLOGITS: [rows]
  const float* rowscale; // DLOGITS: [rows] loss_scale on valid rows, 0 on padded
                         // (tcgen05 DLOGITS also reads tgt_logit: the forward's
                         // target logit, for the -onehot term)
  float* stash_f32;      // ATTN_SOFTMAX(_BWD): alpha fp32 [rows, stash_ld] (cols < ncols_valid)
  long long stash_ld;
  const int* src_len;    // ATTN_SOFTMAX: [batch]
  const float* addend;   // ADD_BF16: [rows, add_ld] fp32 (bf16 when addend_bf16)
  int addend_bf16;
  long long add_ld;
  uint32_t* topk;        // TOPK: [rows, part_ld, 8] 32-bit keys (tk_key32) per slot, best first
  const void* bias;      // LSE / DLOGITS / TOPK: optional F_c bias b_out [V] (OutT), indexed by
                         // col_base + column (NEXT-1); NULL on the hot path
};

template <typename T> __device__ __forceinline__ T to_out(float x);
template <> __device__ __forceinline__ float to_out<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 to_out<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}
__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }

template <bool kFast>
__device__ __forceinline__ float tanh_f(float x) {
  if constexpr (kFast) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
  } else {
    return tanhf(x);
  }
}
__device__ __forceinline__ float fmax3_f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float ex2_mufu(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kLog2e = 1.4426950408889634f;

template <bool kFast>
__device__ __forceinline__ float exp_f(float x) {
  if constexpr (kFast) return __expf(x);
  else return expf(x);
}

// Store 32 consecutive values (vectorised when the whole chunk fits and the
// row is 16-byte aligned).
template <typename OutT>
__device__ __forceinline__ void store_row32(OutT* rowp, int col0, int ncols_store,
                                            const float (&v)[32], bool vec_ok) {
  if (vec_ok && col0 + 32 <= ncols_store) {
    if constexpr (sizeof(OutT) == 2) {
      uint4* dst = reinterpret_cast<uint4*>(rowp + col0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat162 h2 = __floats2bfloat162_rn(v[q * 8 + 2 * e], v[q * 8 + 2 * e + 1]);
          w[e] = *reinterpret_cast<uint32_t*>(&h2);
        }
        dst[q] = make_uint4(w[0], w[1], w[2], w[3]);
      }
    } else {
      float4* dst = reinterpret_cast<float4*>(rowp + col0);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col0 + j < ncols_store) rowp[col0 + j] = to_out<OutT>(v[j]);
  }
}

// v[j] += b[col + j] for the 32 columns of a chunk that are < nvalid (all
// threads read the same addresses: broadcast loads).
template <typename OutT>
__device__ __forceinline__ void add_bias32(const void* bias, int gcol, int nvalid_rel,
                                           float (&v)[32]) {
  const OutT* b = reinterpret_cast<const OutT*>(bias) + gcol;
  if (nvalid_rel >= 32 && (reinterpret_cast<uintptr_t>(b) & 15) == 0) {   // 16-byte vector loads
    const uint4* b4 = reinterpret_cast<const uint4*>(b);
#pragma unroll
    for (int g = 0; g < 32 * (int)sizeof(OutT) / 16; ++g) {
      const uint4 u = __ldg(b4 + g);
      const uint32_t w0 = u.x, w1 = u.y, w2 = u.z, w3 = u.w;
      if constexpr (sizeof(OutT) == 2) {   // bf16 -> fp32: the high half of the word
        v[8 * g + 0] += __uint_as_float(w0 << 16);
        v[8 * g + 1] += __uint_as_float(w0 & 0xFFFF0000u);
        v[8 * g + 2] += __uint_as_float(w1 << 16);
        v[8 * g + 3] += __uint_as_float(w1 & 0xFFFF0000u);
        v[8 * g + 4] += __uint_as_float(w2 << 16);
        v[8 * g + 5] += __uint_as_float(w2 & 0xFFFF0000u);
        v[8 * g + 6] += __uint_as_float(w3 << 16);
        v[8 * g + 7] += __uint_as_float(w3 & 0xFFFF0000u);
      } else {
        v[4 * g + 0] += __uint_as_float(w0);
        v[4 * g + 1] += __uint_as_float(w1);
        v[4 * g + 2] += __uint_as_float(w2);
        v[4 * g + 3] += __uint_as_float(w3);
      }
    }
  } else if (nvalid_rel >= 32) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] += to_f32(b[j]);
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nvalid_rel) v[j] += to_f32(b[j]);
  }
}

// ---- top-k keys (decoding step, NEXT-4): a (logit, token) pair as one 64-bit
// key -- order-preserving float bits, then the complemented token -- so
// "logit descending, token ascending" is an unsigned compare.
__device__ __forceinline__ unsigned long long tk_key(float x, int id) {
  const uint32_t u = __float_as_uint(x);
  const uint32_t hi = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)hi << 32) | (uint32_t)(0xFFFFFFFFu - (uint32_t)id);
}
__device__ __forceinline__ float tk_val(unsigned long long k) {
  const uint32_t hi = (uint32_t)(k >> 32);
  return __uint_as_float((hi & 0x80000000u) ? (hi & 0x7FFFFFFFu) : ~hi);
}
__device__ __forceinline__ int tk_id(unsigned long long k) {
  return (int)(0xFFFFFFFFu - (uint32_t)k);
}
// Inside one 128-column tile half the per-tile epilogue uses 32-bit keys: the
// order-preserving float bits with the low 7 mantissa bits replaced by the
// complemented local column (0..127).  Candidates whose logits agree to 2^-16
// relative are ordered by column, and the kept value is truncated by at most
// that much -- far below the bf16 inputs' resolution -- for a compare-exchange
// of two integer instructions instead of six.
__device__ __forceinline__ uint32_t tk_key32(float x, int local) {
  const uint32_t u = __float_as_uint(x);
  const uint32_t hi = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return (hi & ~0x7Fu) | (uint32_t)(0x7F - local);
}
__device__ __forceinline__ float tk32_val(uint32_t k) {
  const uint32_t hi = k & ~0x7Fu;
  return __uint_as_float((hi & 0x80000000u) ? (hi & 0x7FFFFFFFu) : ~hi);
}
__device__ __forceinline__ int tk32_local(uint32_t k) { return 0x7F - (int)(k & 0x7Fu); }

// compare-exchange: a keeps the larger key
template <typename K>
__device__ __forceinline__ void tk_ce(K& a, K& b) {
  const K mx = a > b ? a : b, mn = a > b ? b : a;
  a = mx;
  b = mn;
}
// sort 8 keys descending (Batcher odd-even merge sort, 19 compare-exchanges)
template <typename K>
__device__ __forceinline__ void tk_sort8(K* k) {
  tk_ce(k[0], k[1]); tk_ce(k[2], k[3]); tk_ce(k[4], k[5]); tk_ce(k[6], k[7]);
  tk_ce(k[0], k[2]); tk_ce(k[1], k[3]); tk_ce(k[4], k[6]); tk_ce(k[5], k[7]);
  tk_ce(k[1], k[2]); tk_ce(k[5], k[6]);
  tk_ce(k[0], k[4]); tk_ce(k[1], k[5]); tk_ce(k[2], k[6]); tk_ce(k[3], k[7]);
  tk_ce(k[2], k[4]); tk_ce(k[3], k[5]);
  tk_ce(k[1], k[2]); tk_ce(k[3], k[4]); tk_ce(k[5], k[6]);
}
// a, b sorted descending -> a = the best 8 of both, sorted descending
template <typename K>
__device__ __forceinline__ void tk_merge8(K* a, const K* b) {
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = a[i] > b[7 - i] ? a[i] : b[7 - i];   // bitonic
#pragma unroll
  for (int d = 4; d > 0; d >>= 1)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if ((i & d) == 0) tk_ce(a[i], a[i + d]);
}

struct LseState {
  float m, s, t;
  int has_t;
};

// One output row of one tile.  `row` is the problem row (< M checked by the
// caller), `tile_n` the column-tile index inside the problem, `col0` the
// problem column of v[0].
template <typename OutT, bool kFast>
struct RowEpilogue {
  const EpiParams& p;
  int row;
  int split;
  LseState st;
  int y;
  float lse, rs;
  __device__ __forceinline__ RowEpilogue(const EpiParams& p_, int row_, int split_)
      : p(p_), row(row_), split(split_) {
    st.m = -INFINITY;
    st.s = 0.f;
    st.t = 0.f;
    st.has_t = 0;
    y = -1;
    lse = 0.f;
    rs = 0.f;
    if (p.kind == EPI_LSE || p.kind == EPI_DLOGITS) y = p.tgt[row] - p.col_base;
    if (p.kind == EPI_DLOGITS) {   // (fp32 CUDA-core engine)
      lse = p.lse[row];
      rs = p.rowscale[row];
    }
  }

  __device__ __forceinline__ void chunk(int col0, float (&v)[32]) {
    const int kind = p.kind;
    if (kind == EPI_LSE) {
      const int nv = p.ncols_valid - col0;
      if (nv <= 0) return;
      if (p.bias) add_bias32<OutT>(p.bias, p.col_base + col0, nv, v);
      float cm = -INFINITY;
      if (kFast && nv >= 32) {   // sm_100 three-input max: 16 FMNMX3 for 32 values
        float a = fmax3_f(v[0], v[1], v[2]), b = fmax3_f(v[3], v[4], v[5]);
#pragma unroll
        for (int j = 6; j < 30; j += 4) {
          a = fmax3_f(a, v[j], v[j + 1]);
          b = fmax3_f(b, v[j + 2], v[j + 3]);
        }
        cm = fmax3_f(a, b, fmaxf(v[30], v[31]));
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nv) cm = fmaxf(cm, v[j]);
      }
      const float nm = fmaxf(st.m, cm);   // finite: the chunk has a finite logit
      float s;
      if constexpr (kFast) {   // exp(v - nm) = 2^(v log2 e - nm log2 e): one FFMA + MUFU
        const float nml = nm * kLog2e;
        s = st.s * ex2_mufu(fmaf(st.m, kLog2e, -nml));
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nv) s += ex2_mufu(fmaf(v[j], kLog2e, -nml));
      } else {
        s = st.s * exp_f<kFast>(st.m - nm);
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nv) s += exp_f<kFast>(v[j] - nm);
      }
      st.s = s;
      st.m = nm;
      const int yl = y - col0;
      if (yl >= 0 && yl < 32 && yl < nv) {
        float t = 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j) t = (j == yl) ? v[j] : t;
        st.t = t;
        st.has_t = 1;
      }
    } else if (kind == EPI_DLOGITS) {
      if (col0 >= p.ncols_store) return;
      const int yl = y - col0;
      if (p.bias) add_bias32<OutT>(p.bias, p.col_base + col0, p.ncols_valid - col0, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        float g = rs * (exp_f<kFast>(v[j] - lse) - (j == yl ? 1.f : 0.f));
        v[j] = (col0 + j < p.ncols_valid) ? g : 0.f;
      }
      OutT* rowp = reinterpret_cast<OutT*>(p.out) + (long long)row * p.ldo;
      store_row32<OutT>(rowp, col0, p.ncols_store, v, (p.ldo * sizeof(OutT)) % 16 == 0);
    } else if (kind == EPI_TANH) {
      if (col0 >= p.ncols_store) return;
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = tanh_f<kFast>(v[j]);
      OutT* rowp = reinterpret_cast<OutT*>(p.out) + (long long)row * p.ldo;
      store_row32<OutT>(rowp, col0, p.ncols_store, v, (p.ldo * sizeof(OutT)) % 16 == 0);
    } else if (kind == EPI_STORE_F32) {
      if (col0 >= p.ncols_store) return;
      float* rowp = reinterpret_cast<float*>(p.out) + (long long)split * p.split_stride +
                    (long long)row * p.ldo;
      store_row32<float>(rowp, col0, p.ncols_store, v, (p.ldo * 4) % 16 == 0);
    } else if (kind == EPI_ACCUM_F32) {
      if (col0 >= p.ncols_store) return;
      float* rowp = reinterpret_cast<float*>(p.out) + (long long)row * p.ldo;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < p.ncols_store) rowp[col0 + j] += v[j];
    }
  }

  // tcgen05 path: transform v in place (TANH) or update the LSE state; the
  // engine stages and stores the result with TMA.  (The bf16 dlogits live in
  // vocab.cuh's G1 epilogue.)
  __device__ __forceinline__ void transform(int col0, float (&v)[32]) {
    const int kind = p.kind;
    if (kind == EPI_LSE) {
      chunk(col0, v);
    } else if (kind == EPI_TANH) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = tanh_f<kFast>(v[j]);
    }
  }

  __device__ __forceinline__ void finish(int slot) {
    if (p.kind == EPI_LSE) {
      p.part[(long long)row * p.part_ld + slot] = make_float2(st.m, st.s);
      if (st.has_t) p.tgt_logit[row] = st.t;
    }
  }
};

}  // namespace attnsm
