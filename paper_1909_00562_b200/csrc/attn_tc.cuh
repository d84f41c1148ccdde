// attn_tc.cuh -- the attention steps of the stage as one tcgen05 kernel per
// direction, ONE CTA PER SENTENCE (bf16 path, N <= 128 decoder rows, M <= 128
// source positions, d % 64 == 0):
//
//   attn_fwd_kernel   F1 + Eq. 1 + F2 (Eqs. 1-3):
//       E = Q S^T (K = d streamed through a TMA ring, fp32 in TMEM), the
//       length-masked row softmax in registers (alpha = 0 exactly for
//       j >= src_len), alpha written once (the fp32 stash the backward reads)
//       and kept in shared memory as the bf16 A operand of the context MMA
//       C = alpha S, S streamed a second time (from L2) as the MN-major B.
//   attn_bwd_kernel   B3 (the backward of Eqs. 1-3):
//       dalpha = dC S^T (TMEM), de = alpha (dalpha - sum_j alpha dalpha) in
//       registers -> bf16 in shared memory; then per 64-column chunk of d
//       dQ = de S and dH_enc = alpha^T dC + de^T Q (two K segments), S / dC /
//       Q streamed by TMA, fp32 accumulators in TMEM.  dQ leaves as bf16: the
//       projection backward adds it to dz W_c[:, :d] in its epilogue (dot
//       score: dH_dec = dz W_c[:, :d] + dQ), so no fp32 dH_part round trip.
//
// They replace the two (forward) and two (backward) batched launches of the
// generic engine, where each sentence's rows took a 128-row tile of a
// separate score and context GEMM and alpha / de made an HBM round trip in
// between.  The kernels are latency-bound (26 MB / 41 MB of HBM reads at C1):
// the ring holds as many operand blocks as fit (boxes cut to the sentence's
// rows rounded to 16), and each epilogue warp double-buffers its TMA stores.
//
// Shared-memory operand layouts (128-byte swizzle, DESIGN.md "tcgen05
// encodings"): a [rows, 64] K-major block of bf16 is rows x 128 B, 8-row
// groups 1024 B apart; the SAME bytes, read as an MN-major operand, are one
// 64-element MN atom with K = rows (LBO = the distance to the next 64-element
// atom, SBO = 1024 B, K step 16 rows = 2048 B).  So one TMA box of S_b
// [mbox rows, 64 columns] serves as the K-major B of the score MMA and as an
// MN-major B atom of the context MMA, and the bf16 alpha / de tiles [128 rows
// i][128 columns j] serve as K-major A (K = j) and, for dH_enc, as MN-major A
// (M = j, K = i).
//
// Rows past a sentence: A-operand rows >= qrows (the Q / dC box) hold stale
// shared memory, which only reaches accumulator rows >= N (clipped by the
// TMA stores; the backward zeroes alpha / de there); S rows in [M, mbox) and
// dC / Q rows in [N, qrows) are zero-filled by TMA because they are K rows of
// a product.
//
// Roles (320 threads): warps 0-7 softmax / epilogue (warp w: TMEM lanes
// 32 (w % 4).., column half w / 4), warp 8 TMA producer + TMEM allocator,
// warp 9 MMA issuer (one elected lane).
#pragma once
#include "gemm_tc.cuh"

namespace attnsm {

constexpr int AT_THREADS = 320;
constexpr int AT_STG = 8192;                          // staging per epilogue warp: 2 x 4 KB
constexpr int AT_SLOTS = 4;                           // TMEM: 4 x 128 fp32 columns
constexpr int AT_OPA = 32 * 1024;                     // one bf16 [128 x 128] A tile (2 atoms)
constexpr int AT_MAXST = 8;                           // ring stages (barrier slots)
constexpr int ATF_RING = 112 * 1024;
constexpr int ATF_SMEM = ATF_RING + AT_OPA + 8 * AT_STG + 1024 + 512;
constexpr int ATB_RING = 96 * 1024;
constexpr int ATB_SMEM = ATB_RING + 2 * AT_OPA + 8 * AT_STG + 1024 + 512;

struct alignas(64) AttnFwdParams {
  CUtensorMap m_q;      // Q [B][N][d] bf16 (H_dec, or H W_alpha), box {64, qrows, 1}
  CUtensorMap m_s;      // S = H_enc [B][M][d] bf16, box {64, mbox, 1}
  CUtensorMap m_c;      // C store [B][N][d] bf16, box {64, 32, 1}
  CUtensorMap m_stash;  // alpha fp32 [B][N][ald], dims {M, N, B}, box {32, 32, 1}
  CUtensorMap m_abf;    // alpha bf16 [B][N][Mp], dims {Mp, N, B}, box {32, 32, 1}, 64-byte swizzle
  const int* src_len;   // [B] (device)
  int d, mbox, qrows;   // mbox = M rounded up to 64, qrows = N rounded up to 16
  int store_abf;        // also store the bf16 alpha copy (the generic backward's operand)
  long long* trace;     // debug (option "attn_trace"): 8 globaltimer stamps per CTA, NULL = off
};

struct alignas(64) AttnBwdParams {
  CUtensorMap m_dc;     // dC [B][N][d] bf16, box {64, qrows, 1}
  CUtensorMap m_s;      // S [B][M][d] bf16, box {64, mbox, 1}
  CUtensorMap m_q;      // Q [B][N][d] bf16 (H_dec, or H W_alpha), box {64, qrows, 1}
  CUtensorMap m_dq;     // dQ = de S store [B][N][d] bf16, box {64, 32, 1}
  CUtensorMap m_dhe;    // dH_enc store [B][M][d] bf16, box {64, 32, 1}
  const float* alpha;   // fp32 stash [B*N][ald]
  int N, M, d, ald, mbox, qrows;
  long long* trace;     // debug: 8 globaltimer stamps per CTA, NULL = off
};

// stamp i of this CTA's trace record (lane 0 of the calling warp)
#define AT_TRACE(i)                                                           \
  do {                                                                        \
    if (P.trace && lane == 0) P.trace[(long long)blockIdx.x * 16 + (i)] = gtime(); \
  } while (0)

// phase-2 chunk stamps of the backward: [B][64 chunks][4] after the stage's 8-word record block
#define AT_TRACE2(j, i)                                                                   \
  do {                                                                                    \
    if (P.trace && lane == 0 && (j) < 64)                                                 \
      P.trace[(long long)gridDim.x * 16 + ((long long)blockIdx.x * 64 + (j)) * 4 + (i)] = gtime(); \
  } while (0)

// bf16 of 32 consecutive row values into a K-major [128 x 128] A tile
// (two 64-wide atoms of 16 KB): row r, columns [c32 * 32, c32 * 32 + 32)
__device__ __forceinline__ void at_put_row32(uint32_t tile, int r, int c32, const float (&v)[32]) {
  const uint32_t base = tile + (c32 >> 1) * 16384 + r * 128;
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      __nv_bfloat162 h2 = __floats2bfloat162_rn(v[8 * g + 2 * e], v[8 * g + 2 * e + 1]);
      w[e] = *reinterpret_cast<uint32_t*>(&h2);
    }
    const uint32_t gi = (c32 & 1) * 4 + g;
    st_shared_v4(base + ((gi ^ (r & 7)) << 4), w[0], w[1], w[2], w[3]);
  }
}

// 32 rows x 64 bf16 columns of this warp through half `buf` of its staging
// (128-byte swizzle) to a {64, 32, 1} TMA box at (col, row0, b); the other
// half's store may still be reading shared memory
__device__ __forceinline__ void at_store64_bf16(uint8_t* stg, int buf, const CUtensorMap* m,
                                                const float (&v)[64], int col, int row0, int b,
                                                uint32_t lane) {
  uint8_t* half = stg + buf * 4096;
  const uint32_t s = smem_u32(half);
  if (lane == 0) bulk_wait_read1();
  __syncwarp();
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      __nv_bfloat162 h2 = __floats2bfloat162_rn(v[8 * g + 2 * e], v[8 * g + 2 * e + 1]);
      w[e] = *reinterpret_cast<uint32_t*>(&h2);
    }
    st_shared_v4(s + lane * 128 + ((g ^ (lane & 7)) << 4), w[0], w[1], w[2], w[3]);
  }
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_store_3d(m, half, col, row0, b);
    bulk_commit();
  }
}

__device__ __forceinline__ void at_ld64(uint32_t taddr, float (&v)[64]) {
  float a[32], c[32];
  tmem_ld32(taddr, a);
  tmem_ld32(taddr + 32, c);
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    v[i] = a[i];
    v[32 + i] = c[i];
  }
}

// ============================================================== forward
__global__ void __launch_bounds__(AT_THREADS, 1) attn_fwd_kernel(const __grid_constant__ AttnFwdParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint8_t* ptile = ring + ATF_RING;        // alpha bf16, the A operand of Eq. 3
  uint8_t* staging = ptile + AT_OPA;
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + 8 * AT_STG);
  uint64_t* full = bars;                   // [AT_MAXST]
  uint64_t* empty = full + AT_MAXST;       // [AT_MAXST]
  uint64_t* sfull = empty + AT_MAXST;      // scores complete in TMEM
  uint64_t* pfull = sfull + 1;             // alpha tile written (4 softmax warps)
  uint64_t* tfull = pfull + 1;             // [AT_SLOTS] context chunk accumulated
  uint64_t* tempty = tfull + AT_SLOTS;     // [AT_SLOTS] context chunk drained (8 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + AT_SLOTS);

  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();
  const int b = blockIdx.x;
  const int nkb = P.d / 64;
  const int nch = (nkb + 1) / 2;                      // context chunks of 128 columns
  const uint32_t sbytes = (uint32_t)P.mbox * 128;     // one S block [mbox, 64]
  const uint32_t qbytes = (uint32_t)P.qrows * 128;    // one Q block [qrows, 64]
  const uint32_t stage = max(qbytes + sbytes, 2 * sbytes);
  const int nst = min(AT_MAXST, (int)(ATF_RING / stage));

  if (warp == 8) {
    if (lane == 0) {
      for (int i = 0; i < AT_MAXST; ++i) {
        mbar_init(&full[i], 1);
        mbar_init(&empty[i], 1);
      }
      mbar_init(sfull, 1);
      mbar_init(pfull, 4);
      for (int i = 0; i < AT_SLOTS; ++i) {
        mbar_init(&tfull[i], 1);
        mbar_init(&tempty[i], 8);
      }
      fence_barrier_init();
      tma_prefetch_desc(&P.m_q);
      tma_prefetch_desc(&P.m_s);
      tma_prefetch_desc(&P.m_c);
    }
    __syncwarp();
    tmem_alloc(tmem_slot, 512);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();
  if (threadIdx.x == 0) pdl_trigger();
  if (warp == 8) AT_TRACE(0);

  if (warp == 8) {
    // ---------------- TMA producer: (Q, S) blocks over d, then S again per 128-column chunk
    int s = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      mbar_wait(&empty[s], ph ^ 1);
      if (elect_one()) {
        uint8_t* st = ring + s * stage;
        mbar_arrive_expect_tx(&full[s], qbytes + sbytes);
        tma_load_3d(st, &P.m_q, &full[s], kb * 64, 0, b);
        tma_load_3d(st + qbytes, &P.m_s, &full[s], kb * 64, 0, b);
      }
      __syncwarp();
      if (++s == nst) { s = 0; ph ^= 1; }
    }
    AT_TRACE(1);
    for (int j = 0; j < nch; ++j) {
      const int nb = min(2, nkb - 2 * j);
      mbar_wait(&empty[s], ph ^ 1);
      if (elect_one()) {
        uint8_t* st = ring + s * stage;
        mbar_arrive_expect_tx(&full[s], nb * sbytes);
        for (int i = 0; i < nb; ++i) tma_load_3d(st + i * sbytes, &P.m_s, &full[s], (2 * j + i) * 64, 0, b);
      }
      __syncwarp();
      if (++s == nst) { s = 0; ph ^= 1; }
    }
  } else if (warp == 9) {
    // ---------------- MMA issuer
    int s = 0;
    uint32_t ph = 0;
    const uint32_t idesc_s = umma_idesc_bf16(128, P.mbox, 0, 0);
    for (int kb = 0; kb < nkb; ++kb) {
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sa = smem_u32(ring + s * stage);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_bf16(tmem_base, umma_sdesc(sa + k * 32, 16, 1024),
                    umma_sdesc(sa + qbytes + k * 32, 16, 1024), idesc_s, (kb | k) ? 1u : 0u);
        umma_commit(&empty[s]);
      }
      __syncwarp();
      if (++s == nst) { s = 0; ph ^= 1; }
    }
    if (elect_one()) umma_commit(sfull);
    __syncwarp();
    AT_TRACE(2);
    // Eq. 3: C chunk j = alpha S[:, 128 j ..]: A = alpha (K-major, K = mbox), B = S (MN-major)
    mbar_wait(pfull, 0);
    tc_fence_after();
    const int ksteps = P.mbox / 16;
    const uint32_t pa = smem_u32(ptile);
    for (int j = 0; j < nch; ++j) {
      const int slot = j % AT_SLOTS, use = j / AT_SLOTS;
      if (use > 0) mbar_wait(&tempty[slot], (use - 1) & 1);
      mbar_wait(&full[s], ph);
      tc_fence_after();
      const int nb = min(2, nkb - 2 * j);
      const uint32_t idesc_c = umma_idesc_bf16(128, 64 * nb, 0, 1);
      if (elect_one()) {
        const uint32_t sb = smem_u32(ring + s * stage);
        for (int k = 0; k < ksteps; ++k)
          umma_bf16(tmem_base + slot * 128,
                    umma_sdesc(pa + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024),
                    umma_sdesc(sb + k * 2048, sbytes, 1024), idesc_c, k ? 1u : 0u);
        umma_commit(&empty[s]);
        umma_commit(&tfull[slot]);
      }
      __syncwarp();
      if (++s == nst) { s = 0; ph ^= 1; }
    }
    AT_TRACE(5);
  } else {
    // ---------------- softmax (warps 0-3) and context epilogue (warps 0-7)
    const uint32_t q = warp & 3, h = warp >> 2;
    uint8_t* stg = staging + warp * AT_STG;
    const int r = (int)(q * 32 + lane);                    // tile row = decoder step i
    int sb = 0;                                            // staging half of the next store
    if (h == 0) {
      const int L = P.src_len[b];
      const int nact = P.mbox / 32;
      const uint32_t taddr = tmem_base + ((q * 32u) << 16);
      mbar_wait(sfull, 0);
      tc_fence_after();
      if (warp == 0) AT_TRACE(3);
      // branch-free masked softmax: independent exponentials (MUFU ex2), four partial sums
      float v[32];
      float mx = -INFINITY;
      for (int c = 0; c < nact; ++c) {
        tmem_ld32(taddr + c * 32, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) mx = fmaxf(mx, (c * 32 + j < L) ? v[j] : -INFINITY);
      }
      if (warp == 0) AT_TRACE(8);
      const float nml = -mx * kLog2e;
      float s4[4] = {0.f, 0.f, 0.f, 0.f};
      for (int c = 0; c < nact; ++c) {
        tmem_ld32(taddr + c * 32, v);
#pragma unroll
        for (int j = 0; j < 32; ++j)
          s4[j & 3] += ex2_mufu((c * 32 + j < L) ? fmaf(v[j], kLog2e, nml) : -INFINITY);
      }
      const float inv = 1.f / ((s4[0] + s4[1]) + (s4[2] + s4[3]));
      if (warp == 0) AT_TRACE(9);
      const uint32_t pa = smem_u32(ptile);
      for (int c = 0; c < nact; ++c) {
        tmem_ld32(taddr + c * 32, v);
#pragma unroll
        for (int j = 0; j < 32; ++j)
          v[j] = ex2_mufu((c * 32 + j < L) ? fmaf(v[j], kLog2e, nml) : -INFINITY) * inv;
        at_put_row32(pa, r, c, v);
        if (warp == 0 && c == 0) AT_TRACE(10);
        if (c == nact - 1) {
          // every score read: TMEM columns 0..127 become context slot 0, and
          // the alpha tile is visible to the tensor cores
          tc_fence_before();
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(pfull);
          if (warp == 0) AT_TRACE(4);
        }
        // alpha leaves through TMA: fp32 stash (+ the bf16 copy for the generic backward)
        uint8_t* half = stg + sb * 4096;
        if (lane == 0) bulk_wait_read1();
        __syncwarp();
        const uint32_t hs = smem_u32(half);
#pragma unroll
        for (int g = 0; g < 8; ++g)
          st_shared_v4(hs + lane * 128 + ((g ^ (lane & 7)) << 4), __float_as_uint(v[4 * g]),
                       __float_as_uint(v[4 * g + 1]), __float_as_uint(v[4 * g + 2]),
                       __float_as_uint(v[4 * g + 3]));
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&P.m_stash, half, c * 32, q * 32, b);
          bulk_commit();
        }
        sb ^= 1;
        if (warp == 0) AT_TRACE(11 + c);
        if (P.store_abf) {
          stage_store_bf16(stg + sb * 4096, &P.m_abf, v, c * 32, q * 32, b, lane);
          sb ^= 1;
        }
      }
    }
    for (int j = 0; j < nch; ++j) {
      const int slot = j % AT_SLOTS, use = j / AT_SLOTS;
      const int ncol = min(128, P.d - j * 128);
      mbar_wait(&tfull[slot], use & 1);
      tc_fence_after();
      float v[64];
      if ((int)h * 64 < ncol) at_ld64(tmem_base + ((q * 32u) << 16) + slot * 128 + h * 64, v);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[slot]);
      if ((int)h * 64 < ncol) {
        at_store64_bf16(stg, sb, &P.m_c, v, j * 128 + h * 64, q * 32, b, lane);
        sb ^= 1;
      }
    }
    if (lane == 0) bulk_wait0();
    if (warp == 0) AT_TRACE(6);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 8) {
    tmem_dealloc(tmem_base, 512);
    if (P.trace && lane == 0) P.trace[(long long)blockIdx.x * 16 + 7] = smid();
  }
}

// ============================================================== backward
__global__ void __launch_bounds__(AT_THREADS, 1) attn_bwd_kernel(const __grid_constant__ AttnBwdParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  // one byte ring: phase-1 stages (dC block, S block) and, once every phase-1
  // MMA has completed, phase-2 stages (S, dC and Q blocks of one 64-column chunk)
  uint8_t* ring = smem;
  uint8_t* atile = ring + ATB_RING;        // alpha bf16 [i][j]
  uint8_t* dtile = atile + AT_OPA;         // de bf16 [i][j]
  uint8_t* staging = dtile + AT_OPA;
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + 8 * AT_STG);
  uint64_t* full1 = bars;                  // [AT_MAXST]
  uint64_t* empty1 = full1 + AT_MAXST;     // [AT_MAXST]
  uint64_t* full2 = empty1 + AT_MAXST;     // [AT_MAXST]
  uint64_t* empty2 = full2 + AT_MAXST;     // [AT_MAXST]
  uint64_t* sfull = empty2 + AT_MAXST;     // dalpha complete (also: phase-1 operands consumed)
  uint64_t* pfull = sfull + 1;             // alpha / de tiles written (4 warps)
  uint64_t* tfull = pfull + 1;             // [AT_SLOTS]
  uint64_t* tempty = tfull + AT_SLOTS;     // [AT_SLOTS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + AT_SLOTS);

  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();
  const int b = blockIdx.x;
  const int nkb = P.d / 64;
  const uint32_t sbytes = (uint32_t)P.mbox * 128;
  const uint32_t qbytes = (uint32_t)P.qrows * 128;
  const uint32_t st1 = qbytes + sbytes, st2 = sbytes + 2 * qbytes;
  const int n1 = min(AT_MAXST, (int)(ATB_RING / st1)), n2 = min(AT_MAXST, (int)(ATB_RING / st2));

  if (warp == 8) {
    if (lane == 0) {
      for (int i = 0; i < AT_MAXST; ++i) {
        mbar_init(&full1[i], 1);
        mbar_init(&empty1[i], 1);
        mbar_init(&full2[i], 1);
        mbar_init(&empty2[i], 1);
      }
      mbar_init(sfull, 1);
      mbar_init(pfull, 4);
      for (int i = 0; i < AT_SLOTS; ++i) {
        mbar_init(&tfull[i], 1);
        mbar_init(&tempty[i], 8);
      }
      fence_barrier_init();
      tma_prefetch_desc(&P.m_dc);
      tma_prefetch_desc(&P.m_s);
      tma_prefetch_desc(&P.m_q);
    }
    __syncwarp();
    tmem_alloc(tmem_slot, 512);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();
  if (threadIdx.x == 0) pdl_trigger();
  if (warp == 8) AT_TRACE(0);
  if (warp < 4) {
    // the idle softmax warps, during phase 1: this sentence's alpha rows
    // (fp32 stash) into the staging area, [128 rows][128 columns] with the
    // 16-byte chunks of row r XOR-swizzled by r (conflict-free)
    const int r = (int)(warp * 32 + lane);
    if (r < P.N) {
      const float* arow = P.alpha + ((long long)b * P.N + r) * P.ald;
      const uint32_t dst = smem_u32(staging) + r * 512;
      for (int k = 0; k < P.mbox / 4; ++k)
        cp_async16(dst + ((k ^ (r & 31)) << 4), arow + 4 * k);
    }
  }

  if (warp == 8) {
    // ---------------- TMA producer
    int s = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      mbar_wait(&empty1[s], ph ^ 1);
      if (elect_one()) {
        uint8_t* st = ring + s * st1;
        mbar_arrive_expect_tx(&full1[s], st1);
        tma_load_3d(st, &P.m_dc, &full1[s], kb * 64, 0, b);
        tma_load_3d(st + qbytes, &P.m_s, &full1[s], kb * 64, 0, b);
      }
      __syncwarp();
      if (++s == n1) { s = 0; ph ^= 1; }
    }
    AT_TRACE(1);
    // phase 2 reuses the ring's bytes once every phase-1 MMA has completed
    mbar_wait(sfull, 0);
    s = 0;
    ph = 0;
    for (int j = 0; j < nkb; ++j) {
      mbar_wait(&empty2[s], ph ^ 1);
      if (elect_one()) {
        uint8_t* st = ring + s * st2;
        mbar_arrive_expect_tx(&full2[s], st2);
        tma_load_3d(st, &P.m_s, &full2[s], j * 64, 0, b);
        tma_load_3d(st + sbytes, &P.m_dc, &full2[s], j * 64, 0, b);
        tma_load_3d(st + sbytes + qbytes, &P.m_q, &full2[s], j * 64, 0, b);
      }
      __syncwarp();
      if (++s == n2) { s = 0; ph ^= 1; }
    }
  } else if (warp == 9) {
    // ---------------- MMA issuer
    int s = 0;
    uint32_t ph = 0;
    const uint32_t idesc_s = umma_idesc_bf16(128, P.mbox, 0, 0);
    for (int kb = 0; kb < nkb; ++kb) {
      mbar_wait(&full1[s], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sa = smem_u32(ring + s * st1);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_bf16(tmem_base, umma_sdesc(sa + k * 32, 16, 1024),
                    umma_sdesc(sa + qbytes + k * 32, 16, 1024), idesc_s, (kb | k) ? 1u : 0u);
        umma_commit(&empty1[s]);
      }
      __syncwarp();
      if (++s == n1) { s = 0; ph ^= 1; }
    }
    if (elect_one()) umma_commit(sfull);
    __syncwarp();
    AT_TRACE(2);
    mbar_wait(pfull, 0);
    tc_fence_after();
    const uint32_t at = smem_u32(atile), dt = smem_u32(dtile);
    const uint32_t idesc_dh = umma_idesc_bf16(128, 64, 0, 1);    // de (K-major) x S (MN-major)
    const uint32_t idesc_de = umma_idesc_bf16(128, 64, 1, 1);    // alpha^T, de^T (MN-major) x dC, Q (MN-major)
    const int ks_dh = P.mbox / 16, ks_de = P.qrows / 16;
    s = 0;
    ph = 0;
    for (int j = 0; j < nkb; ++j) {
      const int slot = j % AT_SLOTS, use = j / AT_SLOTS;
      if (use > 0) mbar_wait(&tempty[slot], (use - 1) & 1);
      AT_TRACE2(j, 0);
      mbar_wait(&full2[s], ph);
      tc_fence_after();
      AT_TRACE2(j, 1);
      if (elect_one()) {
        const uint32_t sb = smem_u32(ring + s * st2);
        const uint32_t acc = tmem_base + slot * 128;
        // dQ chunk = de S[:, chunk]   (K = source positions)
        for (int k = 0; k < ks_dh; ++k)
          umma_bf16(acc, umma_sdesc(dt + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024),
                    umma_sdesc(sb + k * 2048, 16, 1024), idesc_dh, k ? 1u : 0u);
        // dH_enc chunk = alpha^T dC[:, chunk] + de^T Q[:, chunk]   (K = decoder rows, 2 segments)
        for (int k = 0; k < ks_de; ++k)
          umma_bf16(acc + 64, umma_sdesc(at + k * 2048, 16384, 1024),
                    umma_sdesc(sb + sbytes + k * 2048, 16, 1024), idesc_de, k ? 1u : 0u);
        for (int k = 0; k < ks_de; ++k)
          umma_bf16(acc + 64, umma_sdesc(dt + k * 2048, 16384, 1024),
                    umma_sdesc(sb + sbytes + qbytes + k * 2048, 16, 1024), idesc_de, 1u);
        umma_commit(&empty2[s]);
        umma_commit(&tfull[slot]);
      }
      __syncwarp();
      if (++s == n2) { s = 0; ph ^= 1; }
    }
    AT_TRACE(5);
  } else {
    // ---------------- softmax backward (warps 0-3), then the epilogue (warps 0-7)
    const uint32_t q = warp & 3, h = warp >> 2;
    uint8_t* stg = staging + warp * AT_STG;
    const int r = (int)(q * 32 + lane);
    if (h == 0) {
      const bool row_ok = r < P.N;
      const uint32_t taddr = tmem_base + ((q * 32u) << 16);
      const int nact = P.mbox / 32;
      const uint32_t arow = smem_u32(staging) + r * 512;
      // alpha chunk c of this row from the staging copy (0 past M, past mbox
      // and on rows past the sentence: the stash is not written there)
      auto load_alpha = [&](int c, float (&a)[32]) {
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
          if (row_ok && c < nact) x = ld_shared_f4(arow + (((c * 8 + g) ^ (r & 31)) << 4));
          a[4 * g] = x.x; a[4 * g + 1] = x.y; a[4 * g + 2] = x.z; a[4 * g + 3] = x.w;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c * 32 + j >= P.M) a[j] = 0.f;
      };
      cp_async_wait_all();
      mbar_wait(sfull, 0);
      tc_fence_after();
      if (warp == 0) AT_TRACE(3);
      const uint32_t at = smem_u32(atile), dt = smem_u32(dtile);
      float v[32], a[32];
      float D4[4] = {0.f, 0.f, 0.f, 0.f};
      for (int c = 0; c < 4; ++c) {   // all 128 columns: the tiles' unused atom holds zeros
        load_alpha(c, a);
        if (c < nact) {
          tmem_ld32(taddr + c * 32, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) D4[j & 3] = fmaf(a[j], v[j], D4[j & 3]);
        }
        at_put_row32(at, r, c, a);
      }
      const float D = row_ok ? (D4[0] + D4[1]) + (D4[2] + D4[3]) : 0.f;
      if (warp == 0) AT_TRACE(8);
      for (int c = 0; c < 4; ++c) {
        load_alpha(c, a);
        if (c < nact) tmem_ld32(taddr + c * 32, v);
        // rows past the sentence (stale A rows) and columns past mbox: de = 0
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = (c < nact && row_ok) ? a[j] * (v[j] - D) : 0.f;
        at_put_row32(dt, r, c, v);
      }
      if (warp == 0) AT_TRACE(9);
      tc_fence_before();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(pfull);
      if (warp == 0) AT_TRACE(4);
    }
    // the staging area held the alpha rows until here: every epilogue warp
    // passes this barrier before writing its staging half (the tfull chain
    // already orders it; the barrier makes the order explicit)
    named_bar_sync(2, 256);
    int sb = 0;
    for (int j = 0; j < nkb; ++j) {
      const int slot = j % AT_SLOTS, use = j / AT_SLOTS;
      float v[64];
      mbar_wait(&tfull[slot], use & 1);
      tc_fence_after();
      if (warp == 0 || warp == 4) AT_TRACE2(j, warp == 0 ? 2 : 3);
      at_ld64(tmem_base + ((q * 32u) << 16) + slot * 128 + h * 64, v);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[slot]);
      at_store64_bf16(stg, sb, h == 0 ? &P.m_dq : &P.m_dhe, v, j * 64, q * 32, b, lane);
      sb ^= 1;
    }
    if (lane == 0) bulk_wait0();
    if (warp == 0) AT_TRACE(6);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 8) {
    tmem_dealloc(tmem_base, 512);
    if (P.trace && lane == 0) P.trace[(long long)blockIdx.x * 16 + 7] = smid();
  }
}

}  // namespace attnsm
