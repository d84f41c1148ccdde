// attn_tc.cuh -- the attention steps of the stage as one tcgen05 kernel per
// direction, ONE CTA PER SENTENCE (bf16 path, N <= 128 decoder rows, M <= 128
// source positions):
//
//   attn_fwd_kernel   F1 + Eq. 1 + F2 (Eqs. 1-3):
//       E = Q S^T (K = d streamed through a TMA ring, fp32 in TMEM), the
//       length-masked row softmax in registers (alpha = 0 exactly for
//       j >= src_len), alpha written once (fp32 stash for the backward, bf16
//       copy) and kept in shared memory as the bf16 A operand of the context
//       MMA C = alpha S, S streamed a second time (L2) as the MN-major B.
//   attn_bwd_kernel   B3 (the backward of Eqs. 1-3):
//       dalpha = dC S^T (TMEM), de = alpha (dalpha - sum_j alpha dalpha) in
//       registers -> bf16 in shared memory; then per 64-column chunk of d
//       dH_dec = dH_part + de S and dH_enc = alpha^T dC + de^T Q (two K
//       segments), S / dC / Q streamed by TMA, fp32 accumulators in TMEM.
//
// Replaces the two (forward) and two (backward) batched launches of the
// generic engine, in which each sentence's 50 rows took a 128-row tile in a
// separate score and context GEMM and alpha / de made an HBM round trip
// between them.
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
// Roles (320 threads): warps 0-7 softmax / epilogue (warp w: TMEM lanes
// 32 (w % 4).., column half w / 4), warp 8 TMA producer + TMEM allocator,
// warp 9 MMA issuer (one elected lane).
#pragma once
#include "gemm_tc.cuh"

namespace attnsm {

constexpr int AT_THREADS = 320;
constexpr int AT_STG = 4096;                          // staging per epilogue warp
constexpr int AT_SLOTS = 4;                           // TMEM: 4 x 128 fp32 columns
constexpr int AT_OPA = 32 * 1024;                     // one bf16 [128 x 128] A tile (2 atoms)

// forward: 4 x 32 KB stages (Q block 16 KB + S block <= 16 KB; or two S blocks)
constexpr int ATF_STAGE = 32 * 1024;
constexpr int ATF_STAGES = 4;
constexpr int ATF_SMEM = ATF_STAGES * ATF_STAGE + AT_OPA + 8 * AT_STG + 1024 + 256;
// backward: a 96 KB ring, 3 x 32 KB stages in phase 1 (dC block 16 KB + S
// block) and 2 x 48 KB in phase 2 (S, dC and Q blocks of one 64-column chunk,
// 16 KB each), then the alpha and de tiles
constexpr int ATB_STAGE = 48 * 1024;
constexpr int ATB_STAGES = 2;
constexpr int ATB_SMEM = ATB_STAGES * ATB_STAGE + 2 * AT_OPA + 8 * AT_STG + 1024 + 256;

struct alignas(64) AttnFwdParams {
  CUtensorMap m_q;      // Q [B][N][d] bf16 (H_dec, or H W_alpha), box {64, 128, 1}
  CUtensorMap m_s;      // S = H_enc [B][M][d] bf16, box {64, mbox, 1}
  CUtensorMap m_c;      // C store [B][N][d] bf16, box {64, 32, 1}
  CUtensorMap m_stash;  // alpha fp32 [B][N][ald], dims {M, N, B}, box {32, 32, 1}
  CUtensorMap m_abf;    // alpha bf16 [B][N][Mp], dims {Mp, N, B}, box {32, 32, 1}, 64-byte swizzle
  const int* src_len;   // [B] (device)
  int d, mbox;          // mbox = M rounded up to 64 (UMMA N of the scores, K of the context)
};

struct alignas(64) AttnBwdParams {
  CUtensorMap m_dc;     // dC [B][N][d] bf16, box {64, 128, 1}
  CUtensorMap m_s;      // S [B][M][d] bf16, box {64, mbox, 1}
  CUtensorMap m_q;      // Q [B][N][d] bf16 (H_dec, or H W_alpha), box {64, 128, 1}
  CUtensorMap m_dh;     // dH_dec (dot score) or dQ (general score) store [B][N][d] bf16, box {64, 32, 1}
  CUtensorMap m_dhe;    // dH_enc store [B][M][d] bf16, box {64, 32, 1}
  const float* alpha;   // fp32 stash [B*N][ald]
  const float* dh_part; // dot score: dH_part fp32 [B*N][d] added to dH_dec; NULL: store dQ
  int N, M, d, ald, mbox;
};

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

// 32 rows x 64 bf16 columns of this warp through its 4 KB staging buffer
// (128-byte swizzle) to a {64, 32, 1} TMA box at (col, row0, b)
__device__ __forceinline__ void at_store64_bf16(uint8_t* stg, const CUtensorMap* m, const float (&v)[64],
                                                int col, int row0, int b, uint32_t lane) {
  const uint32_t s = smem_u32(stg);
  if (lane == 0) bulk_wait_read0();
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
    tma_store_3d(m, stg, col, row0, b);
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
  uint8_t* ptile = ring + ATF_STAGES * ATF_STAGE;    // alpha bf16, the A operand of Eq. 3
  uint8_t* staging = ptile + AT_OPA;
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + 8 * AT_STG);
  uint64_t* full = bars;                   // [ATF_STAGES]
  uint64_t* empty = full + ATF_STAGES;     // [ATF_STAGES]
  uint64_t* sfull = empty + ATF_STAGES;    // scores complete in TMEM
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

  if (warp == 8) {
    if (lane == 0) {
      for (int i = 0; i < ATF_STAGES; ++i) {
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

  if (warp == 8) {
    // ---------------- TMA producer: (Q, S) blocks over d, then S again per 128-column chunk
    int s = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      mbar_wait(&empty[s], ph ^ 1);
      if (elect_one()) {
        uint8_t* st = ring + s * ATF_STAGE;
        mbar_arrive_expect_tx(&full[s], 16384 + sbytes);
        tma_load_3d(st, &P.m_q, &full[s], kb * 64, 0, b);
        tma_load_3d(st + 16384, &P.m_s, &full[s], kb * 64, 0, b);
      }
      __syncwarp();
      if (++s == ATF_STAGES) { s = 0; ph ^= 1; }
    }
    for (int j = 0; j < nch; ++j) {
      const int nb = min(2, nkb - 2 * j);
      mbar_wait(&empty[s], ph ^ 1);
      if (elect_one()) {
        uint8_t* st = ring + s * ATF_STAGE;
        mbar_arrive_expect_tx(&full[s], nb * sbytes);
        for (int i = 0; i < nb; ++i) tma_load_3d(st + i * sbytes, &P.m_s, &full[s], (2 * j + i) * 64, 0, b);
      }
      __syncwarp();
      if (++s == ATF_STAGES) { s = 0; ph ^= 1; }
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
        const uint32_t sa = smem_u32(ring + s * ATF_STAGE);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_bf16(tmem_base, umma_sdesc(sa + k * 32, 16, 1024),
                    umma_sdesc(sa + 16384 + k * 32, 16, 1024), idesc_s, (kb | k) ? 1u : 0u);
        umma_commit(&empty[s]);
      }
      __syncwarp();
      if (++s == ATF_STAGES) { s = 0; ph ^= 1; }
    }
    if (elect_one()) umma_commit(sfull);
    __syncwarp();
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
        const uint32_t sb = smem_u32(ring + s * ATF_STAGE);
        for (int k = 0; k < ksteps; ++k)
          umma_bf16(tmem_base + slot * 128,
                    umma_sdesc(pa + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024),
                    umma_sdesc(sb + k * 2048, sbytes, 1024), idesc_c, k ? 1u : 0u);
        umma_commit(&empty[s]);
        umma_commit(&tfull[slot]);
      }
      __syncwarp();
      if (++s == ATF_STAGES) { s = 0; ph ^= 1; }
    }
  } else {
    // ---------------- softmax (warps 0-3) and context epilogue (warps 0-7)
    const uint32_t q = warp & 3, h = warp >> 2;
    uint8_t* stg = staging + warp * AT_STG;
    const int r = (int)(q * 32 + lane);                    // tile row = decoder step i
    if (h == 0) {
      const int L = P.src_len[b];
      const int nact = P.mbox / 32;
      const uint32_t taddr = tmem_base + ((q * 32u) << 16);
      mbar_wait(sfull, 0);
      tc_fence_after();
      float v[32];
      float mx = -INFINITY;
      for (int c = 0; c < nact; ++c) {
        tmem_ld32(taddr + c * 32, v);
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c * 32 + j < L) mx = fmaxf(mx, v[j]);
      }
      float sum = 0.f;
      for (int c = 0; c < nact; ++c) {
        tmem_ld32(taddr + c * 32, v);
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c * 32 + j < L) sum += __expf(v[j] - mx);
      }
      const float inv = 1.f / sum;
      const uint32_t pa = smem_u32(ptile);
      for (int c = 0; c < nact; ++c) {
        tmem_ld32(taddr + c * 32, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = (c * 32 + j < L) ? __expf(v[j] - mx) * inv : 0.f;
        at_put_row32(pa, r, c, v);
        stage_store_f32(stg, &P.m_stash, v, c * 32, q * 32, b, lane);
        stage_store_bf16(stg, &P.m_abf, v, c * 32, q * 32, b, lane);
      }
      // the scores are consumed (TMEM columns 0..127 become context slot 0)
      // and the alpha tile is visible to the tensor cores
      tc_fence_before();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(pfull);
    }
    for (int j = 0; j < nch; ++j) {
      const int slot = j % AT_SLOTS, use = j / AT_SLOTS;
      const int ncol = min(128, P.d - j * 128);
      mbar_wait(&tfull[slot], use & 1);
      tc_fence_after();
      if ((int)h * 64 < ncol) {
        float v[64];
        at_ld64(tmem_base + ((q * 32u) << 16) + slot * 128 + h * 64, v);
        at_store64_bf16(stg, &P.m_c, v, j * 128 + h * 64, q * 32, b, lane);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[slot]);
    }
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 8) tmem_dealloc(tmem_base, 512);
}

// ============================================================== backward
__global__ void __launch_bounds__(AT_THREADS, 1) attn_bwd_kernel(const __grid_constant__ AttnBwdParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  // one 96 KB byte ring: phase 1 as 3 x 32 KB stages (dC block, S block),
  // phase 2 as 2 x 48 KB stages (S, dC, Q blocks of one 64-column chunk)
  uint8_t* ring = smem;
  uint8_t* atile = ring + ATB_STAGES * ATB_STAGE;    // alpha bf16 [i][j]
  uint8_t* dtile = atile + AT_OPA;                   // de bf16 [i][j]
  uint8_t* staging = dtile + AT_OPA;
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + 8 * AT_STG);
  uint64_t* full1 = bars;                  // [3]
  uint64_t* empty1 = full1 + 3;            // [3]
  uint64_t* full2 = empty1 + 3;            // [2]
  uint64_t* empty2 = full2 + 2;            // [2]
  uint64_t* sfull = empty2 + 2;            // dalpha complete (also: phase-1 operands consumed)
  uint64_t* pfull = sfull + 1;             // alpha / de tiles written (4 warps)
  uint64_t* tfull = pfull + 1;             // [AT_SLOTS]
  uint64_t* tempty = tfull + AT_SLOTS;     // [AT_SLOTS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + AT_SLOTS);

  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();
  const int b = blockIdx.x;
  const int nkb = P.d / 64;
  const uint32_t sbytes = (uint32_t)P.mbox * 128;

  if (warp == 8) {
    if (lane == 0) {
      for (int i = 0; i < 3; ++i) {
        mbar_init(&full1[i], 1);
        mbar_init(&empty1[i], 1);
      }
      for (int i = 0; i < 2; ++i) {
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

  if (warp == 8) {
    // ---------------- TMA producer
    int s = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      mbar_wait(&empty1[s], ph ^ 1);
      if (elect_one()) {
        uint8_t* st = ring + s * 32768;
        mbar_arrive_expect_tx(&full1[s], 16384 + sbytes);
        tma_load_3d(st, &P.m_dc, &full1[s], kb * 64, 0, b);
        tma_load_3d(st + 16384, &P.m_s, &full1[s], kb * 64, 0, b);
      }
      __syncwarp();
      if (++s == 3) { s = 0; ph ^= 1; }
    }
    // phase 2 reuses the ring's bytes once every phase-1 MMA has completed
    mbar_wait(sfull, 0);
    s = 0;
    ph = 0;
    for (int j = 0; j < nkb; ++j) {
      mbar_wait(&empty2[s], ph ^ 1);
      if (elect_one()) {
        uint8_t* st = ring + s * ATB_STAGE;
        mbar_arrive_expect_tx(&full2[s], sbytes + 32768);
        tma_load_3d(st, &P.m_s, &full2[s], j * 64, 0, b);
        tma_load_3d(st + 16384, &P.m_dc, &full2[s], j * 64, 0, b);
        tma_load_3d(st + 32768, &P.m_q, &full2[s], j * 64, 0, b);
      }
      __syncwarp();
      if (++s == 2) { s = 0; ph ^= 1; }
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
        const uint32_t sa = smem_u32(ring + s * 32768);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_bf16(tmem_base, umma_sdesc(sa + k * 32, 16, 1024),
                    umma_sdesc(sa + 16384 + k * 32, 16, 1024), idesc_s, (kb | k) ? 1u : 0u);
        umma_commit(&empty1[s]);
      }
      __syncwarp();
      if (++s == 3) { s = 0; ph ^= 1; }
    }
    if (elect_one()) umma_commit(sfull);
    __syncwarp();
    mbar_wait(pfull, 0);
    tc_fence_after();
    const uint32_t at = smem_u32(atile), dt = smem_u32(dtile);
    const uint32_t idesc_dh = umma_idesc_bf16(128, 64, 0, 1);    // de (K-major) x S (MN-major)
    const uint32_t idesc_de = umma_idesc_bf16(128, 64, 1, 1);    // alpha^T, de^T (MN-major) x dC, Q (MN-major)
    const int ks_dh = P.mbox / 16;
    s = 0;
    ph = 0;
    for (int j = 0; j < nkb; ++j) {
      const int slot = j % AT_SLOTS, use = j / AT_SLOTS;
      if (use > 0) mbar_wait(&tempty[slot], (use - 1) & 1);
      mbar_wait(&full2[s], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sb = smem_u32(ring + s * ATB_STAGE);
        const uint32_t acc = tmem_base + slot * 128;
        // dH_dec (or dQ) chunk = de S[:, chunk]   (K = source positions)
        for (int k = 0; k < ks_dh; ++k)
          umma_bf16(acc, umma_sdesc(dt + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024),
                    umma_sdesc(sb + k * 2048, 16, 1024), idesc_dh, k ? 1u : 0u);
        // dH_enc chunk = alpha^T dC[:, chunk] + de^T Q[:, chunk]   (K = decoder rows, 2 segments)
#pragma unroll 1
        for (int k = 0; k < 8; ++k)
          umma_bf16(acc + 64, umma_sdesc(at + k * 2048, 16384, 1024),
                    umma_sdesc(sb + 16384 + k * 2048, 16, 1024), idesc_de, k ? 1u : 0u);
#pragma unroll 1
        for (int k = 0; k < 8; ++k)
          umma_bf16(acc + 64, umma_sdesc(dt + k * 2048, 16384, 1024),
                    umma_sdesc(sb + 32768 + k * 2048, 16, 1024), idesc_de, 1u);
        umma_commit(&empty2[s]);
        umma_commit(&tfull[slot]);
      }
      __syncwarp();
      if (++s == 2) { s = 0; ph ^= 1; }
    }
  } else {
    // ---------------- softmax backward (warps 0-3), then the epilogue (warps 0-7)
    const uint32_t q = warp & 3, h = warp >> 2;
    uint8_t* stg = staging + warp * AT_STG;
    const int r = (int)(q * 32 + lane);
    if (h == 0) {
      const bool row_ok = r < P.N;
      const float* arow = P.alpha + ((long long)b * P.N + (row_ok ? r : 0)) * P.ald;
      const uint32_t taddr = tmem_base + ((q * 32u) << 16);
      const int nact = P.mbox / 32;
      auto load_alpha = [&](int c, float (&a)[32]) {
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
          if (row_ok && c < nact) x = __ldg(reinterpret_cast<const float4*>(arow + c * 32) + g);
          a[4 * g] = x.x; a[4 * g + 1] = x.y; a[4 * g + 2] = x.z; a[4 * g + 3] = x.w;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c * 32 + j >= P.M) a[j] = 0.f;   // (stash columns past M are not written)
      };
      mbar_wait(sfull, 0);
      tc_fence_after();
      const uint32_t at = smem_u32(atile), dt = smem_u32(dtile);
      float v[32], a[32];
      float D = 0.f;
      for (int c = 0; c < 4; ++c) {   // all 128 columns: the tiles' unused atom holds zeros
        load_alpha(c, a);
        if (c < nact) {
          tmem_ld32(taddr + c * 32, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) D += a[j] * v[j];
        }
        at_put_row32(at, r, c, a);
      }
      for (int c = 0; c < 4; ++c) {
        load_alpha(c, a);
        if (c < nact) {
          tmem_ld32(taddr + c * 32, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = a[j] * (v[j] - D);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.f;
        }
        at_put_row32(dt, r, c, v);
      }
      tc_fence_before();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(pfull);
    }
    const bool add = P.dh_part != nullptr && h == 0 && r < P.N;
    const float* prow = add ? P.dh_part + ((long long)b * P.N + r) * P.d : nullptr;
    for (int j = 0; j < nkb; ++j) {
      const int slot = j % AT_SLOTS, use = j / AT_SLOTS;
      float v[64];
      float4 ad[16];
      if (add) {
#pragma unroll
        for (int g = 0; g < 16; ++g) ad[g] = __ldg(reinterpret_cast<const float4*>(prow + j * 64) + g);
      }
      mbar_wait(&tfull[slot], use & 1);
      tc_fence_after();
      at_ld64(tmem_base + ((q * 32u) << 16) + slot * 128 + h * 64, v);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[slot]);
      if (add) {
#pragma unroll
        for (int g = 0; g < 16; ++g) {
          v[4 * g] += ad[g].x; v[4 * g + 1] += ad[g].y; v[4 * g + 2] += ad[g].z; v[4 * g + 3] += ad[g].w;
        }
      }
      at_store64_bf16(stg, h == 0 ? &P.m_dh : &P.m_dhe, v, j * 64, q * 32, b, lane);
    }
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 8) tmem_dealloc(tmem_base, 512);
}

}  // namespace attnsm
