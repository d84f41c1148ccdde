// gemm_tc.cuh -- persistent, warp-specialised tcgen05 GEMM engine (sm_100a).
//
//   D[M,N] (fp32, in TMEM) = A[M,K] * B[N,K]^T,  bf16 operands staged by TMA
//   (128-byte swizzle) into a 4-stage shared-memory ring; the epilogue reads
//   the accumulator with tcgen05.ld and runs one of the epilogues below.
//   One launch runs a GROUP of up to kMaxProblems independent problems (e.g.
//   the V-chunk c dW_out and dHc GEMMs together with the chunk c+1 dlogits
//   GEMM); CTAs pull tiles from a global atomic counter so long-K and
//   short-K tiles balance across the 148 SMs.  A problem may be BATCHED (one
//   small GEMM per sentence: the attention steps), in which case every
//   tensor map carries the sentence as its outermost coordinate and rows past
//   a sentence's extent are zero-filled (loads) or clipped (stores) by TMA.
//
// Roles (384 threads, one CTA per SM).  The warp scheduler of an SM
// sub-partition issues the highest eligible warp id first, so the two
// latency-critical roles get the highest ids:
//   warps 0..7   epilogue: warp w reads TMEM lanes 32*(w%4)..+31 (tile rows)
//                and column half w/4; results are staged in shared memory
//                (128-byte swizzle, conflict-free) and written with TMA bulk
//                stores, or TMA reduce-adds for accumulation
//   warp 8       TMEM allocator (512 columns = two 128x256 fp32 accumulators)
//   warp 10      tile scheduler + TMA producer (one elected lane issues)
//   warp 11      MMA issuer (one elected lane issues tcgen05.mma for the CTA)
//
// Operand tiles:
//   mode 0  K-major  [rows, K]: one 3D box {64 (K), rows, 1 (batch)}
//   mode 1  MN-major [K, MN]:   one 4D box {64, 64 (K), rows/64 (atoms), 1}
//   mode 2  MN-major [K, MN]:   one 3D box {64, 64, 1} per 64-wide atom
// A K range may be split into two SEGMENTS (k-blocks < kseg read maps 0, the
// rest read maps 1 from K = 0 again): [H | C] of Eq. 4, and the two terms of
// the attention backward dH_enc = alpha^T dC + de^T H.
#pragma once
#include "epilogue.cuh"
#include "ptx.cuh"

namespace attnsm {

constexpr int TC_BM = 128;    // accumulator rows per CTA (TMEM lanes)
constexpr int TC_BN = 256;    // tile columns
constexpr int TC_BK = 64;
constexpr int TC_THREADS = 384;
constexpr int TC_EPI_WARPS = 8;
constexpr int TC_STG_BYTES = 4096;                        // per epilogue warp
constexpr int TC_A_BYTES = TC_BM * TC_BK * 2;             // 16 KB
constexpr int TC_RING_BYTES = 192 * 1024;                 // operand ring
constexpr int TC_SCHED = 4;
constexpr int TC_SMEM_BYTES =
    TC_RING_BYTES + TC_EPI_WARPS * TC_STG_BYTES + 1024 /*align*/ + 512 /*barriers*/;
constexpr int kMaxProblems = 4;

// kPair = 1: one CTA computes a 128 x 256 tile (tcgen05 cta_group::1).
// kPair = 2: a CTA pair (cluster of 2 on one TPC) computes a 256 x 256 tile
//            with cta_group::2: each CTA stages its 128 rows of A and 128 rows
//            of B (32 KB stages, 6 of them); the MMA reads the peer's B half.
// kPair = 3: a cluster of 2 CTAs computes two vertically adjacent 128 x 256
//            tiles that share the B tile: each CTA loads half of B and TMA-
//            multicasts it to both, so both MMAs (cta_group::1) read local
//            shared memory while the L2 -> SM operand traffic per FLOP drops
//            by a third (48 KB stages, 4 of them).
// kPair = 4 ("wide"): one CTA computes a 256 x 256 tile as two M = 128 MMAs
//            per K step that share the B tile (accumulators in TMEM columns
//            0-255 and 256-511): twice the MMA work per staged byte of the
//            128 x 256 tile, at the price of one tile in TMEM at a time (the
//            epilogue is not overlapped with the next tile's MMAs).  64 KB
//            stages, 3 of them.
// kPair = 5 ("mixed"): wide 256 x 256 tiles and, for problems flagged
//            `narrow`, 128 x 256 tiles in the same launch.  The operand ring
//            is a byte ring of variable-size stages (64 KB wide, 48 KB narrow:
//            3 or 4 in flight) with 8 barrier slots, and the two 256-column
//            TMEM accumulator slots are handed out per 128-row half, so a
//            narrow tile's epilogue overlaps the next tile's MMAs.
// kPair = 6 ("wide multicast"): a cluster of 2 CTAs computes two vertically
//            adjacent 256 x 256 wide tiles that share the B tile (kPair 3's
//            multicast on kPair 4's tiles): each CTA loads its 256 A rows and
//            half of B, multicast into both; L2 -> SM operand bytes per FLOP
//            drop by a quarter against kPair 4 (48 of 64 KB per stage).
template <int kPair>
struct TcCfg {
  static constexpr bool WIDE = kPair == 4 || kPair == 5 || kPair == 6;
  static constexpr bool VAR = kPair == 5;
  static constexpr int TILE_M = kPair == 1 ? TC_BM : kPair == 6 ? 4 * TC_BM : 2 * TC_BM;   // rows per scheduled tile
  static constexpr int MMA_M = kPair == 2 ? 2 * TC_BM : TC_BM;     // UMMA M
  static constexpr int B_ROWS = (kPair == 2 || kPair == 3 || kPair == 6) ? TC_BN / 2 : TC_BN;   // B rows loaded per CTA
  static constexpr int A_SMEM = (WIDE ? 2 : 1) * TC_A_BYTES;
  static constexpr int B_SMEM = (kPair == 2 ? TC_BN / 2 : TC_BN) * TC_BK * 2;
  static constexpr int STAGE = A_SMEM + B_SMEM;                    // 48 | 32 | 48 | 64 | - | 64 KB
  static constexpr int CTA_ROWS = WIDE ? 2 * TC_BM : TC_BM;        // A rows per CTA of a cluster
  static constexpr int STAGES = VAR ? 8 : TC_RING_BYTES / STAGE;   // 4 | 6 | 4 | 3 | 8 slots
  static constexpr int CLUSTER = (kPair == 2 || kPair == 3 || kPair == 6) ? 2 : 1;
  static constexpr int ACCS = WIDE ? 1 : 2;                        // tiles resident in TMEM
};

struct TcProblem {
  int M, N, K;      // per batch item
  int batch;
  int tiles_m, tiles_n, kb_total;
  int tile_begin;
  int a_mn, b_mn;   // UMMA majorness
  int a_mode, b_mode;
  int kseg;         // k-blocks in segment 0 (0 = one segment)
  int b_seg;        // B switches to map b1 in segment 1 (else continues in b0)
  int b_nsplit;     // B column split between maps b0 / b1 (MN-major B, 0 = none)
  int b_koff;       // added to B's K coordinate (elements)
  int bn;           // tile columns (UMMA N): 256, or 16..240 for K-major B on single CTAs
  int narrow;       // kPair = 5: this problem uses 128 x 256 tiles
  int n_fast;       // dispatch order: column tiles fastest (tiles sharing an A row block adjacent)
  EpiParams epi;
};

struct alignas(64) TcParams {
  CUtensorMap maps[kMaxProblems][5];  // a0, a1, b0, b1, out
  TcProblem prob[kMaxProblems];
  int nprob;
  int total_tiles;
  int* tile_counter;
  long long* trace;   // debug: per-tile timestamps (null = off); 8 x int64 per tile
};

// trace record layout per tile t (clock64 of the SM that ran it):
//   [0] smid  [1] producer: first load issued  [2] producer: last load issued
//   [3] MMA: tile id seen  [4] MMA: first MMA issued  [5] MMA: last commit
//   [6] epilogue warp 4: accumulator ready (tfull)  [7] epilogue warp 4: done
__device__ __forceinline__ long long clk64() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
// stamp taken by every lane of a converged warp, stored by lane 2 (never lane
// 0, whose mbarrier arrives have release semantics and would wait for it)
#define TC_TRACE(t, i)                                                  \
  do {                                                                  \
    if (P.trace) {                                                      \
      const long long c_ = clk64();                                     \
      if (lane == 2) P.trace[(long long)(t) * 16 + (i)] = c_;           \
    }                                                                   \
  } while (0)
__device__ __forceinline__ long long gtime() {
  long long c;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(c));
  return c;
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ int tc_find_problem(const TcParams& P, int t) {
  int p = 0;
#pragma unroll
  for (int i = 1; i < kMaxProblems; ++i)
    if (i < P.nprob && t >= P.prob[i].tile_begin) p = i;
  return p;
}

struct TcTile {
  int p, b, m0, n0, tn;
  int nsub;   // 128-row accumulator halves: 2 for wide tiles, else 1
};

template <int kPair>
__device__ __forceinline__ TcTile tc_decode(const TcParams& P, int t) {
  TcTile r;
  r.p = tc_find_problem(P, t);
  const TcProblem& pr = P.prob[r.p];
  int local = t - pr.tile_begin;
  const int per_b = pr.tiles_m * pr.tiles_n;
  r.b = local / per_b;
  local -= r.b * per_b;
  const int tm = pr.n_fast ? local / pr.tiles_n : local % pr.tiles_m;
  r.tn = pr.n_fast ? local % pr.tiles_n : local / pr.tiles_m;
  r.nsub = (TcCfg<kPair>::WIDE && !(TcCfg<kPair>::VAR && pr.narrow)) ? 2 : 1;
  r.m0 = tm * (TcCfg<kPair>::VAR ? TC_BM * r.nsub : TcCfg<kPair>::TILE_M);
  r.n0 = r.tn * pr.bn;
  return r;
}

// TMA load issue: single CTA (local barrier) or pair (leader's barrier).
template <int kPair>
__device__ __forceinline__ void tl3(void* dst, const CUtensorMap* m, uint64_t* bar, uint32_t barc,
                                    int c0, int c1, int c2) {
  if constexpr (kPair == 2) tma_load_3d_pair(dst, m, barc, c0, c1, c2);
  else tma_load_3d(dst, m, bar, c0, c1, c2);
}
template <int kPair>
__device__ __forceinline__ void tl4(void* dst, const CUtensorMap* m, uint64_t* bar, uint32_t barc,
                                    int c0, int c1, int c2, int c3) {
  if constexpr (kPair == 2) tma_load_4d_pair(dst, m, barc, c0, c1, c2, c3);
  else tma_load_4d(dst, m, bar, c0, c1, c2, c3);
}
// multicast-to-both variants (kPair == 3, B operand)
__device__ __forceinline__ void tc_load_operand_mc(uint8_t* dst, const CUtensorMap* m, uint64_t* bar,
                                                   int mode, int rows, int r0, int k0, int b) {
  if (mode == 0) {
    tma_load_3d_mc(dst, m, bar, k0, r0, b, 3);
  } else if (mode == 1) {
    tma_load_4d_mc(dst, m, bar, 0, k0, r0 / 64, b, 3);
  } else {
    for (int i = 0; i < rows / 64; ++i) tma_load_3d_mc(dst + i * 8192, m, bar, r0 + 64 * i, k0, b, 3);
  }
}
// Load one operand tile (rows x 64 K) of k-block kb into smem.
template <int kPair>
__device__ __forceinline__ void tc_load_operand(uint8_t* dst, const CUtensorMap* m, uint64_t* bar,
                                                uint32_t barc, int mode, int rows, int r0, int k0,
                                                int b) {
  if (mode == 0) {
    tl3<kPair>(dst, m, bar, barc, k0, r0, b);
  } else if (mode == 1) {
    tl4<kPair>(dst, m, bar, barc, 0, k0, r0 / 64, b);
  } else {
    for (int i = 0; i < rows / 64; ++i) tl3<kPair>(dst + i * 8192, m, bar, barc, r0 + 64 * i, k0, b);
  }
}

// ---------------------------------------------------------------- attention epilogues
// Stage one 32-row x 32-column chunk of this warp's rows in its shared-memory
// staging buffer and TMA-store it (the previous store's smem read is waited
// for first).  fp32: 128-byte rows, 128-byte swizzle; bf16: 64-byte rows,
// 64-byte swizzle (the tensor map's box is {32, 32}).
__device__ __forceinline__ void stage_store_f32(uint8_t* stg, const CUtensorMap* m,
                                                const float (&v)[32], int col, int row0, int b,
                                                uint32_t lane) {
  const uint32_t s = smem_u32(stg);
  if (lane == 0) bulk_wait_read0();
  __syncwarp();
#pragma unroll
  for (int g = 0; g < 8; ++g)
    st_shared_v4(s + lane * 128 + ((g ^ (lane & 7)) << 4), __float_as_uint(v[4 * g]),
                 __float_as_uint(v[4 * g + 1]), __float_as_uint(v[4 * g + 2]),
                 __float_as_uint(v[4 * g + 3]));
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_store_3d(m, stg, col, row0, b);
    bulk_commit();
  }
}
__device__ __forceinline__ void stage_store_bf16(uint8_t* stg, const CUtensorMap* m,
                                                 const float (&v)[32], int col, int row0, int b,
                                                 uint32_t lane) {
  const uint32_t s = smem_u32(stg);
  if (lane == 0) bulk_wait_read0();
  __syncwarp();
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      __nv_bfloat162 h2 = __floats2bfloat162_rn(v[8 * g + 2 * e], v[8 * g + 2 * e + 1]);
      w[e] = *reinterpret_cast<uint32_t*>(&h2);
    }
    st_shared_v4(s + lane * 64 + ((g ^ ((lane >> 1) & 3)) << 4), w[0], w[1], w[2], w[3]);
  }
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_store_3d(m, stg, col, row0, b);
    bulk_commit();
  }
}

// Masked row softmax of the scores tile (Eq. 1): one thread per decoder row,
// M_src <= 128 columns (column half 0 only).  alpha (fp32 stash, row stride
// stash_ld, tensor map `mstash`) and its bf16 copy (row stride ldo = Mp, map
// `mbf`, the operand of Eq. 3 and of the backward) leave through TMA stores;
// both are exactly 0 for j >= src_len.
__device__ __forceinline__ void epi_attn_softmax(uint32_t taddr, int n_act, int L, uint8_t* stg,
                                                 const CUtensorMap* mstash, const CUtensorMap* mbf,
                                                 int row0, int b, uint32_t lane) {
  float v[32];
  float mx = -INFINITY;
  for (int c = 0; c < n_act; ++c) {
    tmem_ld32(taddr + c * 32, v);
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (c * 32 + j < L) mx = fmaxf(mx, v[j]);
  }
  float s = 0.f;
  for (int c = 0; c < n_act; ++c) {
    tmem_ld32(taddr + c * 32, v);
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (c * 32 + j < L) s += __expf(v[j] - mx);
  }
  const float inv = 1.f / s;
  for (int c = 0; c < n_act; ++c) {
    tmem_ld32(taddr + c * 32, v);
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = (c * 32 + j < L) ? __expf(v[j] - mx) * inv : 0.f;
    stage_store_f32(stg, mstash, v, c * 32, row0, b, lane);
    stage_store_bf16(stg, mbf, v, c * 32, row0, b, lane);
  }
}

// Backward of Eq. 1 on the dalpha tile: de = alpha (dalpha - sum_j alpha dalpha),
// written as bf16 (row stride ldo = Mp, map `mbf`), exactly 0 where alpha is.
__device__ __forceinline__ void epi_attn_softmax_bwd(const EpiParams& e, uint32_t taddr, int n_act,
                                                     int rowg, bool row_ok, uint8_t* stg,
                                                     const CUtensorMap* mbf, int row0, int b,
                                                     uint32_t lane) {
  float v[32];
  const float* af = e.stash_f32 + (long long)rowg * e.stash_ld;
  auto load_alpha = [&](int c, float (&a)[32]) {
    if (row_ok) {
      const float4* a4 = reinterpret_cast<const float4*>(af + c * 32);
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const float4 x = a4[g];
        a[4 * g] = x.x; a[4 * g + 1] = x.y; a[4 * g + 2] = x.z; a[4 * g + 3] = x.w;
      }
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (c * 32 + j >= e.ncols_valid) a[j] = 0.f;
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) a[j] = 0.f;
    }
  };
  float D = 0.f;
  for (int c = 0; c < n_act; ++c) {
    float a[32];
    tmem_ld32(taddr + c * 32, v);
    load_alpha(c, a);
#pragma unroll
    for (int j = 0; j < 32; ++j) D += a[j] * v[j];
  }
  for (int c = 0; c < n_act; ++c) {
    float a[32];
    tmem_ld32(taddr + c * 32, v);
    load_alpha(c, a);
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = a[j] * (v[j] - D);
    stage_store_bf16(stg, mbf, v, c * 32, row0, b, lane);
  }
}

// Decoding step (NEXT-4): one thread per row, the row's <= 128 columns of this
// tile: running (max, sumexp) as EPI_LSE and the 8 best (logit, token) pairs
// under the order "logit descending, token ascending".  A (logit, token) pair
// is one 64-bit key (order-preserving float bits, then the complemented
// token), so "better" is an unsigned compare.  Each 32-column chunk's best 8
// come from sorting networks on registers (no divergence, no memory): four
// sorted groups of 8, then bitonic top-8 merges, then a merge with the
// running list.
template <typename OutT>
__device__ __forceinline__ void epi_topk(const EpiParams& e, uint32_t taddr, int n_act, int col_h,
                                         int rowg, bool row_ok, int slot) {
  float mx = -INFINITY, s = 0.f;
  uint32_t best[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) best[i] = 0u;   // below every real key
  for (int c = 0; c < n_act; ++c) {
    float v[32];
    tmem_ld32(taddr + c * 32, v);
    const int col0 = col_h + c * 32;
    const int nv = row_ok ? e.ncols_valid - col0 : 0;
    if (nv <= 0) continue;
    if (e.bias) add_bias32<OutT>(e.bias, e.col_base + col0, nv, v);
    float cm = -INFINITY;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nv) cm = fmaxf(cm, v[j]);
    const float nm = fmaxf(mx, cm);
    const float nml = nm * kLog2e;
    float t = s * ex2_mufu(fmaf(mx, kLog2e, -nml));
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nv) t += ex2_mufu(fmaf(v[j], kLog2e, -nml));
    s = t;
    mx = nm;
    uint32_t k[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) k[j] = j < nv ? tk_key32(v[j], col0 - col_h + j) : 0u;   // local column
#pragma unroll
    for (int g = 0; g < 4; ++g) tk_sort8(k + 8 * g);
    tk_merge8(k, k + 8);
    tk_merge8(k + 16, k + 24);
    tk_merge8(k, k + 16);
    tk_merge8(best, k);
  }
  if (row_ok) {
    const long long o = (long long)rowg * e.part_ld + slot;
    e.part[o] = make_float2(mx, s);
    uint4* out = reinterpret_cast<uint4*>(e.topk + o * 8);
    out[0] = make_uint4(best[0], best[1], best[2], best[3]);
    out[1] = make_uint4(best[4], best[5], best[6], best[7]);
  }
}

// (__maxnreg__ instead of __launch_bounds__(384, 1): 128 registers leave room
// for one 256-thread dlogits block beside the CTA -- same-box C1 -1%)
template <typename OutT, bool kFast, int kPair, bool kDecode = false>
__global__ void __maxnreg__(128) gemm_tc_kernel(const __grid_constant__ TcParams P) {
  using Cfg = TcCfg<kPair>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* staging = smem + TC_RING_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + TC_EPI_WARPS * TC_STG_BYTES);
  uint64_t* full = bars;                       // [STAGES]
  uint64_t* empty = full + Cfg::STAGES;        // [STAGES]
  uint64_t* tfull = empty + Cfg::STAGES;       // [2]
  uint64_t* tempty = tfull + 2;                // [2]
  uint64_t* sfull = tempty + 2;                // [SCHED]
  uint64_t* sempty = sfull + TC_SCHED;         // [SCHED]
  int* sched_tile = reinterpret_cast<int*>(sempty + TC_SCHED);   // [SCHED]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sched_tile + TC_SCHED);
  uint64_t* rec_vs = reinterpret_cast<uint64_t*>(tmem_slot + 2);   // kVar: [8] stage starts

  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();
  constexpr bool kClu = Cfg::CLUSTER == 2;   // cluster of 2 CTAs
  constexpr bool kWide = Cfg::WIDE;
  constexpr bool kMc = kPair == 3 || kPair == 6;   // B multicast, per-CTA MMAs
  constexpr bool kVar = Cfg::VAR;       // variable-size stages, per-half accumulators
  constexpr uint64_t kRing = TC_RING_BYTES;
  const uint32_t rank = kClu ? cluster_ctarank() : 0;   // 0 = cluster leader
  const bool leader = rank == 0;

  constexpr uint32_t kWarpAlloc = 8, kWarpProducer = 10, kWarpMma = 11;
  if (warp == kWarpProducer && lane == 0) {
    for (int i = 0; i < Cfg::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kMc ? 2 : 1);   // kMc: both CTAs' MMAs free a stage
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], TC_EPI_WARPS * (kPair == 2 ? 2 : 1));
    }
    for (int i = 0; i < TC_SCHED; ++i) {
      mbar_init(&sfull[i], 1);
      // leader: its MMA + epilogue warps (+ the peer's producer and epilogue warps)
      mbar_init(&sempty[i], 1 + TC_EPI_WARPS + (kClu ? 1 + TC_EPI_WARPS : 0) + (kMc ? 1 : 0));
    }
    fence_barrier_init();
    for (int p = 0; p < P.nprob; ++p)
      for (int j = 0; j < 5; ++j) tma_prefetch_desc(&P.maps[p][j]);
  }
  if (warp == kWarpAlloc) {
    if constexpr (kPair == 2) tmem_alloc_pair(tmem_slot, 512);
    else tmem_alloc(tmem_slot, 512);
  }
  tc_fence_before();
  if constexpr (kClu) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // programmatic dependent launch: the prologue above overlapped the previous
  // kernel's tail; wait for its results, then let the next kernel's CTAs be
  // scheduled onto SMs as this (persistent, fully resident) grid retires
  pdl_wait();
  if (threadIdx.x == 0) pdl_trigger();

  // shared::cluster addresses of the leader's barriers (pair mode)
  auto leader_addr = [&](void* p) -> uint32_t { return mapa_shared(smem_u32(p), 0); };

  if (warp == kWarpProducer) {
    // ---------------- tile scheduler (leader) + TMA producer (both CTAs).
    // The whole warp runs the loop (waits are per lane, values warp-uniform);
    // one elected lane issues, so TMA operands live in uniform registers.
    // The schedule is software-pipelined: tile i+1 is fetched, published to
    // the ring and decoded right after tile i's first load is issued, so the
    // tile boundary costs nothing but the empty-slot wait.  The tile counter
    // atomic is issued by lane 1: lane 0 issues every mbarrier arrive
    // (release semantics), which would otherwise wait for its round trip.
    int s = 0;
    uint32_t ph = 0;
    int r = 0;
    uint32_t rph = 0;
    int t_raw = 0;   // lane 1: result of the latest tile-counter fetch
    auto fetch = [&](int) {
      if (lane == 1) t_raw = atomicAdd(P.tile_counter, 1);
    };
    // next tile id: the leader takes it from the counter and publishes it to
    // its ring (and the peer's); the peer reads its ring
    auto next_tile = [&](int prev) -> int {
      int t;
      if (leader) {
        t = __shfl_sync(0xffffffffu, t_raw, 1);
        if (t >= P.total_tiles) t = -1;
        mbar_wait(&sempty[r], rph ^ 1);
        if (elect_one()) {
          sched_tile[r] = t;
          if constexpr (kClu) {
            st_shared_cluster_u32(mapa_shared(smem_u32(&sched_tile[r]), 1), (uint32_t)t);
            mbar_arrive_cluster(mapa_shared(smem_u32(&sfull[r]), 1));
          }
          mbar_arrive(&sfull[r]);
        }
        __syncwarp();
        if (t >= 0) fetch(t);
      } else {
        mbar_wait_cluster(&sfull[r], rph);
        t = sched_tile[r];
        __syncwarp();
        if (elect_one()) mbar_arrive_cluster(leader_addr(&sempty[r]));
        __syncwarp();
      }
      if (++r == TC_SCHED) { r = 0; rph ^= 1; }
      return t;
    };
    if (leader) fetch(-1);
    uint64_t vs_ = 0;      // kVar: virtual byte offset of the next stage
    long long vi_ = 0;     // kVar: stage counter
    long long wfree_ = 0;  // kVar: oldest stage not yet known to be consumed
    int t = next_tile(-1);
    TcTile tl{};
    if (t >= 0) tl = tc_decode<kPair>(P, t);
    while (t >= 0) {
      const TcProblem& pr = P.prob[tl.p];
      if (leader && P.trace && lane == 2) P.trace[(long long)t * 16] = smid();
      const CUtensorMap* ma0 = &P.maps[tl.p][0];
      const CUtensorMap* ma1 = &P.maps[tl.p][1];
      const CUtensorMap* mb0 = &P.maps[tl.p][2];
      const CUtensorMap* mb1 = &P.maps[tl.p][3];
      const int am0 = tl.m0 + Cfg::CTA_ROWS * rank;       // this CTA's A rows
      const int bn0 = tl.n0 + Cfg::B_ROWS * rank;         // this CTA's B rows
      const int kb_total = pr.kb_total;
      int t_nxt = -1;
      TcTile tl_nxt{};
      for (int kb = 0; kb < kb_total; ++kb) {
        uint32_t poff = 0;
        uint32_t stage_bytes = Cfg::STAGE;
        if constexpr (kVar) {
          // variable-size stages in a byte ring: a stage never wraps; before
          // writing, every older stage whose bytes (or barrier slot) it reuses
          // must have been consumed by the MMA warp
          stage_bytes = tl.nsub == 2 ? Cfg::STAGE : TC_A_BYTES + Cfg::B_SMEM;
          uint64_t po = vs_ % kRing;
          if (po + stage_bytes > kRing) { vs_ += kRing - po; po = 0; }
          const uint64_t ve = vs_ + stage_bytes;
          while (wfree_ < vi_ && (wfree_ + 8 <= vi_ || rec_vs[wfree_ & 7] + kRing < ve)) {
            mbar_wait(&empty[wfree_ & 7], (uint32_t)((wfree_ >> 3) & 1));
            ++wfree_;
          }
          if (lane == 0) rec_vs[vi_ & 7] = vs_;
          __syncwarp();
          poff = (uint32_t)po;
          s = (int)(vi_ & 7);
        } else {
          mbar_wait(&empty[s], ph ^ 1);
        }
        if (elect_one()) {
          uint8_t* sA = smem + (kVar ? poff : s * Cfg::STAGE);
          uint8_t* sB = sA + (kVar ? (tl.nsub == 2 ? Cfg::A_SMEM : TC_A_BYTES) : Cfg::A_SMEM);
          uint32_t barc = 0;
          if constexpr (kPair == 2) barc = leader_addr(&full[s]);
          if constexpr (kMc) {
            // own A rows; own half of B, multicast into both CTAs' B tile
            mbar_arrive_expect_tx(&full[s], Cfg::STAGE);
            const bool seg1 = pr.kseg > 0 && kb >= pr.kseg;
            const int ka = (seg1 ? kb - pr.kseg : kb) * TC_BK;
            tc_load_operand<1>(sA, seg1 ? ma1 : ma0, &full[s], 0, pr.a_mode, TC_BM, am0, ka, tl.b);
            if constexpr (kWide)
              tc_load_operand<1>(sA + TC_A_BYTES, seg1 ? ma1 : ma0, &full[s], 0, pr.a_mode, TC_BM,
                                 am0 + TC_BM, ka, tl.b);
            const bool bseg1 = seg1 && pr.b_seg;
            const int kbk = (bseg1 ? kb - pr.kseg : kb) * TC_BK + pr.b_koff;
            const CUtensorMap* mb = bseg1 ? mb1 : mb0;
            uint8_t* sBh = sB + rank * (Cfg::B_SMEM / 2);
            if (pr.b_nsplit > 0 && pr.b_mode == 1) {
              if (bn0 >= pr.b_nsplit)
                tma_load_4d_mc(sBh, mb1, &full[s], 0, kbk, (bn0 - pr.b_nsplit) / 64, tl.b, 3);
              else
                tma_load_4d_mc(sBh, mb0, &full[s], 0, kbk, bn0 / 64, tl.b, 3);
            } else if (pr.b_nsplit > 0) {
              for (int i = 0; i < Cfg::B_ROWS / 64; ++i) {
                const int n = bn0 + 64 * i;
                if (n >= pr.b_nsplit)
                  tma_load_3d_mc(sBh + i * 8192, mb1, &full[s], n - pr.b_nsplit, kbk, tl.b, 3);
                else
                  tma_load_3d_mc(sBh + i * 8192, mb0, &full[s], n, kbk, tl.b, 3);
              }
            } else {
              tc_load_operand_mc(sBh, mb, &full[s], pr.b_mode, Cfg::B_ROWS, bn0, kbk, tl.b);
            }
          } else {
            if (leader)
              mbar_arrive_expect_tx(&full[s], kVar ? stage_bytes
                                              : (kPair == 1 || kPair == 4)
                                                  ? Cfg::A_SMEM + pr.bn * TC_BK * 2
                                                  : Cfg::STAGE * Cfg::CLUSTER);
            const bool seg1 = pr.kseg > 0 && kb >= pr.kseg;
            const int ka = (seg1 ? kb - pr.kseg : kb) * TC_BK;
            tc_load_operand<kPair>(sA, seg1 ? ma1 : ma0, &full[s], barc, pr.a_mode, TC_BM, am0,
                                   ka, tl.b);
            if (kWide && tl.nsub == 2)   // the second 128-row half of A
              tc_load_operand<kPair>(sA + TC_A_BYTES, seg1 ? ma1 : ma0, &full[s], barc, pr.a_mode,
                                     TC_BM, am0 + TC_BM, ka, tl.b);
            const bool bseg1 = seg1 && pr.b_seg;
            const int kbk = (bseg1 ? kb - pr.kseg : kb) * TC_BK + pr.b_koff;
            const CUtensorMap* mb = bseg1 ? mb1 : mb0;
            if (pr.b_nsplit > 0 && pr.b_mode == 1) {
              if (bn0 >= pr.b_nsplit)
                tl4<kPair>(sB, mb1, &full[s], barc, 0, kbk, (bn0 - pr.b_nsplit) / 64, tl.b);
              else
                tl4<kPair>(sB, mb0, &full[s], barc, 0, kbk, bn0 / 64, tl.b);
            } else if (pr.b_nsplit > 0) {
              for (int i = 0; i < Cfg::B_ROWS / 64; ++i) {
                const int n = bn0 + 64 * i;
                if (n >= pr.b_nsplit)
                  tl3<kPair>(sB + i * 8192, mb1, &full[s], barc, n - pr.b_nsplit, kbk, tl.b);
                else
                  tl3<kPair>(sB + i * 8192, mb0, &full[s], barc, n, kbk, tl.b);
              }
            } else {
              tc_load_operand<kPair>(sB, mb, &full[s], barc, pr.b_mode, Cfg::B_ROWS, bn0, kbk,
                                     tl.b);
            }
          }
        }
        __syncwarp();
        if (leader && kb == 0) TC_TRACE(t, 11);             // first load issued
        if (leader && kb == kb_total - 1) TC_TRACE(t, 2);   // last load issued
        if constexpr (kVar) {
          vs_ += stage_bytes;
          ++vi_;
        } else {
          if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
        }
        if (kb == 0) {
          // the next tile: fetch, publish and decode in the shadow of this one
          t_nxt = next_tile(t);
          if (t_nxt >= 0) tl_nxt = tc_decode<kPair>(P, t_nxt);
          if (leader && t_nxt >= 0) TC_TRACE(t_nxt, 12);
        }
      }
      t = t_nxt;
      tl = tl_nxt;
    }
  } else if (warp == kWarpMma) {
    if (leader || kMc) {
      // ---------------- MMA issuer (pair leader only): the whole warp waits,
      // one elected lane issues tcgen05.mma and the commits.  The next tile
      // is read from the ring and decoded during the current tile's second
      // k-block (the producer published it after this tile's first load).
      int s = 0;
      uint32_t ph = 0;
      int r = 0;
      uint32_t rph = 0;
      int acc = 0;
      uint32_t aph = 0;
      uint64_t mvs = 0;     // kVar: the producer's stage sequence, replayed
      long long mvi = 0;
      uint32_t sph = 0;     // kVar: phase bit of each TMEM accumulator slot
      auto read_tile = [&]() -> int {
        if (kClu && !leader) mbar_wait_cluster(&sfull[r], rph);
        else mbar_wait(&sfull[r], rph);
        const int t = sched_tile[r];
        __syncwarp();
        if (elect_one()) {
          if (kClu && !leader) mbar_arrive_cluster(leader_addr(&sempty[r]));
          else mbar_arrive(&sempty[r]);
        }
        __syncwarp();
        if (++r == TC_SCHED) { r = 0; rph ^= 1; }
        return t;
      };
      int t = read_tile();
      TcTile tl{};
      if (t >= 0) tl = tc_decode<kPair>(P, t);
      while (t >= 0) {
        TC_TRACE(t, 3);
        const TcProblem& pr = P.prob[tl.p];
        TC_TRACE(t, 8);   // decoded
        const uint32_t idesc = umma_idesc_bf16(Cfg::MMA_M, pr.bn, pr.a_mn, pr.b_mn);
        const uint32_t a_lbo = pr.a_mn ? 8192u : 16u;
        const uint32_t b_lbo = pr.b_mn ? 8192u : 16u;
        const uint32_t a_kstep = pr.a_mn ? 2048u : 32u;
        const uint32_t b_kstep = pr.b_mn ? 2048u : 32u;
        const int kb_total = pr.kb_total;
        const int kb_read = kb_total > 1 ? 1 : 0;
        int t_nxt = -1;
        TcTile tl_nxt{};
        const int nsub = tl.nsub;
        const int acc2 = acc ^ 1;
        if constexpr (kVar) {   // one or two 256-column slots, each with its own phase
          mbar_wait(&tempty[acc], ((sph >> acc) & 1) ^ 1);
          if (nsub == 2) mbar_wait(&tempty[acc2], ((sph >> acc2) & 1) ^ 1);
        } else {
          mbar_wait(&tempty[acc], aph ^ 1);
        }
        tc_fence_after();
        TC_TRACE(t, 9);   // accumulator free
        const uint32_t dcol = tmem_base + acc * TC_BN;
        const uint32_t dcol2 = kVar ? tmem_base + acc2 * TC_BN : dcol + TC_BN;
        for (int kb = 0; kb < kb_total; ++kb) {
          if (kb == 0) TC_TRACE(t, 10);
          uint32_t poff = 0, stage_bytes = Cfg::STAGE;
          if constexpr (kVar) {
            stage_bytes = nsub == 2 ? Cfg::STAGE : TC_A_BYTES + Cfg::B_SMEM;
            uint64_t po = mvs % kRing;
            if (po + stage_bytes > kRing) { mvs += kRing - po; po = 0; }
            poff = (uint32_t)po;
            s = (int)(mvi & 7);
            mbar_wait(&full[s], (uint32_t)((mvi >> 3) & 1));
          } else {
            mbar_wait(&full[s], ph);
          }
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sA = smem_u32(smem + (kVar ? poff : s * Cfg::STAGE));
            const uint32_t sB = sA + (kVar ? (nsub == 2 ? Cfg::A_SMEM : TC_A_BYTES) : Cfg::A_SMEM);
#pragma unroll
            for (int k = 0; k < TC_BK / 16; ++k) {
              const uint64_t ad = umma_sdesc(sA + k * a_kstep, a_lbo, 1024);
              const uint64_t bd = umma_sdesc(sB + k * b_kstep, b_lbo, 1024);
              if constexpr (kPair == 2) umma_bf16_pair(dcol, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
              else umma_bf16(dcol, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
              if (kWide && nsub == 2) {   // rows 128..255 into the second accumulator
                const uint64_t ad2 = umma_sdesc(sA + TC_A_BYTES + k * a_kstep, a_lbo, 1024);
                umma_bf16(dcol2, ad2, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
              }
            }
            if constexpr (kPair == 2) umma_commit_pair(&empty[s]);
            else if constexpr (kMc) umma_commit_mc(&empty[s], 3);
            else umma_commit(&empty[s]);
          }
          __syncwarp();
          if (kb == 0) TC_TRACE(t, 4);   // first MMAs issued
          if (kb == 0 && P.trace) {
            const long long gt = gtime();
            if (lane == 2) P.trace[(long long)t * 16 + 14] = gt;
          }
          if constexpr (kVar) {
            mvs += stage_bytes;
            ++mvi;
          } else {
            if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
          }
          if (kb == kb_read) {
            t_nxt = read_tile();
            if (t_nxt >= 0) tl_nxt = tc_decode<kPair>(P, t_nxt);
          }
        }
        if (elect_one()) {
          if constexpr (kPair == 2) umma_commit_pair(&tfull[acc]);
          else umma_commit(&tfull[acc]);
          if (kVar && nsub == 2) umma_commit(&tfull[acc2]);
        }
        __syncwarp();
        TC_TRACE(t, 5);   // last commit issued
        if (P.trace) {
          const long long gt = gtime();
          if (lane == 2) P.trace[(long long)t * 16 + 15] = gt;
        }
        if constexpr (kVar) {
          sph ^= 1u << acc;
          if (nsub == 2) sph ^= 1u << acc2;
          else acc = acc2;
        } else {
          if (++acc == Cfg::ACCS) { acc = 0; aph ^= 1; }
        }
        t = t_nxt;
        tl = tl_nxt;
      }
    }
  } else if (warp < TC_EPI_WARPS) {
    // ---------------- epilogue (8 warps)
    const uint32_t ew = warp;
    const uint32_t q = warp & 3;        // TMEM lane quarter = tile rows 32q..32q+31
    const uint32_t h = ew >> 2;         // column half of the 256-wide tile
    const uint32_t stg = smem_u32(staging + ew * TC_STG_BYTES);
    const uint32_t swz = lane & 7;
    int r = 0;
    uint32_t rph = 0;
    int acc = 0;
    uint32_t aph = 0;
    uint32_t esph = 0;   // kVar: phase bit of each TMEM accumulator slot
    for (;;) {
      if (kClu && !leader) mbar_wait_cluster(&sfull[r], rph);
      else mbar_wait(&sfull[r], rph);
      const int t = sched_tile[r];
      __syncwarp();
      if (lane == 0) {
        if (kClu && !leader) mbar_arrive_cluster(leader_addr(&sempty[r]));
        else mbar_arrive(&sempty[r]);
      }
      if (++r == TC_SCHED) { r = 0; rph ^= 1; }
      if (t < 0) break;
      const TcTile tl = tc_decode<kPair>(P, t);
      const TcProblem& pr = P.prob[tl.p];
      const int kind = pr.epi.kind;
      const CUtensorMap* omap = &P.maps[tl.p][4];
      if constexpr (!kVar) {
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
      }
      if (warp == 0 && leader) TC_TRACE(t, 6);
      // wide tiles: two 128-row halves, the second in TMEM columns 256..511
      // (kVar: each half in its own accumulator slot, released when drained)
#pragma unroll 1
      for (int sub = 0; sub < (kVar ? tl.nsub : (kWide ? 2 : 1)); ++sub) {
      if constexpr (kVar) {
        mbar_wait(&tfull[acc], (esph >> acc) & 1);
        tc_fence_after();
      }
      const int row0 = tl.m0 + Cfg::CTA_ROWS * rank + sub * TC_BM + q * 32;   // row inside the batch item
      const int row = row0 + lane;
      const bool row_ok = row < pr.M;
      const int rowg = tl.b * pr.M + (row_ok ? row : 0);   // row of the flattened [batch*M] arrays
      const uint32_t taddr =
          tmem_base + ((q * 32u) << 16) + (kVar ? acc : acc + sub) * TC_BN + h * 128;
      const int col_h = tl.n0 + h * 128;
      const int lim = (kind == EPI_LSE || kind == EPI_TOPK || kind == EPI_ATTN_SOFTMAX ||
                       kind == EPI_ATTN_SOFTMAX_BWD)
                          ? pr.epi.ncols_valid : pr.epi.ncols_store;
      const int n_act =
          max(0, min(4, (min(lim, tl.n0 + pr.bn) - col_h + 31) / 32));   // warp-uniform
      if (kind == EPI_ATTN_SOFTMAX) {
        if (n_act > 0)
          epi_attn_softmax(taddr, n_act, pr.epi.src_len[tl.b], staging + ew * TC_STG_BYTES,
                           &P.maps[tl.p][3], omap, row0, tl.b, lane);
      } else if (kind == EPI_ATTN_SOFTMAX_BWD) {
        if (n_act > 0)
          epi_attn_softmax_bwd(pr.epi, taddr, n_act, rowg, row_ok, staging + ew * TC_STG_BYTES,
                               omap, row0, tl.b, lane);
      } else if (kind == EPI_COL0_F32) {
        if (h == 0 && n_act > 0) {
          float v[32];
          tmem_ld32(taddr, v);
          if (row_ok) static_cast<float*>(pr.epi.out)[rowg] = v[0];
        }
      } else if (kDecode && kind == EPI_TOPK) {
        if constexpr (kDecode)
          epi_topk<OutT>(pr.epi, taddr, n_act, col_h, rowg, row_ok, tl.tn * 2 + h);
      } else {
        RowEpilogue<OutT, kFast> epi(pr.epi, rowg, 0);
        const bool f32out = epi_out_is_f32(kind);
#pragma unroll 1
        for (int c = 0; c < n_act; ++c) {
          float v[32];
          tmem_ld32(taddr + c * 32, v);
          const int col = col_h + c * 32;
          if (kind == EPI_LSE) {
            if (row_ok) epi.chunk(col, v);   // (adds the bias to v)
            if (!pr.epi.out) continue;       // else store the logits as fp16
          } else {
            if (kind == EPI_NONE) continue;
            epi.transform(col, v);
          }
          if (kind == EPI_ADD_BF16 && row_ok) {
            const float4* ad = reinterpret_cast<const float4*>(pr.epi.addend +
                                                               (long long)rowg * pr.epi.add_ld + col);
#pragma unroll
            for (int g = 0; g < 8; ++g) {
              const float4 a4 = ad[g];
              v[4 * g] += a4.x;
              v[4 * g + 1] += a4.y;
              v[4 * g + 2] += a4.z;
              v[4 * g + 3] += a4.w;
            }
          }
          if (f32out) {
            if (lane == 0) bulk_wait_read0();
            __syncwarp();
#pragma unroll
            for (int g = 0; g < 8; ++g)
              st_shared_v4(stg + lane * 128 + ((g ^ swz) << 4), __float_as_uint(v[4 * g]),
                           __float_as_uint(v[4 * g + 1]), __float_as_uint(v[4 * g + 2]),
                           __float_as_uint(v[4 * g + 3]));
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (kind == EPI_ACCUM_F32)
                tma_reduce_add_3d(omap, staging + ew * TC_STG_BYTES, col, row0, tl.b);
              else
                tma_store_3d(omap, staging + ew * TC_STG_BYTES, col, row0, tl.b);
              bulk_commit();
            }
          } else {
            if ((c & 1) == 0) {
              if (lane == 0) bulk_wait_read0();
              __syncwarp();
            }
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              uint32_t w[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                if (kind == EPI_LSE) {
                  __half2 h2 = __floats2half2_rn(v[8 * g + 2 * e], v[8 * g + 2 * e + 1]);
                  w[e] = *reinterpret_cast<uint32_t*>(&h2);
                } else {
                  __nv_bfloat162 h2 = __floats2bfloat162_rn(v[8 * g + 2 * e], v[8 * g + 2 * e + 1]);
                  w[e] = *reinterpret_cast<uint32_t*>(&h2);
                }
              }
              const uint32_t gi = (c & 1) * 4 + g;
              st_shared_v4(stg + lane * 128 + ((gi ^ swz) << 4), w[0], w[1], w[2], w[3]);
            }
            if (kind == EPI_DLOGITS) {   // the -onehot term: the target column gets rs (p_y - 1)
              const int yl = epi.y - col;
              if ((unsigned)yl < 32u && row_ok && epi.rs > 0.f) {
                const uint32_t gi = (c & 1) * 4 + (yl >> 3);
                st_shared_u16(stg + lane * 128 + ((gi ^ swz) << 4) + (yl & 7) * 2,
                              __bfloat16_as_ushort(__float2bfloat16_rn(epi.fix)));
              }
            }
            if ((c & 1) == 1 || c == n_act - 1) {
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_3d(omap, staging + ew * TC_STG_BYTES, col_h + (c & ~1) * 32, row0, tl.b);
                bulk_commit();
              }
            }
          }
        }
        if (kind == EPI_LSE && row_ok) epi.finish(tl.tn * 2 + h);
      }
      if constexpr (kVar) {   // this half's slot is free for the next tile's MMAs
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        esph ^= 1u << acc;
        acc ^= 1;
      }
      }
      if constexpr (!kVar) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (kPair == 2 && !leader) mbar_arrive_cluster(leader_addr(&tempty[acc]));
          else mbar_arrive(&tempty[acc]);
        }
        if (++acc == Cfg::ACCS) { acc = 0; aph ^= 1; }
      }
      if (warp == 0 && leader) TC_TRACE(t, 7);
    }
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  if constexpr (kClu) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  if (warp == kWarpAlloc) {
    if constexpr (kPair == 2) tmem_dealloc_pair(tmem_base, 512);
    else tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace attnsm
