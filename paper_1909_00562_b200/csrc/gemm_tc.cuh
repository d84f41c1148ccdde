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

// kPair = 1: one CTA computes a 128 x 256 tile (tcgen05 cta_group::1), two
//            accumulators in TMEM so a tile's epilogue overlaps the next
//            tile's MMAs; 4 x 48 KB stages.
// kPair = 4 ("wide"): one CTA computes a 256 x 256 tile as two M = 128 MMAs
//            per K step that share the B tile (accumulators in TMEM columns
//            0-255 and 256-511): twice the MMA work per staged byte of the
//            128 x 256 tile, at the price of one tile in TMEM at a time (the
//            epilogue is not overlapped with the next tile's MMAs).  64 KB
//            stages, 3 of them.  (Used by the stored-logits ablation's
//            vocab-backward launches; CTA pairs live in vocab.cuh.)
template <int kPair>
struct TcCfg {
  static_assert(kPair == 1 || kPair == 4, "tile modes: 1 (128 x 256) and 4 (wide 256 x 256)");
  static constexpr bool WIDE = kPair == 4;
  static constexpr int TILE_M = WIDE ? 2 * TC_BM : TC_BM;     // rows per scheduled tile
  static constexpr int A_SMEM = (WIDE ? 2 : 1) * TC_A_BYTES;
  static constexpr int B_SMEM = TC_BN * TC_BK * 2;
  static constexpr int STAGE = A_SMEM + B_SMEM;                // 48 | 64 KB
  static constexpr int STAGES = TC_RING_BYTES / STAGE;         // 4 | 3
  static constexpr int ACCS = WIDE ? 1 : 2;                    // tiles resident in TMEM
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
  int bn;           // tile columns (UMMA N): 256, or 16..240 for K-major B
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
  int claim_late;     // claim the next tile two k-blocks before the end of the current
                      // one's loads (default: right after its first load)
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
  r.m0 = tm * TcCfg<kPair>::TILE_M;
  r.n0 = r.tn * pr.bn;
  return r;
}

// Load one operand tile (rows x 64 K) of k-block kb into smem.
__device__ __forceinline__ void tc_load_operand(uint8_t* dst, const CUtensorMap* m, uint64_t* bar,
                                                int mode, int rows, int r0, int k0, int b) {
  if (mode == 0) {
    tma_load_3d(dst, m, bar, k0, r0, b);
  } else if (mode == 1) {
    tma_load_4d(dst, m, bar, 0, k0, r0 / 64, b);
  } else {
    for (int i = 0; i < rows / 64; ++i) tma_load_3d(dst + i * 8192, m, bar, r0 + 64 * i, k0, b);
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
// for one 256-thread elementwise block beside the CTA -- the stored-logits
// ablation's overlapped dlogits kernels)
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

  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();
  constexpr bool kWide = Cfg::WIDE;

  constexpr uint32_t kWarpAlloc = 8, kWarpProducer = 10, kWarpMma = 11;
  if (warp == kWarpProducer && lane == 0) {
    for (int i = 0; i < Cfg::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], TC_EPI_WARPS);
    }
    for (int i = 0; i < TC_SCHED; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sempty[i], 1 + TC_EPI_WARPS);   // MMA warp + epilogue warps
    }
    fence_barrier_init();
    for (int p = 0; p < P.nprob; ++p)
      for (int j = 0; j < 5; ++j) tma_prefetch_desc(&P.maps[p][j]);
  }
  if (warp == kWarpAlloc) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // programmatic dependent launch: the prologue above overlapped the previous
  // kernel's tail; wait for its results, then let the next kernel's CTAs be
  // scheduled onto SMs as this (persistent, fully resident) grid retires
  pdl_wait();
  if (threadIdx.x == 0) pdl_trigger();

  // the scheduler ring: tile ids published by the producer warp
  auto ring_read = [&](int& r, uint32_t& rph, bool lane0) -> int {
    mbar_wait(&sfull[r], rph);
    const int t = sched_tile[r];
    __syncwarp();
    if (lane0 ? lane == 0 : elect_one()) mbar_arrive(&sempty[r]);
    __syncwarp();
    if (++r == TC_SCHED) { r = 0; rph ^= 1; }
    return t;
  };

  if (warp == kWarpProducer) {
    // ---------------- tile scheduler + TMA producer.  The whole warp runs the
    // loop (waits are per lane, values warp-uniform); one elected lane issues,
    // so TMA operands live in uniform registers.  The schedule is
    // software-pipelined: tile i+1 is fetched, published and decoded right
    // after tile i's first load is issued.  The tile counter atomic is issued
    // by lane 1: lane 0 issues every mbarrier arrive (release semantics),
    // which would otherwise wait for its round trip.
    int s = 0;
    uint32_t ph = 0;
    int r = 0;
    uint32_t rph = 0;
    int t_raw = 0;   // lane 1: result of the latest tile-counter fetch
    auto fetch = [&]() {
      if (lane == 1) t_raw = atomicAdd(P.tile_counter, 1);
    };
    auto next_tile = [&]() -> int {
      int t = __shfl_sync(0xffffffffu, t_raw, 1);
      if (t >= P.total_tiles) t = -1;
      mbar_wait(&sempty[r], rph ^ 1);
      if (elect_one()) {
        sched_tile[r] = t;
        mbar_arrive(&sfull[r]);
      }
      __syncwarp();
      if (t >= 0 && !P.claim_late) fetch();
      if (++r == TC_SCHED) { r = 0; rph ^= 1; }
      return t;
    };
    fetch();
    int t = next_tile();
    TcTile tl{};
    if (t >= 0) tl = tc_decode<kPair>(P, t);
    while (t >= 0) {
      const TcProblem& pr = P.prob[tl.p];
      if (P.trace && lane == 2) P.trace[(long long)t * 16] = smid();
      const CUtensorMap* ma0 = &P.maps[tl.p][0];
      const CUtensorMap* ma1 = &P.maps[tl.p][1];
      const CUtensorMap* mb0 = &P.maps[tl.p][2];
      const CUtensorMap* mb1 = &P.maps[tl.p][3];
      const int kb_total = pr.kb_total;
      int t_nxt = -1;
      TcTile tl_nxt{};
      for (int kb = 0; kb < kb_total; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        if (elect_one()) {
          uint8_t* sA = smem + s * Cfg::STAGE;
          uint8_t* sB = sA + Cfg::A_SMEM;
          mbar_arrive_expect_tx(&full[s], Cfg::A_SMEM + pr.bn * TC_BK * 2);
          const bool seg1 = pr.kseg > 0 && kb >= pr.kseg;
          const int ka = (seg1 ? kb - pr.kseg : kb) * TC_BK;
          tc_load_operand(sA, seg1 ? ma1 : ma0, &full[s], pr.a_mode, TC_BM, tl.m0, ka, tl.b);
          if (kWide)   // the second 128-row half of A
            tc_load_operand(sA + TC_A_BYTES, seg1 ? ma1 : ma0, &full[s], pr.a_mode, TC_BM,
                            tl.m0 + TC_BM, ka, tl.b);
          const bool bseg1 = seg1 && pr.b_seg;
          const int kbk = (bseg1 ? kb - pr.kseg : kb) * TC_BK + pr.b_koff;
          const CUtensorMap* mb = bseg1 ? mb1 : mb0;
          if (pr.b_nsplit > 0 && pr.b_mode == 1) {
            if (tl.n0 >= pr.b_nsplit)
              tma_load_4d(sB, mb1, &full[s], 0, kbk, (tl.n0 - pr.b_nsplit) / 64, tl.b);
            else
              tma_load_4d(sB, mb0, &full[s], 0, kbk, tl.n0 / 64, tl.b);
          } else if (pr.b_nsplit > 0) {
            for (int i = 0; i < TC_BN / 64; ++i) {
              const int n = tl.n0 + 64 * i;
              if (n >= pr.b_nsplit)
                tma_load_3d(sB + i * 8192, mb1, &full[s], n - pr.b_nsplit, kbk, tl.b);
              else
                tma_load_3d(sB + i * 8192, mb0, &full[s], n, kbk, tl.b);
            }
          } else {
            tc_load_operand(sB, mb, &full[s], pr.b_mode, pr.bn, tl.n0, kbk, tl.b);
          }
        }
        __syncwarp();
        if (kb == 0) TC_TRACE(t, 11);             // first load issued
        if (kb == kb_total - 1) TC_TRACE(t, 2);   // last load issued
        if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
        if (P.claim_late) {
          if (kb == max(0, kb_total - 2)) fetch();
        } else if (kb == 0) {
          // the next tile: fetch, publish and decode in the shadow of this one
          t_nxt = next_tile();
          if (t_nxt >= 0) tl_nxt = tc_decode<kPair>(P, t_nxt);
          if (t_nxt >= 0) TC_TRACE(t_nxt, 12);
        }
      }
      if (P.claim_late) {
        t_nxt = next_tile();
        if (t_nxt >= 0) tl_nxt = tc_decode<kPair>(P, t_nxt);
      }
      t = t_nxt;
      tl = tl_nxt;
    }
  } else if (warp == kWarpMma) {
    // ---------------- MMA issuer: the whole warp waits, one elected lane
    // issues tcgen05.mma and the commits.  The next tile is read from the ring
    // and decoded during the current tile's second k-block.
    int s = 0;
    uint32_t ph = 0;
    int r = 0;
    uint32_t rph = 0;
    int acc = 0;
    uint32_t aph = 0;
    int t = ring_read(r, rph, false);
    TcTile tl{};
    if (t >= 0) tl = tc_decode<kPair>(P, t);
    while (t >= 0) {
      TC_TRACE(t, 3);
      const TcProblem& pr = P.prob[tl.p];
      const uint32_t idesc = umma_idesc_bf16(TC_BM, pr.bn, pr.a_mn, pr.b_mn);
      const uint32_t a_lbo = pr.a_mn ? 8192u : 16u;
      const uint32_t b_lbo = pr.b_mn ? 8192u : 16u;
      const uint32_t a_kstep = pr.a_mn ? 2048u : 32u;
      const uint32_t b_kstep = pr.b_mn ? 2048u : 32u;
      const int kb_total = pr.kb_total;
      const int kb_read = kb_total > 1 ? 1 : 0;
      int t_nxt = -1;
      TcTile tl_nxt{};
      mbar_wait(&tempty[acc], aph ^ 1);
      tc_fence_after();
      TC_TRACE(t, 9);   // accumulator free
      const uint32_t dcol = tmem_base + acc * TC_BN;
      for (int kb = 0; kb < kb_total; ++kb) {
        if (kb == 0) TC_TRACE(t, 10);
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sA = smem_u32(smem + s * Cfg::STAGE);
          const uint32_t sB = sA + Cfg::A_SMEM;
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k) {
            const uint64_t ad = umma_sdesc(sA + k * a_kstep, a_lbo, 1024);
            const uint64_t bd = umma_sdesc(sB + k * b_kstep, b_lbo, 1024);
            umma_bf16(dcol, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
            if (kWide) {   // rows 128..255 into the second accumulator
              const uint64_t ad2 = umma_sdesc(sA + TC_A_BYTES + k * a_kstep, a_lbo, 1024);
              umma_bf16(dcol + TC_BN, ad2, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
            }
          }
          umma_commit(&empty[s]);
        }
        __syncwarp();
        if (kb == 0) TC_TRACE(t, 4);   // first MMAs issued
        if (kb == 0 && P.trace) {
          const long long gt = gtime();
          if (lane == 2) P.trace[(long long)t * 16 + 14] = gt;
        }
        if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
        if (kb == kb_read && !P.claim_late) {
          t_nxt = ring_read(r, rph, false);
          if (t_nxt >= 0) tl_nxt = tc_decode<kPair>(P, t_nxt);
        }
      }
      if (elect_one()) umma_commit(&tfull[acc]);
      __syncwarp();
      if (P.claim_late) {   // after the commit: the epilogue starts first
        t_nxt = ring_read(r, rph, false);
        if (t_nxt >= 0) tl_nxt = tc_decode<kPair>(P, t_nxt);
      }
      TC_TRACE(t, 5);   // last commit issued
      if (P.trace) {
        const long long gt = gtime();
        if (lane == 2) P.trace[(long long)t * 16 + 15] = gt;
      }
      if (++acc == Cfg::ACCS) { acc = 0; aph ^= 1; }
      t = t_nxt;
      tl = tl_nxt;
    }
  } else if (warp < TC_EPI_WARPS) {
    // ---------------- epilogue (8 warps)
    const uint32_t q = warp & 3;        // TMEM lane quarter = tile rows 32q..32q+31
    const uint32_t h = warp >> 2;       // column half of the 256-wide tile
    const uint32_t stg = smem_u32(staging + warp * TC_STG_BYTES);
    const uint32_t swz = lane & 7;
    int r = 0;
    uint32_t rph = 0;
    int acc = 0;
    uint32_t aph = 0;
    for (;;) {
      const int t = ring_read(r, rph, true);
      if (t < 0) break;
      const TcTile tl = tc_decode<kPair>(P, t);
      const TcProblem& pr = P.prob[tl.p];
      const int kind = pr.epi.kind;
      const CUtensorMap* omap = &P.maps[tl.p][4];
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      if (warp == 0) TC_TRACE(t, 6);
      // wide tiles: two 128-row halves, the second in TMEM columns 256..511
#pragma unroll 1
      for (int sub = 0; sub < (kWide ? 2 : 1); ++sub) {
      const int row0 = tl.m0 + sub * TC_BM + q * 32;   // row inside the batch item
      const int row = row0 + lane;
      const bool row_ok = row < pr.M;
      const int rowg = tl.b * pr.M + (row_ok ? row : 0);   // row of the flattened [batch*M] arrays
      const uint32_t taddr = tmem_base + ((q * 32u) << 16) + (acc + sub) * TC_BN + h * 128;
      const int col_h = tl.n0 + h * 128;
      const int lim = (kind == EPI_LSE || kind == EPI_TOPK || kind == EPI_ATTN_SOFTMAX ||
                       kind == EPI_ATTN_SOFTMAX_BWD)
                          ? pr.epi.ncols_valid : pr.epi.ncols_store;
      const int n_act =
          max(0, min(4, (min(lim, tl.n0 + pr.bn) - col_h + 31) / 32));   // warp-uniform
      if (kind == EPI_ATTN_SOFTMAX) {
        if (n_act > 0)
          epi_attn_softmax(taddr, n_act, pr.epi.src_len[tl.b], staging + warp * TC_STG_BYTES,
                           &P.maps[tl.p][3], omap, row0, tl.b, lane);
      } else if (kind == EPI_ATTN_SOFTMAX_BWD) {
        if (n_act > 0)
          epi_attn_softmax_bwd(pr.epi, taddr, n_act, rowg, row_ok, staging + warp * TC_STG_BYTES,
                               omap, row0, tl.b, lane);
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
            if (pr.epi.addend_bf16) {
              const uint4* ad = reinterpret_cast<const uint4*>(
                  reinterpret_cast<const __nv_bfloat16*>(pr.epi.addend) + (long long)rowg * pr.epi.add_ld + col);
#pragma unroll
              for (int g = 0; g < 4; ++g) {
                const uint4 u = ad[g];
                const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[e]));
                  v[8 * g + 2 * e] += f.x;
                  v[8 * g + 2 * e + 1] += f.y;
                }
              }
            } else {
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
                tma_reduce_add_3d(omap, staging + warp * TC_STG_BYTES, col, row0, tl.b);
              else
                tma_store_3d(omap, staging + warp * TC_STG_BYTES, col, row0, tl.b);
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
            if ((c & 1) == 1 || c == n_act - 1) {
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_3d(omap, staging + warp * TC_STG_BYTES, col_h + (c & ~1) * 32, row0, tl.b);
                bulk_commit();
              }
            }
          }
        }
        if (kind == EPI_LSE && row_ok) epi.finish(tl.tn * 2 + h);
      }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == Cfg::ACCS) { acc = 0; aph ^= 1; }
      if (warp == 0) TC_TRACE(t, 7);
    }
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kWarpAlloc) tmem_dealloc(tmem_base, 512);
}

}  // namespace attnsm
