// vocab.cuh -- the vocabulary part of the stage as ONE persistent tcgen05
// launch: F4 (Eq. 5 logits -> per-tile log-sum-exp partials), F5 (lse, token
// NLL, loss; Eq. 6) and B1 (their backward).  The logits are never stored:
// the forward keeps per-tile (max, sum exp) partials only, and the backward
// recomputes the logits per V-chunk on the tensor cores, turning them into
// dL = rs (softmax - onehot) (bf16) in a chunk scratch sized for the L2 that
// the same launch consumes for dW_out and dHc (north_star
// "full logits are never round-tripped through HBM").  Measured: the dL lines
// are written back to DRAM once and, with dispatch orders 0 / 1, read back by
// their consumers; order 2 keeps the reads in L2.
//
// Tile types (T = B*N rows, chunk c = vocabulary columns [c0, c0 + vcc)):
//   G0       logits H_c W_out^T tile -> (max, sum exp) per row of the tile,
//            and the target logit                           M = T, N = V, K = d
//   LSE      lse_t, nll_t, rowscale_t of one row block from its G0 partials,
//            and the loss: not a dispatched tile -- the otherwise idle warps
//            8-9 of CTA pair p do it for row blocks p, p + pairs, ..., beside
//            the pair's tiles
//   G1(c)    dL_c = rs (exp(H_c W_out[c]^T - lse) - onehot)   M = T, N = vcc, K = d
//   G3(c)    dHc += dL_c W_out[c]                            M = T, N = d, K = vcc
//   G2(c)    dW_out[c] = dL_c^T H_c                           M = vcc, N = d, K = T
// MMA tiles are TM x 256 with fp32 accumulators in TMEM, two per CTA so a
// tile's epilogue overlaps the next tile's MMAs:
//   kPair = false: TM = 128, one CTA per tile (tcgen05 cta_group::1);
//   kPair = true:  TM = 256, a CTA pair (cluster of 2) per tile
//                  (cta_group::2): each CTA stages its 128 rows of A and its
//                  128 rows (N-columns) of B, both CTAs' TMA loads complete on
//                  the leader's barrier, the leader issues M = 256 MMAs that
//                  read the peer's shared memory, and each CTA's epilogue
//                  drains its own 128 accumulator rows.  L2 -> SM operand
//                  bytes per FLOP are 2/3 of the single-CTA tile's.
// The tiles form one dispatch list, pulled from a global atomic:
//   forward        G0(rb, all columns) for each row block rb
//   block 0        G1(0)
//   block c+1      G1(c+1), G3(c), G2(c)       (option order 0: G3(c), G2(c), G1(c+1))
// (the last block has no G1 and may put G2 first, so its long tiles do not form
// the tail).  Data dependencies between tiles are tracked with counters in
// global memory (release / acquire at gpu scope; async-proxy fences around the
// TMA traffic):
//   LSE(rb) waits for the G0 tiles of row block rb (g0done[rb]);
//   G1(c)   reads lse of its row block only after LSE(rb) (lsedone[rb]), and
//           writes dL buffer c % NB only after every G2 / G3 tile of chunk
//           c - NB has loaded it (consumed[c - NB]);
//   G3(c)   tile (row block rb) waits for every G1(c) tile of row block rb
//           (rowdone[c][rb]) -- and, before its reduce-add into dHc, for the G3
//           tile of chunk c-1 at the same place (dhcdone[rb][nt]): dHc is summed
//           in chunk order, so the result is deterministic;
//   G2(c)   tile waits for the G1(c) tiles of its columns over all row blocks
//           (coldone[c][cb]), and counts its finished dW_out stores (g2done[c])
//           so an allreduce of chunk c can start while the launch runs.
// Every wait targets tiles earlier in the dispatch list and all CTAs are
// resident (one per SM), so the waits cannot deadlock.  Counters count
// epilogue-warp portions (8 per CTA and tile), so their targets scale with the
// CTAs per tile.
//
// Roles (384 threads): warps 0-7 epilogue (warp w: TMEM lanes 32 (w % 4).., tile
// column half w / 4), warp 8 TMEM allocator, warps 8-9 the LSE row blocks,
// warp 10 scheduler + TMA producer, warp 11 MMA issuer (one elected lane; the
// pair leader's only).
#pragma once
#include "epilogue.cuh"
#include "ptx.cuh"

namespace attnsm {

// VB_DEBUG_MMA=1 compiles the timing-only MMA-issue variants of VbParams::debug
// bits 6 and 8-12 (development builds only: they slow the default issue loop)
#ifndef VB_DEBUG_MMA
#define VB_DEBUG_MMA 0
#endif

constexpr int VB_BN = 256;
constexpr int VB_BK = 64;
constexpr int VB_EPI_WARPS = 8;
// VB_STG_DB = 1 (experiment): two 4 KB staging buffers per epilogue warp (a
// store's shared memory is refilled while the previous one is still being
// read by the TMA unit), paid for with one ring stage (160 instead of 192 KB).
// Measured 6% slower at C1 (1.645 vs 1.549 ms, three alternating same-box
// pairs): the wide G2 / G3 tiles need the sixth stage (666-691 instead of
// ~520 cycles per 512 of work with five)
#ifndef VB_STG_DB
#define VB_STG_DB 0
#endif
// VB_STAGE3 = 1 (default): on CTA pairs a ring stage holds A and two B
// blocks (48 KB, four stages), so a wide k-block fills ONE stage; with 32 KB
// stages a wide k-block took two and left the second A region unused.  Wide
// G2 / G3 tiles: 494-503 instead of 516-552 cycles per 512 of work; vocab
// backward 1.556-1.559 vs 1.566-1.568 ms (three alternating same-box pairs)
#ifndef VB_STAGE3
#define VB_STAGE3 1
#endif
constexpr int VB_STG_BYTES = VB_STG_DB ? 8192 : 4096;   // staging per epilogue warp
constexpr int VB_THREADS = 384;
constexpr int VB_SCHED = 4;
constexpr int VB_RING = (VB_STG_DB ? 160 : 192) * 1024;
constexpr int VB_SMEM_BYTES = VB_RING + VB_EPI_WARPS * VB_STG_BYTES + 1024 + 512;
constexpr int VB_MAX_BLOCKS = 1024;                // chunks + 1

template <bool kPair>
struct VbCfg {
  static constexpr int CTAS = kPair ? 2 : 1;
  static constexpr int TM = 128 * CTAS;            // tile rows (M)
  static constexpr int B_ROWS = VB_BN / CTAS;      // B rows (N) staged per CTA
  static constexpr int A_BYTES = 128 * VB_BK * 2;  // 16 KB
  static constexpr int B_BYTES = B_ROWS * VB_BK * 2;
  // VB_STAGE3 (pairs): a stage holds A and TWO B blocks, so a wide k-block
  // fills one 48 KB stage instead of two 32 KB stages (whose second A region
  // stays unused); narrow k-blocks leave the second B empty
  static constexpr bool S3 = kPair && VB_STAGE3;
  static constexpr int STAGE = A_BYTES + (S3 ? 2 : 1) * B_BYTES;  // 48 KB | 32 KB (48 KB with S3)
  static constexpr int STAGES = VB_RING / STAGE;   // 4 | 6
  static constexpr int WARPS_PER_TILE = VB_EPI_WARPS * CTAS;
};

enum : int { VB_G1 = 0, VB_G3 = 1, VB_G2 = 2, VB_G0 = 3 };

struct alignas(64) VbParams {
  CUtensorMap m_hc_k;    // H_c [T, d] bf16, K-major A of G0 / G1: box {64, 128}
  CUtensorMap m_wo_k;    // W_out [V, d] bf16, K-major B of G0 / G1: box {64, B_ROWS}
  CUtensorMap m_dl_k;    // dL [NB][T][Vc] bf16, K-major A of G3: box {64, 128, 1}
  CUtensorMap m_wo_mn;   // W_out as [K = V][N = d], MN-major B of G3: box {64, 64, B_ROWS/64, 1}
  CUtensorMap m_dl_mn;   // dL as [K = T][M = Vc] per buffer, MN-major A of G2: box {64, 64, 2, 1}
  CUtensorMap m_hc_mn;   // H_c as [K = T][N = d], MN-major B of G2: box {64, 64, B_ROWS/64, 1}
  CUtensorMap m_dl_st;   // dL store: bf16 [NB][T][Vc], box {64, 32, 1}
  CUtensorMap m_dw_st;   // dW_out store: fp32 [V, d], box {32, 32}
  CUtensorMap m_dhc_st;  // dHc store / reduce-add: fp32 [T, d], box {32, 32}
  int T, d, V, Vc, nchunks, nbuf;
  int N;                 // decoder steps per sentence (row t = b N + i)
  int nrb;               // TM-row blocks of T
  int ndt;               // 256-column tiles of d
  int ncolf;             // 256-column blocks of a full chunk (Vc / 256)
  int wide;              // G2 / G3 tiles 512 columns wide (pairs, d % 512 == 0): per k-block two
                         // ring stages (A + B columns [0, 256), then B columns [256, 512)) and
                         // two N = 256 MMAs into both TMEM accumulators -- 3/4 of the operand
                         // bytes per FLOP of the 256-wide tile
  int ndw;               // G2 / G3 column tiles of d (ndt, or ndt / 2 when wide)
  int ntn;               // 256-column tiles of V (forward)
  int fwd_tiles;         // tiles of the forward section (0: forward not in this launch)
  int total_tiles;
  int* tile_counter;
  unsigned* g0done;      // [nrb]             G0 warp-portions done per row block (4 per CTA-tile)
  unsigned* lsedone;     // [nrb]             LSE warp-portions done per row block (2 per CTA)
  unsigned* g5count;     // [1]               LSE CTA-portions done (the last one sums the loss)
  unsigned* rowdone;     // [nchunks][nrb]    G1 warp-portions done per row block
  unsigned* coldone;     // [nchunks][nh][ncolf] G1 warp-portions done per 256-column block
                         // (and row half)
  unsigned* consumed;    // [nchunks][2]      G2 + G3 CTA-tiles whose operands are loaded
                         // (per row half with the order-2 split, else slot 0)
  unsigned* g2done;      // [nchunks]         G2 warp-portions whose dW_out stores completed
  unsigned* dhcdone;     // [nrb][ndt]        G3 warp-portions whose dHc update completed
  // forward outputs / backward row statistics
  float2* part;          // [ntn][T] (max, sum exp) per 256-column tile and row
  float* tgt_logit;      // [T]
  float* lse;            // [T]
  float* nll;            // [T] token NLL (0 on padded rows)
  float* rowscale;       // [T] loss_scale on valid rows, 0 on padded rows
  double* blockpart;     // [nrb * CTAS] per-CTA NLL sums of a row block
  float* loss;           // [1] loss_scale * sum of the NLL (fixed summation order)
  float loss_scale;
  const int* tgt;        // [T] target ids
  const int* tgt_len;    // [B]
  const void* bias;      // F_c bias b_out [V] bf16 (NEXT-1) or NULL
  float* db_part;        // with the bias: [T / 32][V] column sums of dL per 32-row group
  int last_g2_first;     // last block: G2 tiles before G3 tiles
  int order;             // 0: block c+1 = G3(c), G2(c), G1(c+1); 1: G1(c+1), G3(c), G2(c);
                         // 2: row-interleaved (block c = chunk c, see vb_decode_o2)
  int g1wide;            // G1 tiles 512 columns wide on CTA pairs (both accumulators,
                         // two chains at the full tensor rate; the epilogue no longer
                         // overlaps the next tile's MMAs)
  int claim_late;        // > 0: claim the next tile claim_late k-blocks before the end of
                         // the current one's loads; 0: right after its first load
  int nh;                // order 2: G2 split over T in nh (1 or 2) row halves (else 1)
  int h0;                // order 2: row blocks of the first half
  int lag;               // order 2: G3 of row block rb dispatched after G1 of rb + lag
  int n2max;             // G2 tiles of a full chunk (ceil(Vc / TM) * ndw): g2part stride
  unsigned* g2part;      // [nchunks][n2max]  order 2: first-half G2 warp-portions done
  int l2hints;           // bit 0: H_c loads evict-last; bit 1: dHc updates evict-last;
                         // bit 2: dL stores evict-last
  long long* trace;      // debug: 32 int64 per tile and CTA rank (see VB_TRACE), NULL = off
  int debug;             // timing experiments only (WRONG results): bit 0 skip the G1 stores,
                         // bit 1 skip the G1 exponentials, bit 2 skip the G2 / G3 stores,
                         // bit 3 publish tiles without waiting for their stores to land,
                         // bit 4 / 5 skip the B / A operand loads, bit 6 G1 reads its B
                         // operand MN-major (garbage values), bit 7 G1 epilogue skips
                         // its TMEM loads, bits 8 / 9 G1 k-steps as 2 x N = 128 / 4 x N = 64
                         // MMAs sharing A, bits 13 / 14 skip the operand loads of G2 / G3
  int blk_start[VB_MAX_BLOCKS + 2];   // backward blocks, relative to fwd_tiles
};

struct VbTile {
  int type, c, i, j;     // G0: i = row block, j = 256-col tile of V;
                         // G1: i = row block, j = 256-col tile of the chunk;
                         // G3: i = row block, j = d tile; G2: i = vocabulary row block
                         // of the chunk, j = d tile
  int vcc, kb_total;
  int h;                 // G2: row half of the K = T reduction (order 2), else 0
  int k0;                // G2: first row of its K range
};

__device__ __forceinline__ int vb_vcc(const VbParams& P, int c) {
  return min(P.Vc, P.V - c * P.Vc);
}

// G1 tiles per row block of a chunk of vcc columns
__device__ __forceinline__ int vb_g1cols(const VbParams& P, int vcc) {
  const int w = P.g1wide ? 2 * VB_BN : VB_BN;
  return (vcc + w - 1) / w;
}

// G2 tile of row half h: K range [k0, k0 + rows) of the T rows
template <bool kPair>
__device__ __forceinline__ void vb_g2_range(const VbParams& P, int h, int& k0, int& kb) {
  constexpr int TM = VbCfg<kPair>::TM;
  const int split = P.nh == 2 ? P.h0 * TM : P.T;
  k0 = h == 0 ? 0 : split;
  const int k1 = h == 0 ? min(split, P.T) : P.T;
  kb = (k1 - k0 + VB_BK - 1) / VB_BK;
}

// order 2 (row-interleaved), block = chunk c, in dispatch order:
//   for rb = 0 .. nrb-1:  G1(c, rb, all columns),  G3(c, rb - lag, all d tiles) if rb >= lag,
//                         and after the step rb = h0 - 1 + lag: G2(c, half 0, all tiles)
//   tail:                 G3(c, the last lag row blocks), [G2(c, half 0) if not yet],
//                         G2(c, last half)
// so each dL row block is read by G3 a few tile-steps after it is written and the
// first half of the chunk by G2 while the second half is produced: the live part
// of the dL chunk stays a fraction of it (with orders 0 / 1 G3(c) / G2(c) run a
// block after G1(c) and read most of dL back from DRAM)
template <bool kPair>
__device__ __forceinline__ void vb_decode_o2(const VbParams& P, int c, int u, VbTile& r) {
  constexpr int TM = VbCfg<kPair>::TM;
  const int vcc = vb_vcc(P, c);
  const int ncol = vb_g1cols(P, vcc);
  const int n2 = ((vcc + TM - 1) / TM) * P.ndw;
  const int L = P.lag, nrb = P.nrb, ndw = P.ndw;
  auto prefix = [&](int rb) { return rb * ncol + max(0, rb - L) * ndw; };
  const int rbg2 = P.h0 - 1 + L;
  const int pos_g2 = (P.nh == 2 && rbg2 < nrb) ? prefix(rbg2 + 1) : -1;
  r.c = c;
  r.h = 0;
  if (pos_g2 >= 0 && u >= pos_g2) {
    if (u < pos_g2 + n2) {
      u -= pos_g2;
      r.type = VB_G2; r.i = u / ndw; r.j = u % ndw;
      return;
    }
    u -= n2;
  }
  const int rows_total = prefix(nrb);
  if (u < rows_total) {
    if (u < L * ncol) {
      r.type = VB_G1; r.i = u / ncol; r.j = u % ncol;
    } else {
      const int v = u - L * ncol;
      const int rb = L + v / (ncol + ndw), w = v % (ncol + ndw);
      if (w < ncol) { r.type = VB_G1; r.i = rb; r.j = w; }
      else { r.type = VB_G3; r.i = rb - L; r.j = w - ncol; }
    }
    return;
  }
  u -= rows_total;
  const int ntail = min(L, nrb);
  if (u < ntail * ndw) {
    r.type = VB_G3; r.i = nrb - ntail + u / ndw; r.j = u % ndw;
    return;
  }
  u -= ntail * ndw;
  if (P.nh == 2 && pos_g2 < 0) {
    if (u < n2) { r.type = VB_G2; r.i = u / ndw; r.j = u % ndw; return; }
    u -= n2;
  }
  r.type = VB_G2; r.h = P.nh - 1; r.i = u / ndw; r.j = u % ndw;
}


template <bool kPair>
__device__ __forceinline__ VbTile vb_decode(const VbParams& P, int t) {
  constexpr int TM = VbCfg<kPair>::TM;
  VbTile r;
  r.c = 0;
  r.h = 0;
  r.k0 = 0;
  if (t < P.fwd_tiles) {
    r.type = VB_G0; r.i = t / P.ntn; r.j = t % P.ntn;   // row-block major
    r.vcc = P.V;
    r.kb_total = P.d / VB_BK;
    return r;
  }
  t -= P.fwd_tiles;
  int lo = 0, hi = P.order == 2 ? P.nchunks - 1 : P.nchunks;   // blocks
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (P.blk_start[mid] <= t) lo = mid; else hi = mid - 1;
  }
  int u = t - P.blk_start[lo];
  r.h = 0;
  r.k0 = 0;
  if (P.order == 2) {
    vb_decode_o2<kPair>(P, lo, u, r);
    r.vcc = vb_vcc(P, r.c);
    if (r.type == VB_G1) r.kb_total = P.d / VB_BK;
    else if (r.type == VB_G3) r.kb_total = (r.vcc + VB_BK - 1) / VB_BK;
    else vb_g2_range<kPair>(P, r.h, r.k0, r.kb_total);
    return r;
  }
  if (lo == 0) {
    r.type = VB_G1; r.c = 0;
  } else {
    const int c = lo - 1;
    const int n3 = P.nrb * P.ndw;
    const int n2 = ((vb_vcc(P, c) + TM - 1) / TM) * P.ndw;
    const bool g2first = P.last_g2_first && c == P.nchunks - 1;
    const int n1 = (P.order == 1 && c + 1 < P.nchunks) ? P.nrb * vb_g1cols(P, vb_vcc(P, c + 1)) : 0;
    if (u < n1) {   // order 1: the next chunk's G1 tiles open the block
      r.type = VB_G1; r.c = c + 1;
    } else {
      u -= n1;
      if (g2first) {
        if (u < n2) { r.type = VB_G2; r.c = c; }
        else { u -= n2; r.type = VB_G3; r.c = c; }
      } else if (u < n3) {
        r.type = VB_G3; r.c = c;
      } else if (u < n3 + n2) {
        u -= n3; r.type = VB_G2; r.c = c;
      } else {   // order 0: the next chunk's G1 tiles close the block
        u -= n3 + n2; r.type = VB_G1; r.c = c + 1;
      }
    }
  }
  r.vcc = vb_vcc(P, r.c);
  if (r.type == VB_G1) {
    const int ncol = vb_g1cols(P, r.vcc);
    r.i = u / ncol; r.j = u % ncol;
    r.kb_total = P.d / VB_BK;
  } else if (r.type == VB_G3) {
    r.i = u / P.ndw; r.j = u % P.ndw;
    r.kb_total = (r.vcc + VB_BK - 1) / VB_BK;
  } else {
    r.i = u / P.ndw; r.j = u % P.ndw;
    r.kb_total = (P.T + VB_BK - 1) / VB_BK;
  }
  return r;
}

// trace record of tile t and CTA rank r (option "vb_trace"), at (2 t + r) * 32:
// [0] smid [1] type << 16 | chunk  [2] / [3] producer globaltimer before / after
// the dependency wait  [4] / [5] MMA clock64 first MMA issued / last commit
// [6] / [7] epilogue warp 0 clock64 accumulator ready / tile done  [8] / [9] MMA
// globaltimer first MMA / last commit  [10] / [11] epilogue globaltimer ready /
// done  [12] epilogue clock64 after its dependency wait  [13] MMA clock64
// accumulator free  [14] MMA cycles spent waiting for full stages
// [16] epilogue warp 0 clock64 when it releases the (last) accumulator
__device__ __forceinline__ long long vb_clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
__device__ __forceinline__ long long vb_gt() {
  long long c;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(c));
  return c;
}
#define VB_TRACE(t, i, val)                                                  \
  do {                                                                       \
    if (P.trace) {                                                           \
      const long long v_ = (val);                                            \
      if (lane == 2) P.trace[((long long)(t) * 2 + rank) * 32 + (i)] = v_;   \
    }                                                                        \
  } while (0)

__device__ __forceinline__ void vb_wait_geq(const unsigned* p, unsigned target) {
  spin_wait_geq(p, target, 64);
}

template <bool kPair>
__device__ __forceinline__ void vb_load(void* dst, const CUtensorMap* m, uint64_t* bar,
                                        uint32_t barc, int c0, int c1, int c2, uint64_t pol) {
  if constexpr (kPair) tma_load_3d_pair_hint(dst, m, barc, c0, c1, c2, pol);
  else tma_load_3d_hint(dst, m, bar, c0, c1, c2, pol);
}
template <bool kPair>
__device__ __forceinline__ void vb_load4(void* dst, const CUtensorMap* m, uint64_t* bar,
                                         uint32_t barc, int c0, int c1, int c2, int c3,
                                         uint64_t pol) {
  if constexpr (kPair) tma_load_4d_pair_hint(dst, m, barc, c0, c1, c2, c3, pol);
  else tma_load_4d_hint(dst, m, bar, c0, c1, c2, c3, pol);
}

// sum over the 32 lanes of each of 32 values: afterwards lane l holds the
// total of column l (a butterfly reduce-scatter, 31 shuffles per lane)
__device__ __forceinline__ float warp_colsum32(float (&v)[32], uint32_t lane) {
#pragma unroll
  for (int half = 16; half >= 1; half >>= 1) {
    const bool upper = (lane & half) != 0;
#pragma unroll
    for (int j = 0; j < half; ++j) {
      // keep the half of the columns this lane will own, send the other half
      const float send = upper ? v[j] : v[j + half];
      const float keep = upper ? v[j + half] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, half);
    }
  }
  return v[0];
}

#if VB_DEBUG_MMA
// Timing-only MMA-issue variants of G1 k-blocks (VbParams::debug; WRONG
// results): bits 8 / 9 two N = 128 / four N = 64 MMAs sharing A (bit 12: the
// two N = 128 chains 256 columns apart), bits 10 / 11 two N = 256 MMAs into both
// accumulators with the same A and B / the A of another stage.  Returns true if
// it issued the k-block.
template <bool kPair>
__device__ __noinline__ bool vb_debug_mma(const VbParams& P, const VbTile& tl, int kb, int s, int acc,
                                          uint32_t tmem_base, uint8_t* smem, int a_mn, int b_mn,
                                          uint64_t ad, uint64_t bd) {
  using Cfg = VbCfg<kPair>;
  if (tl.type != VB_G1) return false;
  const uint32_t a_k16 = a_mn ? 128u : 2u, b_k16 = b_mn ? 128u : 2u;
  const int nsplit = (P.debug & (256 | 4096)) ? 2 : (P.debug & 512) ? 4 : 1;
  const int dual = (P.debug & 1024) ? 1 : (P.debug & 2048) ? 2 : 0;
  if (nsplit == 1 && !dual) return false;
  const uint32_t dcol = tmem_base + acc * VB_BN;
  if (nsplit > 1) {
    const uint32_t qstride = (P.debug & 4096) ? 256u : (uint32_t)(VB_BN / nsplit);
    const uint32_t idn = umma_idesc_bf16(Cfg::TM, VB_BN / nsplit, a_mn, b_mn);
    for (int k = 0; k < VB_BK / 16; ++k)
      for (int q = 0; q < nsplit; ++q) {
        const uint64_t bq = bd + k * b_k16 + (uint32_t)(q * (Cfg::B_BYTES / nsplit)) / 16;
        const uint32_t d = tmem_base + ((acc * VB_BN + q * qstride) & 511u);
        if constexpr (kPair) umma_bf16_pair(d, ad + k * a_k16, bq, idn, (kb > 0 || k > 0) ? 1u : 0u);
        else umma_bf16(d, ad + k * a_k16, bq, idn, (kb > 0 || k > 0) ? 1u : 0u);
      }
    return true;
  }
  const uint32_t idesc = umma_idesc_bf16(Cfg::TM, VB_BN, a_mn, b_mn);
  const uint64_t ado = ad + (uint32_t)(((s + 1) % Cfg::STAGES - s) * Cfg::STAGE) / 16;
  for (int k = 0; k < VB_BK / 16; ++k) {
    const uint32_t accum = (kb > 0 || k > 0) ? 1u : 0u;
    if constexpr (kPair) {
      umma_bf16_pair(dcol, ad + k * a_k16, bd + k * b_k16, idesc, accum);
      umma_bf16_pair(tmem_base + (acc ^ 1) * VB_BN, (dual == 1 ? ad : ado) + k * a_k16,
                     bd + k * b_k16, idesc, accum);
    }
  }
  return true;
}
#endif

template <bool kPair>
__global__ void __launch_bounds__(VB_THREADS, 1) vocab_kernel(const __grid_constant__ VbParams P) {
  using Cfg = VbCfg<kPair>;
  constexpr int TM = Cfg::TM;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* staging = smem + VB_RING;
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + VB_EPI_WARPS * VB_STG_BYTES);
  uint64_t* full = bars;                        // [STAGES]
  uint64_t* empty = full + STAGES;              // [STAGES]
  uint64_t* tfull = empty + STAGES;             // [2]
  uint64_t* tempty = tfull + 2;                 // [2]
  uint64_t* sfull = tempty + 2;                 // [SCHED]
  uint64_t* sempty = sfull + VB_SCHED;          // [SCHED]
  int* sched_tile = reinterpret_cast<int*>(sempty + VB_SCHED);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sched_tile + VB_SCHED);

  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();
  const uint32_t rank = kPair ? cluster_ctarank() : 0;   // 0 = pair leader
  const bool leader = rank == 0;
  constexpr uint32_t kWarpAlloc = 8, kWarpProducer = 10, kWarpMma = 11;
  // shared::cluster address of a barrier in the leader CTA
  auto leader_addr = [&](void* p) -> uint32_t { return mapa_shared(smem_u32(p), 0); };

  if (warp == kWarpProducer && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], Cfg::WARPS_PER_TILE);   // every epilogue warp of the tile
    }
    for (int i = 0; i < VB_SCHED; ++i) {
      mbar_init(&sfull[i], 1);
      // leader: its MMA warp + epilogue warps (+ the peer's producer and epilogue warps)
      mbar_init(&sempty[i], 1 + VB_EPI_WARPS + (kPair ? 1 + VB_EPI_WARPS : 0));
    }
    fence_barrier_init();
    const CUtensorMap* maps[9] = {&P.m_hc_k, &P.m_wo_k, &P.m_dl_k, &P.m_wo_mn, &P.m_dl_mn,
                                  &P.m_hc_mn, &P.m_dl_st, &P.m_dw_st, &P.m_dhc_st};
    for (int i = 0; i < 9; ++i) tma_prefetch_desc(maps[i]);
  }
  if (warp == kWarpAlloc) {
    if constexpr (kPair) tmem_alloc_pair(tmem_slot, 512);
    else tmem_alloc(tmem_slot, 512);
  }
  tc_fence_before();
  if constexpr (kPair) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();
  if (threadIdx.x == 0) pdl_trigger();

  // the scheduler ring: the leader publishes each tile id into both CTAs' rings
  auto ring_read = [&](int& r, uint32_t& rph, bool lane0) -> int {
    if (kPair && !leader) mbar_wait_cluster(&sfull[r], rph);
    else mbar_wait(&sfull[r], rph);
    const int t = sched_tile[r];
    __syncwarp();
    if (lane0 ? lane == 0 : elect_one()) {
      if (kPair && !leader) mbar_arrive_cluster(leader_addr(&sempty[r]));
      else mbar_arrive(&sempty[r]);
    }
    __syncwarp();
    if (++r == VB_SCHED) { r = 0; rph ^= 1; }
    return t;
  };

  if (warp == kWarpProducer) {
    // ---------------- scheduler (leader) + TMA producer (both CTAs).  The
    // whole warp runs the loop, one elected lane issues; the next tile is
    // fetched, published and decoded right after the current tile's first load.
    int s = 0;
    uint32_t ph = 0;
    int r = 0;
    uint32_t rph = 0;
    int t_raw = 0;
    auto fetch = [&]() {
      if (lane == 1) t_raw = atomicAdd(P.tile_counter, 1);
    };
    auto next_tile = [&]() -> int {
      if (!leader) return ring_read(r, rph, false);
      int t = __shfl_sync(0xffffffffu, t_raw, 1);
      if (t >= P.total_tiles) t = -1;
      mbar_wait(&sempty[r], rph ^ 1);
      if (elect_one()) {
        sched_tile[r] = t;
        if constexpr (kPair) {
          st_shared_cluster_u32(mapa_shared(smem_u32(&sched_tile[r]), 1), (uint32_t)t);
          mbar_arrive_cluster(mapa_shared(smem_u32(&sfull[r]), 1));
        }
        mbar_arrive(&sfull[r]);
      }
      __syncwarp();
      if (t >= 0 && !P.claim_late) fetch();
      if (++r == VB_SCHED) { r = 0; rph ^= 1; }
      return t;
    };
    // L2 residency: H_c is re-read by every chunk (evict-last when option
    // bit 0 of P.l2hints), the streaming operands keep the normal policy
    const uint64_t pol_keep = (P.l2hints & 1) ? l2_policy_evict_last() : l2_policy_evict_normal();
    const uint64_t pol_norm = l2_policy_evict_normal();
    if (leader) fetch();
    int t = next_tile();
    VbTile tl{};
    if (t >= 0) tl = vb_decode<kPair>(P, t);
    while (t >= 0) {
      const int buf = tl.c % P.nbuf;
      const int c0 = tl.c * P.Vc;
      if (P.trace) {
        uint32_t sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        VB_TRACE(t, 0, (long long)sm);
        VB_TRACE(t, 1, ((long long)tl.type << 16) | tl.c);
        VB_TRACE(t, 2, vb_gt());
      }
      // operands of G2 / G3 are the dL chunk: wait for the G1 tiles that write it
      if (tl.type == VB_G3) {
        if (lane == 0)
          vb_wait_geq(P.rowdone + (size_t)tl.c * P.nrb + tl.i,
                      (unsigned)(Cfg::WARPS_PER_TILE * ((tl.vcc + VB_BN - 1) / VB_BN)));
        __syncwarp();
        fence_proxy_async_global();
      } else if (tl.type == VB_G2) {
        if (lane == 0) {
          // this tile's TM vocabulary rows: 256-column blocks of G1
          const int cb0 = tl.i * TM / VB_BN, cb1 = ((tl.i + 1) * TM - 1) / VB_BN;
          // ... over the row blocks of its half (order 2 splits the K = T rows)
          const int nrows = P.nh == 1 ? P.nrb : (tl.h == 0 ? P.h0 : P.nrb - P.h0);
          for (int cb = cb0; cb <= cb1 && cb * VB_BN < tl.vcc; ++cb)
            vb_wait_geq(P.coldone + ((size_t)tl.c * P.nh + tl.h) * P.ncolf + cb,
                        (unsigned)(Cfg::WARPS_PER_TILE * nrows));
        }
        __syncwarp();
        fence_proxy_async_global();
      }
      VB_TRACE(t, 3, vb_gt());
      const bool wide = kPair && ((P.wide && (tl.type == VB_G2 || tl.type == VB_G3)) ||
                                  (P.g1wide && tl.type == VB_G1));
      const int arow = tl.i * TM + 128 * rank;            // this CTA's A rows (M)
      const int bcol = tl.j * (wide ? 2 * VB_BN : VB_BN) + Cfg::B_ROWS * rank;  // this CTA's B rows (N)
      const int bcolg = (tl.type == VB_G0 ? 0 : c0) + bcol;
      int t_nxt = -1;
      VbTile tl_nxt{};
      for (int kb = 0; kb < tl.kb_total; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        if (elect_one()) {
          uint8_t* sA = smem + s * Cfg::STAGE;
          uint8_t* sB = sA + Cfg::A_BYTES;
          const uint32_t barc = kPair ? leader_addr(&full[s]) : 0u;
          // debug bits 4 / 5 (timing only): skip the B / A operand loads
          // bits 13 / 14: skip the operand loads of G2 / G3 tiles only
          const bool skip_t = (tl.type == VB_G2 && (P.debug & 8192)) || (tl.type == VB_G3 && (P.debug & 16384));
          const bool ldA = !(P.debug & 32) && !skip_t, ldB = !(P.debug & 16) && !skip_t;
          const int nb = (Cfg::S3 && wide) ? 2 : 1;   // B blocks in this stage
          if (leader)
            mbar_arrive_expect_tx(&full[s], ((ldA ? Cfg::A_BYTES : 0) + (ldB ? nb * Cfg::B_BYTES : 0)) * Cfg::CTAS);
          const int k0 = kb * VB_BK;
#if VB_DEBUG_MMA
          if (tl.type == VB_G1 && (P.debug & 64)) {
            if (ldA) vb_load<kPair>(sA, &P.m_hc_k, &full[s], barc, k0, arow, 0, pol_keep);
            if (ldB) vb_load4<kPair>(sB, &P.m_wo_mn, &full[s], barc, 0, c0 + k0, (bcol % P.d) / 64, 0, pol_norm);
          } else
#endif
          if (tl.type == VB_G1 || tl.type == VB_G0) {
            if (ldA) vb_load<kPair>(sA, &P.m_hc_k, &full[s], barc, k0, arow, 0, pol_keep);
            if (ldB) vb_load<kPair>(sB, &P.m_wo_k, &full[s], barc, k0, bcolg, 0, pol_norm);
          } else if (tl.type == VB_G3) {
            if (ldA) vb_load<kPair>(sA, &P.m_dl_k, &full[s], barc, k0, arow, buf, pol_norm);
            if (ldB) vb_load4<kPair>(sB, &P.m_wo_mn, &full[s], barc, 0, c0 + k0, bcol / 64, 0, pol_norm);
          } else {
            if (ldA) vb_load4<kPair>(sA, &P.m_dl_mn, &full[s], barc, 0, tl.k0 + k0, arow / 64, buf, pol_norm);
            if (ldB) vb_load4<kPair>(sB, &P.m_hc_mn, &full[s], barc, 0, tl.k0 + k0, bcol / 64, 0, pol_keep);
          }
          if (Cfg::S3 && wide && ldB) {   // the tile's B columns [256, 512) in the same stage
            uint8_t* sB2 = sB + Cfg::B_BYTES;
            if (tl.type == VB_G1)
              vb_load<kPair>(sB2, &P.m_wo_k, &full[s], barc, k0, bcolg + VB_BN, 0, pol_norm);
            else if (tl.type == VB_G3)
              vb_load4<kPair>(sB2, &P.m_wo_mn, &full[s], barc, 0, c0 + k0, (bcol + VB_BN) / 64, 0, pol_norm);
            else
              vb_load4<kPair>(sB2, &P.m_hc_mn, &full[s], barc, 0, tl.k0 + k0, (bcol + VB_BN) / 64, 0, pol_keep);
          }
        }
        __syncwarp();
        if (++s == STAGES) { s = 0; ph ^= 1; }
        if (wide && !Cfg::S3) {
          // the k-block's second stage: B columns [256, 512) of the tile (its A region unused)
          mbar_wait(&empty[s], ph ^ 1);
          if (elect_one()) {
            uint8_t* sB = smem + s * Cfg::STAGE + Cfg::A_BYTES;
            const uint32_t barc = kPair ? leader_addr(&full[s]) : 0u;
            const bool skip_t = (tl.type == VB_G2 && (P.debug & 8192)) || (tl.type == VB_G3 && (P.debug & 16384));
            if (leader) {
              if (skip_t) mbar_arrive(&full[s]);
              else mbar_arrive_expect_tx(&full[s], Cfg::B_BYTES * Cfg::CTAS);
            }
            const int k0 = kb * VB_BK;
            if (skip_t) {
            } else if (tl.type == VB_G1)
              vb_load<kPair>(sB, &P.m_wo_k, &full[s], barc, k0, bcolg + VB_BN, 0, pol_norm);
            else if (tl.type == VB_G3)
              vb_load4<kPair>(sB, &P.m_wo_mn, &full[s], barc, 0, c0 + k0, (bcol + VB_BN) / 64, 0, pol_norm);
            else
              vb_load4<kPair>(sB, &P.m_hc_mn, &full[s], barc, 0, tl.k0 + k0, (bcol + VB_BN) / 64, 0, pol_keep);
          }
          __syncwarp();
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        if (P.claim_late) {
          // claim the next tile only when this one is nearly issued: a tile is
          // never queued behind a long one on a busy pair (order 2's short
          // dependency distances need it)
          if (leader && kb == max(0, tl.kb_total - P.claim_late)) fetch();
        } else if (kb == 0) {
          t_nxt = next_tile();
          if (t_nxt >= 0) tl_nxt = vb_decode<kPair>(P, t_nxt);
        }
      }
      if (P.claim_late) {
        t_nxt = next_tile();
        if (t_nxt >= 0) tl_nxt = vb_decode<kPair>(P, t_nxt);
      }
      t = t_nxt;
      tl = tl_nxt;
    }
  } else if (warp == kWarpMma) {
    // ---------------- MMA issuer: the pair leader's warp runs the loop, one
    // elected lane issues for both CTAs (the uniform datapath: a lane-0-only
    // loop measured 988 instead of 751 cycles per G1 k-block).  The loop is
    // kept lean -- descriptors are templates plus the stage address -- because
    // its issue rate is on the critical path (extra code in it measured 1000
    // cycles per G1 k-block)
    if (leader) {
      int s = 0;
      uint32_t ph = 0;
      int r = 0;
      uint32_t rph = 0;
      int acc = 0;
      uint32_t aph = 0;
      auto ring_read1 = [&]() -> int { return ring_read(r, rph, false); };
      const uint32_t smem16 = smem_u32(smem) >> 4;   // descriptor start-address units
      constexpr uint32_t kStage16 = Cfg::STAGE >> 4, kA16 = Cfg::A_BYTES >> 4;
      int t = ring_read1();
      while (t >= 0) {
        const VbTile tl = vb_decode<kPair>(P, t);
        const int a_mn = tl.type == VB_G2 ? 1 : 0;
#if VB_DEBUG_MMA
        const int b_mn = (tl.type == VB_G3 || tl.type == VB_G2 || (tl.type == VB_G1 && (P.debug & 64))) ? 1 : 0;
#else
        const int b_mn = (tl.type == VB_G3 || tl.type == VB_G2) ? 1 : 0;
#endif
        const uint32_t idesc = umma_idesc_bf16(TM, VB_BN, a_mn, b_mn);
        // descriptor templates (start address 0): + (stage address >> 4) + k-step
        const uint64_t ad0 = umma_sdesc(0, a_mn ? 8192u : 16u, 1024);
        const uint64_t bd0 = umma_sdesc(0, b_mn ? 8192u : 16u, 1024);
        const uint32_t a_k16 = a_mn ? (2048u >> 4) : (32u >> 4);
        const uint32_t b_k16 = b_mn ? (2048u >> 4) : (32u >> 4);
        const int kb_read = tl.kb_total > 1 ? 1 : 0;
        const bool wide = kPair && ((P.wide && (tl.type == VB_G2 || tl.type == VB_G3)) ||
                                    (P.g1wide && tl.type == VB_G1));
        int t_nxt = -1;
        // a wide tile takes both accumulators: slot acc, then the next one
        const int acc2 = acc ^ 1;
        const uint32_t aph2 = acc2 == 0 ? (aph ^ 1) : aph;
        mbar_wait(&tempty[acc], aph ^ 1);
        if (wide) mbar_wait(&tempty[acc2], aph2 ^ 1);
        tc_fence_after();
        VB_TRACE(t, 13, vb_clk());
        long long wait_cyc = 0;
        const uint32_t dcol = tmem_base + acc * VB_BN;
        const uint32_t dcol2 = tmem_base + acc2 * VB_BN;
        for (int kb = 0; kb < tl.kb_total; ++kb) {
          int s2 = s;
          uint32_t ph2 = ph;
          if (wide && !Cfg::S3 && ++s2 == STAGES) { s2 = 0; ph2 ^= 1; }
          if (P.trace) {
            const long long w0 = vb_clk();
            mbar_wait(&full[s], ph);
            if (wide && !Cfg::S3) mbar_wait(&full[s2], ph2);
            wait_cyc += vb_clk() - w0;
          } else {
            mbar_wait(&full[s], ph);
            if (wide && !Cfg::S3) mbar_wait(&full[s2], ph2);
          }
          tc_fence_after();
          const uint32_t sa16 = smem16 + (uint32_t)s * kStage16;
          const uint64_t ad = ad0 + sa16;
          const uint64_t bd = bd0 + sa16 + kA16;
          const uint64_t bd2 = Cfg::S3 ? bd + (uint32_t)(Cfg::B_BYTES >> 4)
                                       : bd0 + smem16 + (uint32_t)s2 * kStage16 + kA16;
          if (elect_one()) {
#if VB_DEBUG_MMA
            if (vb_debug_mma<kPair>(P, tl, kb, s, acc, tmem_base, smem, a_mn, b_mn, ad, bd)) {
            } else
#endif
            {
#pragma unroll
              for (int k = 0; k < VB_BK / 16; ++k) {
                const uint32_t accum = (kb > 0 || k > 0) ? 1u : 0u;
                if constexpr (kPair) {
                  umma_bf16_pair(dcol, ad + k * a_k16, bd + k * b_k16, idesc, accum);
                  if (wide) umma_bf16_pair(dcol2, ad + k * a_k16, bd2 + k * b_k16, idesc, accum);
                } else {
                  umma_bf16(dcol, ad + k * a_k16, bd + k * b_k16, idesc, accum);
                }
              }
            }
            if constexpr (kPair) {
              umma_commit_pair(&empty[s]);
              if (wide && !Cfg::S3) umma_commit_pair(&empty[s2]);
            } else {
              umma_commit(&empty[s]);
            }
          }
          __syncwarp();
          if (kb == 0) {
            VB_TRACE(t, 4, vb_clk());
            VB_TRACE(t, 8, vb_gt());
          }
          s = s2;
          ph = ph2;
          if (++s == STAGES) { s = 0; ph ^= 1; }
          if (kb == kb_read && !P.claim_late) t_nxt = ring_read1();
        }
        if (elect_one()) {
          if constexpr (kPair) {
            umma_commit_pair(&tfull[acc]);
            if (wide) umma_commit_pair(&tfull[acc2]);
          } else {
            umma_commit(&tfull[acc]);
          }
        }
        __syncwarp();
        if (P.claim_late) t_nxt = ring_read1();   // after the commit: the epilogue starts first
        VB_TRACE(t, 5, vb_clk());
        VB_TRACE(t, 9, vb_gt());
        VB_TRACE(t, 14, wait_cyc);
        if (++acc == 2) { acc = 0; aph ^= 1; }
        if (wide && ++acc == 2) { acc = 0; aph ^= 1; }
        t = t_nxt;
      }
    }
    __syncwarp();
  } else if (warp == 8 || warp == 9) {
    // ---------------- LSE (Eq. 6) of row blocks p, p + pairs, ... (pair p):
    // this CTA's 128 rows, two per thread, once the row block's G0 tiles have
    // stored their partials; the partials are slot-major, so a warp's loads
    // are 256 contiguous bytes
    const int tid = (warp - 8) * 32 + lane;
    const int pid = blockIdx.x / Cfg::CTAS, npairs = gridDim.x / Cfg::CTAS;
    double* red = reinterpret_cast<double*>(bars + 48);   // [2] (spare words of the barrier region)
    for (int rb = pid; P.fwd_tiles > 0 && rb < P.nrb; rb += npairs) {
      if (lane == 0) vb_wait_geq(P.g0done + rb, (unsigned)(4 * Cfg::CTAS * P.ntn));
      __syncwarp();
      const int rbase = rb * TM + 128 * rank;
      double wsum = 0.0;
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        const int row = rbase + tid + 64 * half;
        if (row >= P.T) continue;
        float mx = -INFINITY, sm = 0.f;
        int k = 0;
        for (; k + 16 <= P.ntn; k += 16) {
          float2 p2[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) p2[u] = __ldcg(P.part + (long long)(k + u) * P.T + row);
          float bm = p2[0].x;
#pragma unroll
          for (int u = 1; u < 16; ++u) bm = fmaxf(bm, p2[u].x);
          const float nm = fmaxf(mx, bm);
          if (nm == -INFINITY) continue;
          float bs = 0.f;
#pragma unroll
          for (int u = 0; u < 16; ++u) bs += p2[u].y * ex2_mufu((p2[u].x - nm) * kLog2e);
          sm = sm * ex2_mufu((mx - nm) * kLog2e) + bs;
          mx = nm;
        }
        for (; k < P.ntn; ++k) {
          const float2 p2 = __ldcg(P.part + (long long)k * P.T + row);
          const float nm = fmaxf(mx, p2.x);
          if (nm == -INFINITY) continue;
          sm = sm * ex2_mufu((mx - nm) * kLog2e) + p2.y * ex2_mufu((p2.x - nm) * kLog2e);
          mx = nm;
        }
        const float lse = mx + __logf(sm);
        const bool valid = (row % P.N) < P.tgt_len[row / P.N];
        const float nll = valid ? lse - __ldcg(P.tgt_logit + row) : 0.f;
        P.lse[row] = lse;
        P.nll[row] = nll;
        P.rowscale[row] = valid ? P.loss_scale : 0.f;
        wsum += (double)nll;
      }
      // this CTA's NLL sum in a fixed order (lane tree, then warp 8 + warp 9)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
      if (lane == 0) red[warp - 8] = wsum;
      named_bar_sync(6, 64);   // (also: every lse of the CTA's rows is written)
      if (warp == 8 && lane == 0) {
        P.blockpart[rb * Cfg::CTAS + rank] = red[0] + red[1];
        __threadfence();
        const unsigned prev = atomicAdd(P.g5count, 1u);
        if (prev == (unsigned)(P.nrb * Cfg::CTAS) - 1) {
          // the last row block: the loss, summed in block order (deterministic)
          __threadfence();
          double tot = 0.0;
          for (int i = 0; i < P.nrb * Cfg::CTAS; ++i)
            tot += reinterpret_cast<volatile double*>(P.blockpart)[i];
          *P.loss = (float)(tot * (double)P.loss_scale);
        }
      }
      if (lane == 0) {
        __threadfence();
        red_release_gpu_add(P.lsedone + rb, 1u);
      }
      named_bar_sync(6, 64);   // red[] reused by the next row block
    }
  } else if (warp < VB_EPI_WARPS) {
    // ---------------- epilogue (8 warps per CTA): this CTA's 128 rows of the tile
    const uint32_t q = warp & 3;        // TMEM lane quarter: rows 32q..32q+31 of this CTA's 128
    const uint32_t h = warp >> 2;       // column half of the 256-wide tile
    uint8_t* stg_base = staging + warp * VB_STG_BYTES;
    uint32_t stg_seq = 0;   // staged store groups of this warp (buffer = stg_seq & 1)
    const uint32_t stg_base_u = smem_u32(stg_base);
    const uint32_t swz = lane & 7;
    // l2hints bit 2: the dL chunk stores stay in L2 until its G2 / G3 readers come
    const uint64_t pol_dl = l2_policy_evict_last();
    int r = 0;
    uint32_t rph = 0;
    int acc = 0;
    uint32_t aph = 0;
    for (;;) {
      const int t = ring_read(r, rph, true);
      if (t < 0) break;
      const VbTile tl = vb_decode<kPair>(P, t);
      const int buf = tl.c % P.nbuf;
      const int c0 = tl.c * P.Vc;
      const int row0 = tl.i * TM + 128 * rank + q * 32;   // problem row of lane 0
      const int colh = tl.j * VB_BN + h * 128;           // problem column of this warp's first
      const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * VB_BN + h * 128;
      if (tl.type == VB_G0) {
        // ---- Eq. 5 forward: (max, sum exp) of this warp's 128 columns per row,
        // and the target logit when the row's target falls in them
        const int row = row0 + lane;
        const bool row_ok = row < P.T;
        const int yl = row_ok ? P.tgt[row] - colh : -1;
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        if (warp == 0) {
          VB_TRACE(t, 6, vb_clk());
          VB_TRACE(t, 10, vb_gt());
          VB_TRACE(t, 12, vb_clk());
        }
        const int nvalid = P.V - colh;
        float m = -INFINITY, ssum = 0.f, tval = 0.f;
        bool has_t = false;
        uint32_t raw[32];
        tmem_ld32_issue(taddr, raw);
        tmem_ld_wait_regs(raw);
#pragma unroll 1
        for (int cc = 0; cc < 4; ++cc) {
          if (cc * 32 >= nvalid) break;
          float v[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(raw[e]);
          if (cc < 3 && (cc + 1) * 32 < nvalid) tmem_ld32_issue(taddr + (cc + 1) * 32, raw);
          const int nv = nvalid - cc * 32;
          if (P.bias) add_bias32<__nv_bfloat16>(P.bias, colh + cc * 32, nv, v);
          float cm;
          if (nv >= 32) {   // sm_100 three-input max: 16 FMNMX3 for 32 values
            float a = fmax3_f(v[0], v[1], v[2]), b = fmax3_f(v[3], v[4], v[5]);
#pragma unroll
            for (int j = 6; j < 30; j += 4) {
              a = fmax3_f(a, v[j], v[j + 1]);
              b = fmax3_f(b, v[j + 2], v[j + 3]);
            }
            cm = fmax3_f(a, b, fmaxf(v[30], v[31]));
          } else {
            cm = -INFINITY;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < nv) cm = fmaxf(cm, v[j]);
          }
          const float nm = fmaxf(m, cm);
          const float nml = nm * kLog2e;
          float sacc = ssum * ex2_mufu(fmaf(m, kLog2e, -nml));
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < nv) sacc += ex2_mufu(fmaf(v[j], kLog2e, -nml));
          ssum = sacc;
          m = nm;
          const int ycc = yl - cc * 32;
          if ((unsigned)ycc < 32u && ycc < nv) {
#pragma unroll
            for (int j = 0; j < 32; ++j) tval = (j == ycc) ? v[j] : tval;
            has_t = true;
          }
          if (cc < 3 && (cc + 1) * 32 < nvalid) tmem_ld_wait_regs(raw);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (kPair && !leader) mbar_arrive_cluster(leader_addr(&tempty[acc]));
          else mbar_arrive(&tempty[acc]);
        }
        if (warp == 0) VB_TRACE(t, 16, vb_clk());
        if (row_ok && has_t) P.tgt_logit[row] = tval;
        // the two column halves of a row merge through shared memory (warp q
        // + 4 hands its (max, sum) to warp q; named barrier 2 + q, 64 threads)
        float2* xchg = reinterpret_cast<float2*>(staging + q * VB_STG_BYTES) + lane;
        if (h == 1) *xchg = make_float2(m, ssum);
        named_bar_sync(2 + q, 64);
        if (h == 0) {
          const float2 o = *xchg;
          const float nm = fmaxf(m, o.x);   // (-inf, 0) for a half past the vocabulary
          if (nm != -INFINITY) ssum = ssum * ex2_mufu((m - nm) * kLog2e) + o.y * ex2_mufu((o.x - nm) * kLog2e);
          if (row_ok) P.part[(long long)tl.j * P.T + row] = make_float2(nm, ssum);
          __syncwarp();   // (orders the warp's stores before lane 0's release)
          if (lane == 0) red_release_gpu_add(P.g0done + tl.i, 1u);
        }
        named_bar_sync(2 + q, 64);   // xchg may be overwritten by the next tile
        __syncwarp();
      } else if (tl.type == VB_G1) {
        // ---- dL = rs softmax - rs onehot (bf16) into dL buffer `buf`.  The
        // row's statistics are read before the accumulator wait (latency hidden
        // under the tile's MMAs).
        const int row = row0 + lane;
        if (warp == 0) VB_TRACE(t, 15, vb_gt());
        if (P.fwd_tiles > 0) {   // lse of this row block comes from this launch's LSE warps
          if (lane == 0) vb_wait_geq(P.lsedone + tl.i, (unsigned)(2 * Cfg::CTAS));
          __syncwarp();
        }
        float c2 = -1000.f, fix = 0.f;
        int yl0 = -1;   // target column relative to the chunk's first column
        if (row < P.T) {
          const float rs = __ldcg(P.rowscale + row);   // written by this launch's LSE warps
          if (rs > 0.f) {
            const float ls = __ldcg(P.lse + row);
            c2 = __log2f(rs) - ls * kLog2e;
            fix = rs * (__expf(__ldcg(P.tgt_logit + row) - ls) - 1.f);
            yl0 = P.tgt[row] - c0;
          }
        }
        // the buffer rows are free once chunk c - NB's G2 / G3 tiles have loaded
        // them (per row half with the order-2 split: its G3 row blocks and G2 tiles)
        if (tl.c >= P.nbuf) {
          const int cp = tl.c - P.nbuf;
          const int hh = (P.nh == 2 && tl.i >= P.h0) ? 1 : 0;
          const int rows = P.nh == 1 ? P.nrb : (hh == 0 ? P.h0 : P.nrb - P.h0);
          const unsigned need = (unsigned)(Cfg::CTAS * P.ndt *
                                           (rows + ((vb_vcc(P, cp) + TM - 1) / TM)));
          if (lane == 0) vb_wait_geq(P.consumed + 2 * cp + hh, need);
          __syncwarp();
          fence_proxy_async_global();
        }
        if (warp == 0) VB_TRACE(t, 12, vb_gt());   // after the lse / buffer waits
        // a wide G1 tile (option vb_g1wide) is 512 columns: two 256-column
        // halves, one per accumulator, drained in turn
        const int nhalf1 = (kPair && P.g1wide) ? 2 : 1;
#pragma unroll 1
        for (int half = 0; half < nhalf1; ++half) {
        if (half > 0 && ++acc == 2) { acc = 0; aph ^= 1; }
        const int colh = (tl.j * nhalf1 + half) * VB_BN + h * 128;
        const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * VB_BN + h * 128;
        const int yl = yl0 >= 0 ? yl0 - colh : -1;
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        if (warp == 0) {
          VB_TRACE(t, 6, vb_clk());
          VB_TRACE(t, 10, vb_gt());
        }
        const int nvalid = tl.vcc - colh;   // valid columns of this warp's 128 (may be <= 0)
        uint32_t raw[32];
        if (!(P.debug & 128)) {
          tmem_ld32_issue(taddr, raw);
          tmem_ld_wait_regs(raw);
        }
#pragma unroll 1
        for (int cc = 0; cc < 4 && !(P.debug & 128); ++cc) {
          // one store group per two 32-column chunks (32 rows x 64 bf16 = 4 KB)
          const uint32_t sbuf = VB_STG_DB ? ((stg_seq & 1u) << 12) : 0u;
          const uint32_t stg = stg_base_u + sbuf;
          uint8_t* stg_p = stg_base + sbuf;
          float v[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(raw[e]);
          if (P.bias && nvalid - cc * 32 > 0)
            add_bias32<__nv_bfloat16>(P.bias, c0 + colh + cc * 32, nvalid - cc * 32, v);
          const int ycc = yl - cc * 32;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            float x = (P.debug & 2) ? v[e] : ex2_mufu(fmaf(v[e], kLog2e, c2));
            if (nvalid - cc * 32 < 32 && cc * 32 + e >= nvalid) x = 0.f;   // past the vocabulary
            v[e] = x;
          }
          if (P.db_part) {
            // F_c bias (NEXT-1): column sums of dL over this warp's 32 rows,
            // the target column holding rs (p_y - 1)
            float cs[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) cs[e] = (e == ycc) ? fix : v[e];
            const float colsum = warp_colsum32(cs, lane);
            const int gcol = c0 + colh + cc * 32 + (int)lane;
            if (cc * 32 + (int)lane < nvalid && row0 < P.T)
              P.db_part[(long long)(row0 >> 5) * P.V + gcol] = colsum;
          }
          uint32_t w[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            __nv_bfloat162 h2 = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
            w[e] = *reinterpret_cast<uint32_t*>(&h2);
          }
          // next chunk's accumulator columns load while this one is staged
          if (cc < 3) tmem_ld32_issue(taddr + (cc + 1) * 32, raw);
          if ((cc & 1) == 0) {
            if (lane == 0) {
              if (VB_STG_DB) bulk_wait_read1();   // the other buffer may still be read
              else bulk_wait_read0();
            }
            __syncwarp();
          }
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const uint32_t gi = (cc & 1) * 4 + g;
            st_shared_v4(stg + lane * 128 + ((gi ^ swz) << 4), w[4 * g], w[4 * g + 1],
                         w[4 * g + 2], w[4 * g + 3]);
          }
          if ((unsigned)ycc < 32u) {   // the -onehot term: target column holds rs (p_y - 1)
            const uint32_t gi = (cc & 1) * 4 + (ycc >> 3);
            st_shared_u16(stg + lane * 128 + ((gi ^ swz) << 4) + (ycc & 7) * 2,
                          __bfloat16_as_ushort(__float2bfloat16_rn(fix)));
          }
          if (cc & 1) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0 && !(P.debug & 1)) {
              if (P.l2hints & 4)
                tma_store_3d_hint(&P.m_dl_st, stg_p, colh + (cc - 1) * 32, row0, buf, pol_dl);
              else
                tma_store_3d(&P.m_dl_st, stg_p, colh + (cc - 1) * 32, row0, buf);
              bulk_commit();
            }
            ++stg_seq;
          }
          if (cc < 3) tmem_ld_wait_regs(raw);
        }
        // accumulator drained: the next tile's MMAs may use it
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (kPair && !leader) mbar_arrive_cluster(leader_addr(&tempty[acc]));
          else mbar_arrive(&tempty[acc]);
        }
        if (warp == 0) VB_TRACE(t, 16, vb_clk());
        // publish: this warp's 32 x 128 piece of dL_c is in memory
        if (lane == 0) {
          if (!(P.debug & 8)) bulk_wait0();
          fence_proxy_async_global();
          const int hh = (P.nh == 2 && tl.i >= P.h0) ? 1 : 0;
          const int cb = tl.j * nhalf1 + half;   // 256-column block of the chunk
          if (cb * VB_BN < tl.vcc) {   // (a wide tile's second half may lie past the chunk)
            red_release_gpu_add(P.rowdone + (size_t)tl.c * P.nrb + tl.i, 1u);
            red_release_gpu_add(P.coldone + ((size_t)tl.c * P.nh + hh) * P.ncolf + cb, 1u);
          }
        }
        __syncwarp();
        }   // half
      } else {
        // ---- fp32 output: dW_out[c] rows (G2) or dHc (G3; chunk 0 stores, the
        // later chunks reduce-add in chunk order); a wide tile is drained as two
        // 256-column halves, one per accumulator
        const bool g3 = tl.type == VB_G3;
        const bool wide = kPair && P.wide;
        const int nhalf = wide ? 2 : 1;
#pragma unroll 1
        for (int half = 0; half < nhalf; ++half) {
          if (half > 0 && ++acc == 2) { acc = 0; aph ^= 1; }
          const int nt = tl.j * nhalf + half;                // 256-column tile of d
          const int colh = nt * VB_BN + h * 128;
          const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * VB_BN + h * 128;
          const int ncols = min(128, P.d - colh);
          unsigned* dhc_ctr = P.dhcdone + (size_t)tl.i * P.ndt + nt;
          mbar_wait(&tfull[acc], aph);
          tc_fence_after();
          if (warp == 0) {
            VB_TRACE(t, 6, vb_clk());
            VB_TRACE(t, 10, vb_gt());
          }
          if (warp == 0 && lane == 0) {
            // every MMA of the tile has completed, so its dL operand has been read
            fence_proxy_async_global();
            const int hh = P.nh == 1 ? 0 : g3 ? (tl.i >= P.h0 ? 1 : 0) : tl.h;
            red_release_gpu_add(P.consumed + 2 * tl.c + hh, 1u);
          }
          if (g3 && tl.c > 0) {
            if (lane == 0) vb_wait_geq(dhc_ctr, (unsigned)(Cfg::WARPS_PER_TILE * tl.c));
            __syncwarp();
            fence_proxy_async_global();
          }
          // order 2, G2 of the second row half: reduce-add onto the first half's
          // stores of the same tile (fixed order, deterministic)
          const bool g2_first = !g3 && P.nh == 2 && tl.h == 0;
          const bool g2_second = !g3 && P.nh == 2 && tl.h == 1;
          unsigned* g2p_ctr = P.g2part + (size_t)tl.c * P.n2max + tl.i * P.ndw + tl.j;
          if (g2_second && half == 0) {
            if (lane == 0) vb_wait_geq(g2p_ctr, (unsigned)(Cfg::WARPS_PER_TILE * nhalf));
            __syncwarp();
            fence_proxy_async_global();
          }
          if (warp == 0) VB_TRACE(t, 12, vb_clk());
          // dW_out is not read again here (the first half's partials are, by the second)
          const uint64_t pol = g2_first ? l2_policy_evict_last() : l2_policy_evict_first();
          const uint64_t pol_dhc = (P.l2hints & 2) ? l2_policy_evict_last() : l2_policy_evict_normal();
#pragma unroll 1
          for (int cc = 0; cc < 4; ++cc) {
            if (cc * 32 >= ncols) break;
            const uint32_t sbuf = VB_STG_DB ? ((stg_seq & 1u) << 12) : 0u;
            const uint32_t stg = stg_base_u + sbuf;
            uint8_t* stg_p = stg_base + sbuf;
            float v[32];
            tmem_ld32(taddr + cc * 32, v);
            if (lane == 0) {
              if (VB_STG_DB) bulk_wait_read1();   // the other buffer may still be read
              else bulk_wait_read0();
            }
            __syncwarp();
#pragma unroll
            for (int g = 0; g < 8; ++g)
              st_shared_v4(stg + lane * 128 + ((g ^ swz) << 4), __float_as_uint(v[4 * g]),
                           __float_as_uint(v[4 * g + 1]), __float_as_uint(v[4 * g + 2]),
                           __float_as_uint(v[4 * g + 3]));
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0 && !(P.debug & 4)) {
              if (g2_second)
                tma_reduce_add_2d_hint(&P.m_dw_st, stg_p, colh + cc * 32, c0 + row0, pol);
              else if (!g3)
                tma_store_2d_hint(&P.m_dw_st, stg_p, colh + cc * 32, c0 + row0, pol);
              else if (tl.c == 0)
                tma_store_2d_hint(&P.m_dhc_st, stg_p, colh + cc * 32, row0, pol_dhc);
              else
                tma_reduce_add_2d_hint(&P.m_dhc_st, stg_p, colh + cc * 32, row0, pol_dhc);
              bulk_commit();
            }
            ++stg_seq;
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (kPair && !leader) mbar_arrive_cluster(leader_addr(&tempty[acc]));
            else mbar_arrive(&tempty[acc]);
          }
          if (warp == 0) VB_TRACE(t, 16, vb_clk());
          if (lane == 0) {
            if (!(P.debug & 8)) bulk_wait0();
            fence_proxy_async_global();
            red_release_gpu_add(g3 ? dhc_ctr : g2_first ? g2p_ctr : P.g2done + tl.c, 1u);
          }
          __syncwarp();
        }
      }
      if (warp == 0) {
        VB_TRACE(t, 7, vb_clk());
        VB_TRACE(t, 11, vb_gt());
      }
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  if constexpr (kPair) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  if (warp == kWarpAlloc) {
    if constexpr (kPair) tmem_dealloc_pair(tmem_base, 512);
    else tmem_dealloc(tmem_base, 512);
  }
}

// Comm-stream helper: waits until the G2 tiles of chunks [c_lo, c_hi) have
// stored their dW_out rows (one thread; it runs beside the persistent launch
// on an SM it leaves free), so the allreduce enqueued after it starts early.
// `per_tile` = epilogue warps per G2 tile, `tm` = its vocabulary rows.
__global__ void vb_wait_g2_kernel(const unsigned* __restrict__ g2done, int c_lo, int c_hi, int Vc,
                                  int V, int ndt, int per_tile, int tm) {
  if (threadIdx.x != 0) return;
  for (int c = c_lo; c < c_hi; ++c) {
    const int vcc = min(Vc, V - c * Vc);
    vb_wait_geq(g2done + c, (unsigned)(per_tile * ndt * ((vcc + tm - 1) / tm)));
  }
  __threadfence();
}

// db_out[v] = sum over the 32-row groups g of db_part[g][v] (fixed order)
__global__ void __launch_bounds__(256) db_final_kernel(const float* __restrict__ db_part, int groups,
                                                       int V, float* __restrict__ db_out) {
  pdl_wait();
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  float s = 0.f;
  for (int g = 0; g < groups; ++g) s += db_part[(long long)g * V + v];
  db_out[v] = s;
}

}  // namespace attnsm
