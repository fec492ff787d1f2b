// tc_collectives.cu -- B200 (sm_100a) tensor-core segmented reduction and
// scan (arXiv 1811.09736), behind the C ABI in include/tc_collectives.h.
//
// Design (DESIGN.md has the full story):
//
//  * Data view.  The fp16 input is a row-major matrix X[R x 64] (one row =
//    128 B = one SW128 swizzle atom).  A tile is 128 consecutive rows
//    (8192 elements, 16 KB, contiguous in HBM) loaded by one TMA box into a
//    multi-stage shared-memory ring.  Rows past n are zero-filled by TMA;
//    the ragged last row (n % 64 elements) is patched in the epilogue.
//
//  * Tensor-core formulation (the paper's "reduction = P.A.Q, scan = A.U +
//    L.(carries).U").  With granule g = gcd(seg, 64) and GR = 64/g granules
//    per row, one tcgen05.mma chain (M=128, K=64 as 4 x K16) computes
//        reduce: D[128 x N] = X_tile . B_g   (B_g[k][j] = [k/g == j])
//                -> D[r][j] = sum of granule j of row r   (the A.Q step)
//        scan:   D[128 x 64] = X_tile . U_g  (U_g block-diagonal upper-
//                triangular ones with g x g blocks) -> in-granule inclusive
//                prefix sums of every row            (the A.U step)
//    with fp16 operands from SMEM descriptors and fp32 accumulators in TMEM.
//    The P-side / L-side combine across granules, rows, tiles and CTAs is
//    the carry chain, specialised by how segments align with the tiling:
//        MODE_LOCAL    seg == g (divides 64): no carries at all
//        MODE_ROWS     seg = 64*2^k <= 8192: aligned row groups (shuffles)
//        MODE_TILES    seg = 8192*k: whole tiles, CTA-sequential fp64 carry
//        MODE_GENERAL  anything else: segmented (value, flag) pair scan
//        MODE_CHUNK    scan of huge segments / full scan / scan with a
//                      carry-in: L2-resident chunked reduce-then-scan in ONE
//                      kernel (see below)
//    Reductions and bounded-segment scans give every CTA one contiguous
//    tile range; a reduce combines the segments cut by range boundaries in
//    a deterministic last-CTA fixup, a scan recomputes the carry entering
//    its range from the (< seg) preceding elements.
//
//  * MODE_CHUNK (the paper's grid scan, scan.py:249-310, as a single pass
//    over HBM).  The input is cut into chunks of Gc x K tiles; CTA c owns
//    unit (j, c) = K consecutive tiles of chunk j.  Each tile is loaded and
//    multiplied once; its X.U result stays in TMEM (8 tile slots = all 512
//    columns) while the epilogue walks A(0), A(1), O(0), A(2), O(1), ...:
//    A(j) reads the row totals of unit j and publishes the unit's segmented
//    aggregate (value, has-segment-start) with a release flag; O(j), one
//    unit later, reads the same TMEM slots again and writes the prefix sums
//    seeded with the value entering the unit.  That value comes from a
//    dedicated prefix warp which composes, in fixed unit order and fp64,
//    the aggregates of every earlier unit (all of the earlier chunks, the
//    lower CTAs of this chunk) -- no serial chain between CTAs, and its
//    spin-waits overlap the epilogue.  HBM traffic is the minimal 2 + o
//    bytes/element; cooperative launch keeps the spin-waits deadlock-free.
//
//  * Warp specialisation (192 threads, persistent grid, 2 CTAs/SM): warp 0
//    = TMA producer, warp 1 = TMEM allocator + single-thread MMA issuer,
//    warps 2..5 = epilogue (TMEM lane quadrant = warp % 4).  mbarrier
//    rings: full/empty (TMA <-> MMA), tmem_full/tmem_empty (MMA <-> epi).
//  * Scan outputs are staged through swizzled shared memory and written by
//    TMA bulk-tensor stores; reduce outputs use plain coalesced stores.
//
// Reference correspondence (pkg/src/halftile):
//    reduce granule sums     reduce.py:92-106 (Reduction16 P.A), :171-198
//    row/tile/CTA combine    reduce.py:123-141, :278-326, :332-373
//    scan in-granule A.U     scan.py:58-71, :74-91 (RowScan)
//    carry chain             scan.py:102-119, :155-172, :178-243, :249-310
//    padding semantics       segmented.py:57-89
//    MMA numerics            engine.py:326-348 (products exact, one rounding)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <type_traits>
#include <mutex>

#include "sm100_ptx.cuh"
#include "tc_collectives.h"

namespace tc {

constexpr int kRow = 64;                         // elements per row
constexpr int kTileRows = 128;                   // UMMA M
constexpr int kTileElems = kRow * kTileRows;     // 8192
constexpr uint32_t kTileBytes = kTileElems * 2;  // 16 KB of fp16
constexpr int kThreads = 192;                    // 6 warps
constexpr int kEpiThreads = 128;                 // warps 2..5
constexpr int kEpiBar = 1;                       // named barrier id
constexpr int OP_REDUCE = 0;
constexpr int OP_SCAN = 1;
constexpr int MODE_LOCAL = 0;
constexpr int MODE_ROWS = 1;
constexpr int MODE_TILES = 2;
constexpr int MODE_GENERAL = 3;
constexpr int MODE_CHUNK = 4;
constexpr int MODE_IRREG = 5;  // irregular segments from a CSR offsets array
constexpr int MODE_ROWSEG = 7;  // whole segments per TMA row (rowseg_*_kernel)
// scan with at most one segment start per row and few factors of two
// (seg >= 64, gcd(seg, 64) <= 4): granules of 8 (GR = 8) with the one
// granule that a start splits recomputed from its raw elements
constexpr int MODE_SPLIT = 8;
// the same for 9 <= seg < 64 (several starts per row, at most one per
// granule of 8): every split granule re-summed from its raw elements
constexpr int MODE_SPLITM = 9;
constexpr int MODE_GSCR = 6;   // GENERAL reduce with many segment ends per row (2m < GR):
                               // end values staged in SMEM, interior segments stored coalesced
constexpr int kMaxCtas = 1024;                    // persistent grid cap
constexpr long long kScanPrepassMax = 1LL << 18;  // largest seg whose range-entry carry is recomputed
constexpr unsigned kFull = 0xffffffffu;

struct WsHeader {
  unsigned int ticket;
  unsigned int epoch;
  unsigned int pad[62];
};
struct Entry {  // one cross-CTA partial of a reduce
  long long seg;
  double val;
};
// workspace layout
constexpr size_t kWsZeroRow = 256;   // 256 B of zeros: TMA source when R == 0
constexpr size_t kWsDummyOut = 512;  // 512 B scratch: TMA store target when R == 0
constexpr size_t kWsEntries = 1024;
// per-channel arrival tickets of the batch-norm statistics: a region no other
// op writes, so it stays zero between calls (the last block resets its
// channel's ticket)
constexpr size_t kWsBnTickets = kWsEntries + sizeof(Entry) * 2 * kMaxCtas;
constexpr long long kBnMaxTicketC = 2048;
constexpr size_t kWsLookback = kWsBnTickets + sizeof(unsigned) * kBnMaxTicketC;

struct Params {
  const __half* x;      // input bits (binary16, or bfloat16 when in_bf16)
  int in_bf16;          // input dtype: 0 = fp16, 1 = bf16 (same MMA kind::f16, other A/B format)
  void* out;
  long long n;          // elements
  long long seg;        // segment size
  long long m;          // granules per segment (seg / g)
  long long rows_full;  // n / 64
  long long num_tiles;  // ceil(n / 8192)
  long long qlast;      // index of the last granule, (n - 1) / g
  long long nseg;       // ceil(n / seg)
  long long step_div;   // GENERAL: (128 * GR) / m   (granule step per tile)
  long long step_mod;   // GENERAL: (128 * GR) % m
  long long ktiles;     // TILES: tiles per segment
  int log2m;            // ROWS: log2(rows per segment)
  const double* carry_in;
  double* total_out;
  WsHeader* hdr;
  Entry* entries;
  long long ck;        // CHUNK: tiles per unit (K)
  long long lag;       // CHUNK: units between a unit's A pass and its O pass
  uint64_t* u_word;    // CHUNK: per-unit aggregate, two tagged 64-bit words (chunk_publish)
  int exclusive;
  int need_fixup;  // reduce: segments may straddle CTA ranges
  const long long* offs;  // IRREG: nseg + 1 non-decreasing offsets, offs[0] = 0, offs[nseg] = n
  long long* tk0;         // IRREG reduce: first start index per tile (T + 1 entries, workspace)
  void* trec;             // IRREG reduce: per-tile carry records (workspace)
};

template <typename T>
__device__ __forceinline__ T cvt_out(float v);
template <>
__device__ __forceinline__ __half cvt_out<__half>(float v) {
  return __float2half_rn(v);
}
template <>
__device__ __forceinline__ float cvt_out<float>(float v) {
  return v;
}
template <>
__device__ __forceinline__ double cvt_out<double>(float v) {
  return static_cast<double>(v);
}
// one rounding from the fp64 carry chain straight to the output dtype
template <typename T>
__device__ __forceinline__ T cvt_out_d(double v);
template <>
__device__ __forceinline__ __half cvt_out_d<__half>(double v) {
  return __double2half(v);
}
template <>
__device__ __forceinline__ float cvt_out_d<float>(double v) {
  return __double2float_rn(v);
}
template <>
__device__ __forceinline__ double cvt_out_d<double>(double v) {
  return v;
}

__host__ __device__ constexpr int pow2_at_least(int v) {
  return v <= 32 ? 32 : v <= 64 ? 64 : v <= 128 ? 128 : v <= 256 ? 256 : 512;
}

template <int OP, int GR, int MODE, typename OutT>
struct Cfg {
  static constexpr int G = 64 / GR;                                      // granule size
  static constexpr bool IRREG = (MODE == MODE_IRREG);
  // UMMA N: scans and IRREG take the full in-row prefix X.U (64 columns)
  static constexpr int N = (OP == OP_SCAN || IRREG) ? 64 : (GR < 16 ? 16 : GR);
  static constexpr bool CHUNK = (MODE == MODE_CHUNK);
  // CTAs per SM (CHUNK keeps 2-4 units of tiles in TMEM: all 512 columns, 1 CTA/SM)
  // GENERAL reduce with 8..32 granules per row runs 3 CTAs/SM: its per-tile
  // granule walk is latency-bound, so a third resident epilogue pays
  // (measured on B200, 2^30 fp16: s = 300 58 -> 78 %, s = 1000 86 -> 93 %
  // of copy bandwidth; GR = 4 (s = 48) is faster at 2, 95 vs 89 %)
  static constexpr int MINB = (CHUNK || (OP == OP_SCAN && GR >= 32)) ? 1
                              : (OP == OP_REDUCE && MODE == MODE_GENERAL && GR >= 8 && GR <= 32) ? 3
                                                                                       : 2;
  // fp32-output scans at 2 CTAs/SM fit either 4 input stages + 1 output
  // buffer or 2 + 2.  The pair-scan modes (GENERAL, IRREG) prefer 2 + 2
  // (measured: s = 300 79 -> 87 % of copy bandwidth), the others 4 + 1.
  static constexpr bool SCAN32_2BUF =
      (MODE == MODE_GENERAL || MODE == MODE_IRREG || MODE == MODE_SPLIT || MODE == MODE_SPLITM);
  static constexpr int STAGES = CHUNK ? 8
                                : (OP == OP_REDUCE)
                                    ? ((MINB == 3 || MODE == MODE_GSCR || MODE == MODE_IRREG) ? 4
                                       : MINB == 2 ? 6 : 8)
                                : (MINB == 2 && sizeof(OutT) == 4 && SCAN32_2BUF) ? 2
                                                    : (MINB == 2 ? 4 : 6);
  static constexpr int ACC = CHUNK ? 8 : 4;  // TMEM accumulator stages (tiles)
  // CHUNK with one granule per row splits the epilogue: warps 2..5 write the
  // prefix sums, warps 6..9 ("aggregate warps") fold row totals into unit
  // aggregates and publish them
  static constexpr bool AGG = CHUNK && GR == 1;
  // warps: TMA, MMA, 4 epilogue (+ AGG: 4 aggregate) (+ CHUNK: the prefix warp)
  static constexpr int THREADS = kThreads + (AGG ? 128 : 0) + (CHUNK ? 32 : 0);
  // arrivals that free a TMEM slot: per thread (128), or lane 0 of the 4
  // output + 4 aggregate warps
  static constexpr int TEMPTY = AGG ? 8 : kEpiThreads;
  static constexpr int TMEM_COLS = pow2_at_least(ACC * N);
  static constexpr int OUT_BUFS =
      (OP == OP_SCAN) ? ((sizeof(OutT) == 4 && MINB == 2 && !SCAN32_2BUF) ? 1 : 2) : 0;
  static constexpr uint32_t OUT_BYTES = kTileElems * sizeof(OutT);
  static constexpr uint32_t OFF_B = STAGES * kTileBytes;
  static constexpr uint32_t OFF_OUT = OFF_B + ((N * 128 + 1023) / 1024) * 1024;
  // GENERAL reduce with one-element granules (odd s): each thread's row of
  // granule prefixes staged in SMEM (row stride 68 floats: conflict-free
  // 16-B stores) so the row's many segment ends are one load each
  // IRREG reduce: each thread's row of in-row prefixes (row stride 68 floats:
  // conflict-free 16-B stores).  GSCR: each row's segment-end values by
  // granule (row stride GR + 1 floats: the walk's predicated stores and the
  // coalesced read-out are bank-conflict-free for the odd m of this mode).
  static constexpr bool SCR = (OP == OP_REDUCE && (MODE == MODE_GSCR || MODE == MODE_IRREG));
  static constexpr uint32_t SCR_BYTES = !SCR ? 0
                                        : IRREG ? kTileRows * 68 * 4
                                                : ((kTileRows * (GR + 1) * 4 + 127) / 128) * 128;
  static constexpr uint32_t OFF_SCR = OFF_OUT + OUT_BUFS * OUT_BYTES;
  static constexpr uint32_t OFF_MISC = OFF_SCR + SCR_BYTES;
  static constexpr int LD_COLS = (OP == OP_SCAN || IRREG) ? 64 : GR;  // TMEM columns read per tile
  static constexpr bool CONTIG = (MODE != MODE_CHUNK);       // contiguous CTA tile ranges
};

template <int STAGES, int ACC>
struct Misc {
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t tfull[ACC];
  uint64_t tempty[ACC];
  uint32_t tmem_base;
  int is_last;
  float pv[2][4];
  int pf[2][4];
  double dsum[4];
  double ce_base;
  double cev[4];
  int cef[4];
  double pd[2][4];
  double fa[2][4];
  float ov[2][4];
  int of[2][4];
  float apv[2][4];  // aggregate warps' exchange
  int apf[2][4];
  double apd[2][4];
  int icnt[2][kTileRows];  // IRREG: segment starts per row of the tile (double-buffered)
  double irs[kTileRows + 1];  // IRREG reduce: exclusive fp64 prefix of the tile's row totals
  double irw[2][4];           // IRREG reduce: per-warp row-total sums
  double idv[4];           // IRREG scan: carry-in composition scratch
  int idf[4];
  uint64_t pfull[4];   // CHUNK: prefix warp -> epilogue (entry value of unit j ready)
  uint64_t pempty[4];  // CHUNK: epilogue -> prefix warp (slot consumed)
  double entry[4];
  long long head_seg;
  double head_val;
  long long tile_o[2];  // GSCR: first segment ending in the tile (double-buffered)
};

template <int OP, int GR, int MODE, typename OutT>
constexpr uint32_t smem_bytes() {
  using C = Cfg<OP, GR, MODE, OutT>;
  return C::OFF_MISC + sizeof(Misc<C::STAGES, C::ACC>) + 1024;  // +1024: alignment slack
}

// Constant B operand, K-major, 128-B swizzled: row n (N index) holds B[k][n]
// for k = 0..63.  Reduce: granule indicator.  Scan: block-diag upper-tri U.
template <int OP, int GR, int N>
__device__ void build_b(uint8_t* sb, uint16_t one_bits) {
  constexpr int G = 64 / GR;
  for (int idx = threadIdx.x; idx < N * 8; idx += blockDim.x) {
    const int n = idx >> 3, pos = idx & 7;
    const int lc = pos ^ (n & 7);  // logical 16-B chunk stored at physical position pos
    __align__(16) uint16_t h[8];  // 1.0 in the input's format (fp16 0x3C00, bf16 0x3F80)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int k = lc * 8 + e;
      bool one;
      if (OP == OP_REDUCE)
        one = (n < GR) && (k / G == n);
      else
        one = (k / G == n / G) && (k <= n);
      h[e] = one ? one_bits : 0;
    }
    *reinterpret_cast<uint4*>(sb + n * 128 + pos * 16) = *reinterpret_cast<uint4*>(h);
  }
}

// Compose segmented-sum pairs: x then y.  (flag = "a boundary occurred")
__device__ __forceinline__ void compose(float& xv, int& xf, float yv, int yf) {
  xv = yf ? yv : xv + yv;
  xf |= yf;
}

// Inclusive segmented scan of (v, f) pairs across the 32 lanes of a warp.
__device__ __forceinline__ void warp_pair_scan(float& v, int& f, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const float vu = __shfl_up_sync(kFull, v, d);
    const int fu = __shfl_up_sync(kFull, f, d);
    if (lane >= d) {
      if (!f) v += vu;
      f |= fu;
    }
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ float warp_incl_scan(float v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const float u = __shfl_up_sync(kFull, v, d);
    if (lane >= d) v += u;
  }
  return v;
}

// One input element as float (binary16 or bfloat16 bits).
__device__ __forceinline__ float in_to_float(const __half* x, long long e, bool bf16) {
  const unsigned short b = __ldg(reinterpret_cast<const unsigned short*>(x) + e);
  return bf16 ? __uint_as_float(static_cast<uint32_t>(b) << 16)
              : __half2float(__ushort_as_half(b));
}

// Sum of x[lo, hi) in fp64 by the 128 epilogue threads (all get the result).
template <typename MiscT>
__device__ double epi_range_sum(const __half* x, bool bf16, long long lo, long long hi, int et,
                                int lane, int qd, MiscT* misc) {
  double acc = 0.0;
  if (hi > lo) {
    long long a = (lo + 7) & ~7LL;  // 16-B aligned start
    if (a > hi) a = hi;
    if (et == 0)
      for (long long e = lo; e < a; ++e) acc += in_to_float(x, e, bf16);
    const long long nb = (hi - a) >> 3;  // whole 8-element blocks
    const uint4* xv = reinterpret_cast<const uint4*>(x + a);
    float fs = 0.f;
    auto add8 = [&](const uint4& w) {
      if (bf16) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f2 = __bfloat1622float2(h[k]);
          fs += f2.x + f2.y;
        }
      } else {
        const __half2* h = reinterpret_cast<const __half2*>(&w);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f2 = __half22float2(h[k]);
          fs += f2.x + f2.y;
        }
      }
    };
    // eight 16-B loads in flight per thread (this pass can be ~2^21 elements
    // per CTA: one load at a time made it latency-bound); fp32 partials go
    // to fp64 every 8 x 8 elements
    long long b = et;
    for (; b + 7 * kEpiThreads < nb; b += 8 * kEpiThreads) {
      uint4 w[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) w[u] = __ldg(xv + b + u * kEpiThreads);
#pragma unroll
      for (int u = 0; u < 8; ++u) add8(w[u]);
      acc += fs;
      fs = 0.f;
    }
    for (; b < nb; b += kEpiThreads) add8(__ldg(xv + b));
    acc += fs;
    if (et == kEpiThreads - 1)
      for (long long e = a + nb * 8; e < hi; ++e) acc += in_to_float(x, e, bf16);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  if (lane == 0) misc->dsum[qd] = acc;
  ptx::named_bar_sync(kEpiBar, kEpiThreads);
  const double r = misc->dsum[0] + misc->dsum[1] + misc->dsum[2] + misc->dsum[3];
  ptx::named_bar_sync(kEpiBar, kEpiThreads);
  return r;
}

// CHUNK: a unit's aggregate (value, has-segment-start) travels as TWO
// 64-bit words written by one 16-byte relaxed store: the fp64 value as a
// double-float pair hi = fp32(v), lo = fp32(v - hi) (~48 significant bits),
// each word carrying its own validity tag in the low half -- (epoch << 2) |
// state, state 1 = no segment start, 2 = start.  A reader accepts the pair
// only when BOTH tags carry the current epoch, so a torn 16-byte read is
// simply retried: no fences on either side (64-bit single-copy atomicity).
__device__ __forceinline__ uint32_t unit_tag(int f, uint32_t ep) { return (ep << 2) | (f ? 2u : 1u); }
__device__ __forceinline__ void chunk_publish(uint64_t* word, double v, int f, uint32_t ep) {
  const float hi = static_cast<float>(v);
  const float lo = static_cast<float>(v - static_cast<double>(hi));
  const uint64_t tag = unit_tag(f, ep);
  ptx::st_relaxed_v2u64(word, (static_cast<uint64_t>(__float_as_uint(hi)) << 32) | tag,
                        (static_cast<uint64_t>(__float_as_uint(lo)) << 32) | tag);
}
__device__ __forceinline__ double unit_value(uint64_t w0, uint64_t w1) {
  return static_cast<double>(__uint_as_float(static_cast<uint32_t>(w0 >> 32))) +
         static_cast<double>(__uint_as_float(static_cast<uint32_t>(w1 >> 32)));
}

// CHUNK prefix warp: for each unit j of this CTA, the value of the open
// segment entering it, handed to the epilogue through misc->entry[j & 3]
// (mbarriers pfull / pempty).  It keeps P = the value entering chunk j,
// composed from ALL units of the earlier chunks, so no CTA waits on
// another's prefix (no serial chain): per chunk it reads every unit
// aggregate (batched relaxed flag loads + one acquire fence), composes them
// in unit order -- E(j) = P (+) units (j, 0..cta-1), P' = P (+) all units
// of chunk j -- in fp64, the same fixed order on every run.
template <typename MiscT>
__device__ void prefix_warp(const Params& p, MiscT* misc, long long n_units, int cta, int Gc,
                            long long ck, long long T, int lane, uint32_t ep, bool has_carry) {
  constexpr int kMaxPer = 8;  // CHUNK grids have <= 256 CTAs (1 per SM)
  const int per = (Gc + 31) / 32;
  const long long chunk_t = static_cast<long long>(Gc) * ck;
  double P = has_carry ? *p.carry_in : 0.0;
  for (long long j = 0; j < n_units; ++j) {
    // units that exist in chunk j
    const long long left = (T - j * chunk_t + ck - 1) / ck;
    const int cnt = left < Gc ? static_cast<int>(left) : Gc;
    const int c0 = lane * per;
    uint64_t w[kMaxPer], w1[kMaxPer];
    unsigned pending = 0;
#pragma unroll
    for (int k = 0; k < kMaxPer; ++k)
      if (k < per && c0 + k < cnt) pending |= 1u << k;
    while (pending) {  // batched: one round trip per poll, not per unit
#pragma unroll
      for (int k = 0; k < kMaxPer; ++k)
        if (pending & (1u << k)) ptx::ld_relaxed_v2u64(p.u_word + 2 * (j * Gc + c0 + k), w[k], w1[k]);
#pragma unroll
      for (int k = 0; k < kMaxPer; ++k)
        if ((pending & (1u << k)) && (static_cast<uint32_t>(w[k]) >> 2) == ep &&
            (static_cast<uint32_t>(w1[k]) >> 2) == ep)
          pending &= ~(1u << k);
      if (pending) __nanosleep(32);
    }
    // per-lane ordered aggregates: a_all over the lane's units, a_pre over those < cta
    double va = 0.0, vp = 0.0;
    int fa = 0, fp = 0;
#pragma unroll
    for (int k = 0; k < kMaxPer; ++k) {
      const int c2 = c0 + k;
      if (k < per && c2 < cnt) {
        const double y = unit_value(w[k], w1[k]);
        const int yf = (static_cast<uint32_t>(w[k]) & 3u) == 2u;
        va = yf ? y : va + y;
        fa |= yf;
        if (c2 < cta) {
          vp = va;
          fp = fa;
        }
      }
    }
    // inclusive ordered pair scan of a_all over the lanes
    double vi = va;
    int fi = fa;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double vu = __shfl_up_sync(kFull, vi, d);
      const int fu = __shfl_up_sync(kFull, fi, d);
      if (lane >= d) {
        if (!fi) vi += vu;
        fi |= fu;
      }
    }
    double ve = __shfl_up_sync(kFull, vi, 1);
    int fe = __shfl_up_sync(kFull, fi, 1);
    if (lane == 0) {
      ve = 0.0;
      fe = 0;
    }
    // prefix over units < cta: exclusive lanes before Lc, then Lc's partial block
    double e = P;
    if (cta > 0) {
      const int lc = (cta - 1) / per;
      const double xv = __shfl_sync(kFull, ve, lc);
      const int xf = __shfl_sync(kFull, fe, lc);
      const double pv = __shfl_sync(kFull, vp, lc);
      const int pf = __shfl_sync(kFull, fp, lc);
      e = xf ? xv : P + xv;
      e = pf ? pv : e + pv;
    }
    const double tv = __shfl_sync(kFull, vi, 31);
    const int tf = __shfl_sync(kFull, fi, 31);
    P = tf ? tv : P + tv;
    if (lane == 0) {
      const int ps = static_cast<int>(j & 3);
      ptx::mbar_wait(&misc->pempty[ps], static_cast<uint32_t>(((j >> 2) & 1) ^ 1));
      misc->entry[ps] = e;
      ptx::mbar_arrive(&misc->pfull[ps]);
    }
    __syncwarp();
  }
}

// Store GR consecutive outputs out[q0 .. q0+GR) (vectorised when aligned).
template <typename OutT, int GR>
__device__ __forceinline__ void store_run(OutT* out, long long q0, const float (&v)[GR],
                                          long long qlast) {
  if (q0 + GR - 1 <= qlast) {
    if constexpr (sizeof(OutT) == 4 && GR % 4 == 0) {
#pragma unroll
      for (int j = 0; j < GR; j += 4)
        *reinterpret_cast<float4*>(out + q0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      return;
    } else if constexpr (sizeof(OutT) == 2 && GR % 4 == 0) {
#pragma unroll
      for (int j = 0; j < GR; j += 4) {
        __half2 a = __floats2half2_rn(v[j], v[j + 1]);
        __half2 b = __floats2half2_rn(v[j + 2], v[j + 3]);
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&a);
        w.y = *reinterpret_cast<uint32_t*>(&b);
        *reinterpret_cast<uint2*>(out + q0 + j) = w;
      }
      return;
    } else if constexpr (sizeof(OutT) == 4 && GR == 2) {
      *reinterpret_cast<float2*>(out + q0) = make_float2(v[0], v[1]);
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < GR; ++j)
    if (q0 + j <= qlast) out[q0 + j] = cvt_out<OutT>(v[j]);
}

// IRREG: P(b) = sum of the first b elements of a row (b in [0, 64]), read
// from the row's in-row inclusive prefix v = (X.U)[row] at a per-thread
// position: a 6-level select tree over registers (no local-memory indexing).
__device__ __forceinline__ float row_prefix(const float (&v)[64], int b) {
  const int i = b - 1;  // v[i] = sum of elements 0..i
  float a[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) a[j] = (i & 32) ? v[j + 32] : v[j];
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
#pragma unroll
    for (int j = 0; j < w; ++j) a[j] = (i & w) ? a[j + w] : a[j];
  }
  return b <= 0 ? 0.f : a[0];
}

// IRREG: first k in [0, nseg] with offs[k] >= v (offs[nseg] = n).
__device__ __forceinline__ long long offs_lower_bound(const long long* offs, long long nseg,
                                                      long long v) {
  long long lo = 0, hi = nseg + 1;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (__ldg(offs + mid) < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// IRREG: contiguous tile range of CTA c (the main kernel's CONTIG split).
__device__ __forceinline__ void irreg_range(long long T, int c, int G, long long n, long long* rb,
                                            long long* re) {
  const long long tb = T * c / G, te = T * (c + 1) / G;
  *rb = tb * kTileElems;
  *re = te * kTileElems < n ? te * kTileElems : n;
}

// IRREG scan, pass 1 ("range tails"): for CTA range c of the main kernel,
// the value the open segment carries OUT of the range -- the sum from the
// range's last segment start (flag 1), or of the whole range when no
// segment starts in it (flag 0).  Reads only those tails: sum over ranges
// of (range end - last start) <= n, typically a few segments per range.
// Deterministic (fixed per-thread assignment, fixed fp64 tree).
constexpr int kTailThreads = 512;
__global__ void __launch_bounds__(kTailThreads) irreg_tail_kernel(const __half* x, int in_bf16, long long n,
                                                         const long long* offs, long long nseg,
                                                         long long T, Entry* tails) {
  const int c = blockIdx.x;
  long long rb, re;
  irreg_range(T, c, gridDim.x, n, &rb, &re);
  __shared__ long long s_lo;
  __shared__ int s_flag;
  __shared__ double s_part[kTailThreads / 32];
  if (threadIdx.x == 0) {
    long long lo = rb;
    int flag = 0;
    if (re > rb) {
      // last real start (k < nseg) below re
      const long long k = offs_lower_bound(offs, nseg, re) - 1;
      if (k >= 0 && k < nseg && __ldg(offs + k) >= rb) {
        lo = __ldg(offs + k);
        flag = 1;
      }
    }
    s_lo = lo;
    s_flag = flag;
  }
  __syncthreads();
  const long long lo = s_lo;
  const bool bf16 = in_bf16 != 0;
  double acc = 0.0;
  if (re > lo) {
    long long a = (lo + 7) & ~7LL;
    if (a > re) a = re;
    if (threadIdx.x == 0)
      for (long long e = lo; e < a; ++e) acc += in_to_float(x, e, bf16);
    const long long nb = (re - a) >> 3;
    const uint4* xv = reinterpret_cast<const uint4*>(x + a);
    constexpr int U = 4;  // independent 16-B loads in flight per thread
    auto add8 = [&](const uint4& w, float& fs) {
      if (bf16) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f2 = __bfloat1622float2(h[k]);
          fs += f2.x + f2.y;
        }
      } else {
        const __half2* h = reinterpret_cast<const __half2*>(&w);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f2 = __half22float2(h[k]);
          fs += f2.x + f2.y;
        }
      }
    };
    const long long step = static_cast<long long>(blockDim.x) * U;
    long long b = threadIdx.x;
    for (; b + (U - 1) * blockDim.x < nb; b += step) {  // <= 512 elements per thread per fp32 partial
      uint4 w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) w[u] = __ldcs(xv + b + u * blockDim.x);
      float fs = 0.f;
#pragma unroll
      for (int u = 0; u < U; ++u) add8(w[u], fs);
      acc += fs;
    }
    for (; b < nb; b += blockDim.x) {
      float fs = 0.f;
      add8(__ldcs(xv + b), fs);
      acc += fs;
    }
    if (threadIdx.x == blockDim.x - 1)
      for (long long e = a + nb * 8; e < re; ++e) acc += in_to_float(x, e, bf16);
  }
  acc = warp_sum_d(acc);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kTailThreads / 32; ++w) t += s_part[w];
    tails[c].seg = s_flag;
    tails[c].val = t;
  }
}

// ------------------------------------------------------------------------
// Batch-norm statistics (the paper's TCU-reduction consumer, PAPER.md:
// 2185-2217).  x is NCHW-contiguous: the HW
// elements of (n, c) are one segment.  ONE read of x: every (n, c) segment
// gives its shifted-data moments S1 = sum (x - K_c), S2 = sum (x - K_c)^2
// with K_c = x[0, c, 0] (a sample of the channel, so |mean - K_c| is of the
// order of the channel's spread and S2 / M - (S1 / M)^2 does not cancel
// catastrophically), fp32 per lane, fp64 per segment; a per-channel pass
// combines the N segments in fixed order in fp64 (the common shift makes
// the combine a plain sum) and clears the scratch it read.  The squares need
// the elements themselves, which a tensor-core MMA with a constant B cannot
// produce, so this consumer runs on CUDA cores; the mean alone is the
// tensor-core segmented reduce (tc_seg_reduce_ex, s = HW).
constexpr int kBnThreads = 256;
constexpr long long kBnWarpMin = 2048;  // segments this long get a warp each

__device__ __forceinline__ double block_sum_d(double v, double* sred) {
  v = warp_sum_d(v);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += sred[w];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(kBnThreads) bn_moments_kernel(const __half* x, int in_bf16,
                                                                long long N, long long C,
                                                                long long HW, double2* mom) {
  const bool bf16 = in_bf16 != 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kWarps = kBnThreads / 32;
  const long long nsegs = N * C;
  // one warp per (n, c) segment; vector width = the segment alignment
  // (HW % 8 == 0: 16-B loads, % 4: 8-B, % 2: 4-B, else 2-B), four in flight
  auto run = [&](auto vec_tag) {
    constexpr int V = decltype(vec_tag)::value;  // elements per load
    using VT = typename std::conditional<V == 8, uint4,
               typename std::conditional<V == 4, uint2,
               typename std::conditional<V == 2, uint32_t, unsigned short>::type>::type>::type;
    const long long nv = HW / V;
    for (long long q = static_cast<long long>(blockIdx.x) * kWarps + warp; q < nsegs;
         q += static_cast<long long>(gridDim.x) * kWarps) {
      const long long c = q % C;
      const float k = in_to_float(x, c * HW, bf16);
      float s1 = 0.f, s2 = 0.f;
      auto acc = [&](const VT& w) {
        const unsigned short* h = reinterpret_cast<const unsigned short*>(&w);
#pragma unroll
        for (int e = 0; e < V; ++e) {
          const float f = bf16 ? __uint_as_float(static_cast<uint32_t>(h[e]) << 16)
                               : __half2float(__ushort_as_half(h[e]));
          const float a = f - k;
          s1 += a;
          s2 = fmaf(a, a, s2);
        }
      };
      const VT* xv = reinterpret_cast<const VT*>(x + q * HW);
      long long i = lane;
      for (; i + 96 < nv; i += 128) {
        const VT a = __ldcs(xv + i), b = __ldcs(xv + i + 32), cc = __ldcs(xv + i + 64),
                 d = __ldcs(xv + i + 96);
        acc(a);
        acc(b);
        acc(cc);
        acc(d);
      }
      for (; i < nv; i += 32) acc(__ldcs(xv + i));
      const double d1 = warp_sum_d(static_cast<double>(s1));
      const double d2 = warp_sum_d(static_cast<double>(s2));
      if (lane == 0) mom[q] = make_double2(d1, d2);
    }
  };
  // small segments (HW < kBnWarpMin): one THREAD per (n, c) segment -- a
  // warp reads 32 neighbouring segments, so every sector it touches is used
  // within a few iterations (L1), and the per-segment sums need no shuffles
  auto run_thread = [&](auto vec_tag) {
    constexpr int V = decltype(vec_tag)::value;
    using VT = typename std::conditional<V == 8, uint4,
               typename std::conditional<V == 4, uint2,
               typename std::conditional<V == 2, uint32_t, unsigned short>::type>::type>::type;
    const long long nv = HW / V;
    for (long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; q < nsegs;
         q += static_cast<long long>(gridDim.x) * blockDim.x) {
      const long long c = q % C;
      const float k = in_to_float(x, c * HW, bf16);
      // four interleaved accumulators (one per load in flight): shorter
      // fp32 chains, both for latency and for rounding error
      float s1[4] = {0.f, 0.f, 0.f, 0.f}, s2[4] = {0.f, 0.f, 0.f, 0.f};
      auto acc = [&](const VT& w, int u) {
        const unsigned short* h = reinterpret_cast<const unsigned short*>(&w);
#pragma unroll
        for (int e = 0; e < V; ++e) {
          const float f = bf16 ? __uint_as_float(static_cast<uint32_t>(h[e]) << 16)
                               : __half2float(__ushort_as_half(h[e]));
          const float a = f - k;
          s1[u] += a;
          s2[u] = fmaf(a, a, s2[u]);
        }
      };
      const VT* xv = reinterpret_cast<const VT*>(x + q * HW);
      long long i = 0;
      for (; i + 3 < nv; i += 4) {
        const VT a = __ldg(xv + i), b = __ldg(xv + i + 1), cc = __ldg(xv + i + 2),
                 d = __ldg(xv + i + 3);
        acc(a, 0);
        acc(b, 1);
        acc(cc, 2);
        acc(d, 3);
      }
      for (; i < nv; ++i) acc(__ldg(xv + i), 0);
      mom[q] = make_double2(
          (static_cast<double>(s1[0]) + s1[1]) + (static_cast<double>(s1[2]) + s1[3]),
          (static_cast<double>(s2[0]) + s2[1]) + (static_cast<double>(s2[2]) + s2[3]));
    }
  };
  if (HW < kBnWarpMin) {
    if ((HW & 7) == 0)
      run_thread(std::integral_constant<int, 8>{});
    else if ((HW & 3) == 0)
      run_thread(std::integral_constant<int, 4>{});
    else if ((HW & 1) == 0)
      run_thread(std::integral_constant<int, 2>{});
    else
      run_thread(std::integral_constant<int, 1>{});
    return;
  }
  if ((HW & 7) == 0)
    run(std::integral_constant<int, 8>{});
  else if ((HW & 3) == 0)
    run(std::integral_constant<int, 4>{});
  else if ((HW & 1) == 0)
    run(std::integral_constant<int, 2>{});
  else
    run(std::integral_constant<int, 1>{});
}

// Per-channel streaming (HW >= kBnChanMin): block (c, sp) streams channel c
// of samples [n0, n1) as ONE flat index over the V-element vectors of those
// segments (V = 8 / 4 / 2 / 1 by the segment alignment; consecutive threads
// read consecutive vectors), four loads in flight per thread, and
// accumulates ONE (S1, S2) pair for the channel (every element shares K_c),
// so the scratch is [splits][C] instead of [N][C].  The flat index is split
// into (segment, vector) with a 32-bit multiply-shift division (the 64-bit
// division it replaces dominated the issue slots), and the moments use the
// packed fp32x2 pipe (FADD2 / FFMA2): two elements per instruction.
constexpr long long kBnChanMin = 48;

struct FastDiv {  // q = floor(i / d) for 0 <= i < 2^31, 1 <= d < 2^31
  uint32_t d, mul, shr;
};
static FastDiv make_fastdiv(uint32_t d) {
  uint32_t shr = 0;
  while ((1ull << shr) < d) ++shr;
  const uint64_t mul = ((1ull << 32) * ((1ull << shr) - d)) / d + 1;
  return FastDiv{d, static_cast<uint32_t>(mul), shr};
}
__device__ __forceinline__ uint32_t fastdiv(uint32_t i, const FastDiv& f) {
  return (__umulhi(i, f.mul) + i) >> f.shr;
}

template <int V, int U, typename OutT>
__global__ void __launch_bounds__(kBnThreads) bn_chan_kernel(const __half* x, int in_bf16,
                                                             long long N, long long C,
                                                             long long HW, FastDiv fd,
                                                             double2* mom, unsigned* ticket,
                                                             OutT* mean_out, OutT* var_out) {
  using VT = typename std::conditional<V == 8, uint4,
             typename std::conditional<V == 4, uint2,
             typename std::conditional<V == 2, uint32_t, unsigned short>::type>::type>::type;
  __shared__ double sred[kBnThreads / 32];
  const long long c = blockIdx.x;
  const int splits = gridDim.y, sp = blockIdx.y;
  const long long n0 = N * sp / splits, n1 = N * (sp + 1) / splits;
  const bool bf16 = in_bf16 != 0;
  const float k = in_to_float(x, c * HW, bf16);
  const float2 nk = make_float2(-k, -k);
  const uint32_t nv = fd.d;  // vectors per segment (HW / V)
  const uint32_t total = static_cast<uint32_t>((n1 - n0) * nv);
  const VT* base = reinterpret_cast<const VT*>(x) + (n0 * C + c) * static_cast<long long>(nv);
  const long long sstride = C * static_cast<long long>(nv);  // vectors between samples
  auto ld = [&](uint32_t i) -> VT {
    const uint32_t q = fastdiv(i, fd);
    return __ldcs(base + q * sstride + (i - q * nv));
  };
  float2 s1[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  float2 s2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  float tail1 = 0.f, tail2 = 0.f;  // V == 1
  auto acc = [&](const VT& w, int u) {
    if constexpr (V == 1) {
      const float f = bf16 ? __uint_as_float(static_cast<uint32_t>(w) << 16)
                           : __half2float(__ushort_as_half(w));
      const float a = f - k;
      tail1 += a;
      tail2 = fmaf(a, a, tail2);
    } else {
      const uint32_t* h = reinterpret_cast<const uint32_t*>(&w);
#pragma unroll
      for (int e = 0; e < V / 2; ++e) {
        const float2 f = bf16 ? make_float2(__uint_as_float(h[e] << 16),
                                            __uint_as_float(h[e] & 0xffff0000u))
                              : __half22float2(*reinterpret_cast<const __half2*>(&h[e]));
        const float2 a = ptx::add_f32x2(f, nk);
        s1[u] = ptx::add_f32x2(s1[u], a);
        s2[u] = ptx::fma_f32x2(a, a, s2[u]);
      }
    }
  };
  double d1 = 0.0, d2 = 0.0;
  auto flush = [&]() {
    d1 += (static_cast<double>(s1[0].x) + s1[0].y) + (static_cast<double>(s1[1].x) + s1[1].y) +
          static_cast<double>(tail1);
    d2 += (static_cast<double>(s2[0].x) + s2[0].y) + (static_cast<double>(s2[1].x) + s2[1].y) +
          static_cast<double>(tail2);
    s1[0] = s1[1] = s2[0] = s2[1] = make_float2(0.f, 0.f);
    tail1 = tail2 = 0.f;
  };
  constexpr uint32_t step = kBnThreads;
  uint32_t i = threadIdx.x;
  int it = 0;
  for (; i + (U - 1) * step < total; i += U * step) {
    VT w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) w[u] = ld(i + u * step);
#pragma unroll
    for (int u = 0; u < U; ++u) acc(w[u], u & 1);
    if (++it == 256 / (V * U)) {  // fp32 partials to fp64 every 128 elements per slot
      flush();
      it = 0;
    }
  }
  for (; i < total; i += step) acc(ld(i), 0);
  flush();
  const double t1 = block_sum_d(d1, sred);
  const double t2 = block_sum_d(d2, sred);
  // the channel's last block to finish combines the splits' moments in
  // split order (deterministic) -- no second launch -- and re-zeroes the
  // scratch and the ticket for the next call
  __shared__ int last;
  if (threadIdx.x == 0) {
    mom[static_cast<long long>(sp) * C + c] = make_double2(t1, t2);
    __threadfence();
    last = (atomicAdd(&ticket[c], 1u) == static_cast<unsigned>(splits - 1));
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < 32) {
    double a1 = 0.0, a2 = 0.0;
    for (int g = threadIdx.x; g < splits; g += 32) {  // lane-strided, then a fixed tree
      const double2 m = __ldcg(&mom[static_cast<long long>(g) * C + c]);
      a1 += m.x;
      a2 += m.y;
      mom[static_cast<long long>(g) * C + c] = make_double2(0.0, 0.0);
    }
    a1 = warp_sum_d(a1);
    a2 = warp_sum_d(a2);
    if (threadIdx.x == 0) {
      const double m = static_cast<double>(N * HW);
      const double dm = a1 / m;  // mean - K
      double var = a2 / m - dm * dm;
      if (var < 0.0) var = 0.0;
      mean_out[c] = static_cast<OutT>(static_cast<double>(k) + dm);
      var_out[c] = static_cast<OutT>(var);
      ticket[c] = 0u;  // ready for the next call
    }
  }
}

template <typename OutT>
__global__ void __launch_bounds__(kBnThreads) bn_finish_kernel(const __half* x, int in_bf16,
                                                               long long N, long long C,
                                                               long long HW, double2* mom,
                                                               long long groups, OutT* mean_out,
                                                               OutT* var_out) {
  __shared__ double sred[kBnThreads / 32];
  const long long c = blockIdx.x;
  double a1 = 0.0, a2 = 0.0;
  // mom[g * C + c], g < groups: per (n, c) segment or per (split, c) block
  for (long long g = threadIdx.x; g < groups; g += blockDim.x) {
    const double2 m = mom[g * C + c];
    a1 += m.x;
    a2 += m.y;
    mom[g * C + c] = make_double2(0.0, 0.0);  // leave the workspace zeroed
  }
  const double s1 = block_sum_d(a1, sred);
  const double s2 = block_sum_d(a2, sred);
  if (threadIdx.x == 0) {
    const double k = static_cast<double>(in_to_float(x, c * HW, in_bf16 != 0));
    const double m = static_cast<double>(N * HW);
    const double d = s1 / m;  // mean - K
    double var = s2 / m - d * d;
    if (var < 0.0) var = 0.0;
    mean_out[c] = static_cast<OutT>(k + d);
    var_out[c] = static_cast<OutT>(var);
  }
}

template <int OP, int GR, int MODE, typename OutT>
__global__ void __launch_bounds__((Cfg<OP, GR, MODE, OutT>::THREADS), (Cfg<OP, GR, MODE, OutT>::MINB))
    seg_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
               const Params p) {
  using C = Cfg<OP, GR, MODE, OutT>;
  using MiscT = Misc<C::STAGES, C::ACC>;
  constexpr int G = C::G;
  constexpr int N = C::N;
  constexpr int STAGES = C::STAGES;
  constexpr int ACC = C::ACC;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  MiscT* misc = reinterpret_cast<MiscT*>(smem + C::OFF_MISC);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- work assignment: one contiguous tile range per CTA, or (CHUNK)
  // unit (j, cta) = tiles [j*Gc*K + cta*K, +K).  Producer and MMA stream
  // each tile ONCE; the CHUNK epilogue visits every unit twice from TMEM,
  // as A(0), A(1), O(0), A(2), O(1), ... (A = aggregate, O = output).
  const long long T = p.num_tiles;
  const int Gc = gridDim.x;
  const int cta = blockIdx.x;
  long long t_begin = 0, t_end = 0;
  if constexpr (C::CONTIG) {
    t_begin = T * cta / Gc;
    t_end = T * (cta + 1) / Gc;
  }
  const long long ck = p.ck;
  const long long chunk_t = static_cast<long long>(Gc) * ck;
  const long long cbase = static_cast<long long>(cta) * ck;
  const long long n_units = (!C::CONTIG && cbase < T) ? (T - cbase + chunk_t - 1) / chunk_t : 0;
  auto unit_t0 = [&](long long j) { return j * chunk_t + cbase; };
  auto unit_t1 = [&](long long j) { return (unit_t0(j) + ck < T) ? unit_t0(j) + ck : T; };
  // producer / MMA: body(i, t), i = tile index in this CTA's sequence
  auto walk_tiles = [&](auto&& body) {
    int i = 0;
    if constexpr (C::CONTIG) {
      for (long long t = t_begin; t < t_end; ++t) body(i++, t);
    } else {
      for (long long j = 0; j < n_units; ++j)
        for (long long t = unit_t0(j); t < unit_t1(j); ++t) body(i++, t);
    }
  };
  // epilogue: body(i, it, t, pass, j, first_of_unit, last_of_unit); i counts
  // epilogue items, it = the tile's index in the producer sequence (TMEM slot)
  auto walk_epi = [&](auto&& body) {
    int i = 0;
    if constexpr (C::CONTIG) {
      for (long long t = t_begin; t < t_end; ++t) {
        body(i, i, t, 1, 0LL, t == t_begin, t == t_end - 1);
        ++i;
      }
    } else {
      const long long lag = p.lag;
      for (long long q = 0; q < n_units + lag; ++q) {
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
          const long long j = pass ? q - lag : q;
          if (j < 0 || j >= n_units) continue;
          const long long t0 = unit_t0(j), t1 = unit_t1(j);
          for (long long t = t0; t < t1; ++t)
            body(i++, static_cast<int>(j * ck + (t - t0)), t, pass, j, t == t0, t == t1 - 1);
        }
      }
    }
  };

  // ---- one-time setup
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tin);
    if (OP == OP_SCAN) ptx::prefetch_tmap(&tout);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&misc->full[s], 1);
      ptx::mbar_init(&misc->empty[s], (MODE == MODE_SPLIT || MODE == MODE_SPLITM) ? 4 : 1);  // SPLIT: the 4 epilogue warps
    }
    for (int a = 0; a < ACC; ++a) {
      ptx::mbar_init(&misc->tfull[a], 1);
      ptx::mbar_init(&misc->tempty[a], C::TEMPTY);
    }
    for (int k = 0; k < 4; ++k) {
      ptx::mbar_init(&misc->pfull[k], 1);
      ptx::mbar_init(&misc->pempty[k], 4);  // one arrival per epilogue warp
    }
    misc->head_seg = -1;
    misc->head_val = 0.0;
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(&misc->tmem_base, C::TMEM_COLS);
    ptx::tmem_relinquish();
  }
  build_b<(C::IRREG ? OP_SCAN : OP), GR, N>(smem + C::OFF_B, p.in_bf16 ? 0x3F80 : 0x3C00);
  if constexpr (C::IRREG) {
    for (int k = threadIdx.x; k < 2 * kTileRows; k += blockDim.x) (&misc->icnt[0][0])[k] = 0;
  }
  ptx::fence_proxy_async_smem();  // B written by the generic proxy, read by the tensor core
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = misc->tmem_base;

  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0) {
      const uint64_t pol = ptx::policy_evict_first();  // streamed exactly once
      walk_tiles([&](int i, long long t) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        ptx::mbar_wait(&misc->empty[s], ph ^ 1u);
        ptx::mbar_arrive_expect_tx(&misc->full[s], kTileBytes);
        ptx::tma_load_2d(&tin, smem + s * kTileBytes, &misc->full[s], 0,
                         static_cast<int32_t>(t * kTileRows), pol);
      });
    }
  } else if (warp == 1) {
    // ================= MMA issuer (one thread) =================
    if (lane == 0) {
      // kind::f16 with fp32 D; A/B format F16 or BF16 (idesc bits 7-9 / 10-12)
      const uint32_t idesc =
          ptx::idesc_f16_f32(128, N) | (p.in_bf16 ? ((1u << 7) | (1u << 10)) : 0u);
      const uint64_t bdesc = ptx::smem_desc_sw128(smem + C::OFF_B);
      walk_tiles([&](int i, long long) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        const int a = i % ACC;
        const uint32_t aph = (i / ACC) & 1;
        ptx::mbar_wait(&misc->tempty[a], aph ^ 1u);
        ptx::mbar_wait(&misc->full[s], ph);
        ptx::tc_fence_after();
        const uint64_t adesc = ptx::smem_desc_sw128(smem + s * kTileBytes);
#pragma unroll
        for (int k = 0; k < 4; ++k)  // K = 64 = 4 x 16; +32 B per K step inside the SW128 atom
          ptx::mma_f16_ss(tmem + a * N, adesc + 2 * k, bdesc + 2 * k, idesc, k > 0 ? 1u : 0u);
        if constexpr (MODE != MODE_SPLIT && MODE != MODE_SPLITM)
          ptx::mma_commit(&misc->empty[s]);  // SPLIT: the epilogue frees it
        ptx::mma_commit(&misc->tfull[a]);
      });
    }
    __syncwarp();
  } else if (warp < 6) {
    // ================= epilogue (warps 2..5) =================
    const int qd = warp & 3;          // TMEM lane quadrant
    const int rit = qd * 32 + lane;   // row in tile
    const int et = threadIdx.x - 64;  // epilogue thread id 0..127
    const bool leader = (et == 0);
    const uint32_t lane_base = static_cast<uint32_t>(qd * 32) << 16;
    const long long range_first_elem = t_begin * kTileElems;
    const bool has_carry = (p.carry_in != nullptr);
    const uint32_t ep = (p.hdr->epoch + 1u) & 0x3FFFFFFFu;

    // running state
    double carry = 0.0;  // value of the segment open at the current tile's entry
    long long q0 = (t_begin * kTileRows + rit) * GR;     // first granule of this row
    long long qmod = 0, qdiv = 0;                        // GENERAL: q0 % m, q0 / m
    long long tpos = 0, tseg = 0;                        // TILES: t % k, t / k
    if constexpr (MODE == MODE_GENERAL || MODE == MODE_GSCR) {
      qmod = q0 % p.m;
      qdiv = q0 / p.m;
    }
    if constexpr (MODE == MODE_SPLIT || MODE == MODE_SPLITM) {  // element granularity: the row's first element mod seg
      const long long e0 = (t_begin * kTileRows + rit) * kRow;
      qmod = e0 % p.m;
      qdiv = e0 / p.m;
    }
    if constexpr (MODE == MODE_TILES) {
      tpos = t_begin % p.ktiles;
      tseg = t_begin / p.ktiles;
    }
    if constexpr (OP == OP_SCAN &&
                  (MODE == MODE_TILES || MODE == MODE_GENERAL || MODE == MODE_SPLIT ||
                   MODE == MODE_SPLITM)) {
      // carry entering this CTA's range: the (< seg) elements of the open
      // segment that precede the range, re-read from HBM (bounded by
      // kScanPrepassMax), plus the caller's carry for segment 0.
      const long long seg_start = (range_first_elem / p.seg) * p.seg;
      carry = epi_range_sum(p.x, p.in_bf16 != 0, seg_start, range_first_elem, et, lane, qd, misc);
      if (seg_start == 0 && has_carry) carry += *p.carry_in;
    }

    // IRREG: kc = first offsets index whose start is at or after the current
    // tile (= lower_bound(offs, tile base)); krange0 = the same at the range
    // start (segments below it began in an earlier CTA's range)
    long long kc = 0, krange0 = 0;
    if constexpr (C::IRREG) {
      {
        // 128-ary search by the epilogue threads: ~4 dependent rounds
        // instead of log2(nseg) serial loads; answer in [lo, hi], offs[hi] >= v
        const long long v = range_first_elem;
        long long lo = 0, hi = p.nseg;
        while (hi - lo > kEpiThreads) {
          const long long span = hi - lo;
          const long long q = lo + span * et / kEpiThreads;  // increasing in et; et = 0 unprobed
          const bool below = et > 0 && __ldg(p.offs + q) < v;
          const long long c = ptx::named_bar_popc(kEpiBar, kEpiThreads, below);
          const long long lo0 = lo;
          if (c > 0) lo = lo0 + span * c / kEpiThreads + 1;  // probes 1..c are below v
          hi = lo0 + span * (c + 1) / kEpiThreads;           // probe c + 1 (c = 127: hi)
        }
        while (lo < hi) {
          const long long mid = (lo + hi) >> 1;
          if (__ldg(p.offs + mid) < v)
            lo = mid + 1;
          else
            hi = mid;
        }
        kc = lo;
      }
      krange0 = kc;
      if constexpr (OP == OP_SCAN) {
        // value carried into this range: compose pass 1's range tails of the
        // CTAs below, (value, has-start) in CTA order -- the sum of the tails
        // from the last range holding a start on
        const Entry* tails = p.entries;
        int lf = -1;
        for (int c2 = et; c2 < cta; c2 += kEpiThreads)
          if (__ldcg(&tails[c2].seg)) lf = c2;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const int y = __shfl_xor_sync(kFull, lf, o);
          lf = y > lf ? y : lf;
        }
        if (lane == 0) misc->idf[qd] = lf;
        ptx::named_bar_sync(kEpiBar, kEpiThreads);
        int lfa = misc->idf[0];
#pragma unroll
        for (int k = 1; k < 4; ++k) lfa = misc->idf[k] > lfa ? misc->idf[k] : lfa;
        double acc = 0.0;
        for (int c2 = et; c2 < cta; c2 += kEpiThreads)
          if (c2 >= lfa) acc += __ldcg(&tails[c2].val);
        acc = warp_sum_d(acc);
        if (lane == 0) misc->idv[qd] = acc;
        ptx::named_bar_sync(kEpiBar, kEpiThreads);
        carry = (misc->idv[0] + misc->idv[1]) + (misc->idv[2] + misc->idv[3]);
      }
    }
    // IRREG: the starts [lo, hi) of this thread's row in tile t.  Pass A
    // counts the tile's starts per row (smem atomics; the count of starts
    // below the tile end comes back through the barrier's popc, 128 offsets
    // per round), then an exclusive scan of the per-row counts places each
    // row's range.  The global last tile also takes the starts at n (empty
    // trailing segments, and the end offset itself) into its last row.
    // The first two rounds of the next tile's offsets are prefetched into
    // registers at the end of this tile's pass A, so their (HBM / L2)
    // latency overlaps this tile's epilogue.
    constexpr long long kNoStart = 1LL << 62;
    long long pf0 = kNoStart, pf1 = kNoStart;
    bool pf_ok = false;
    auto ld_off = [&](long long k) -> long long {
      return k <= p.nseg ? __ldg(p.offs + k) : kNoStart;
    };
    // (the reduce only needs the tile's start range [tk0, tk1): no per-row counts)
    auto irreg_rows = [&](long long t, int par, long long& lo, long long& hi, long long& tk0,
                          long long& tk1) -> long long {
      constexpr bool kRowsNeeded = (OP == OP_SCAN);
      const long long tb = t * kTileElems;
      const long long te = (t == T - 1) ? kNoStart - 1 : tb + kTileElems;
      int* cnt = misc->icnt[par];
      // the previous tile's counts (other buffer) were read by everyone
      // before that tile's pair-scan barrier: clear this thread's row
      misc->icnt[par ^ 1][rit] = 0;
      long long kb = kc;
      for (int round = 0;; ++round) {
        const long long o = (pf_ok && round == 0) ? pf0
                            : (pf_ok && round == 1) ? pf1
                                                    : ld_off(kb + et);
        const bool in = o < te;
        if (kRowsNeeded && in) {
          long long rr = (o - tb) >> 6;
          rr = rr < 0 ? 0 : (rr > kTileRows - 1 ? kTileRows - 1 : rr);
          atomicAdd(&cnt[rr], 1);
        }
        const int c = static_cast<int>(ptx::named_bar_popc(kEpiBar, kEpiThreads, in));
        kb += c;
        if (c < kEpiThreads) break;
      }
      pf0 = ld_off(kb + et);
      pf1 = ld_off(kb + et + kEpiThreads);
      pf_ok = true;
      // and the next 2 KB of offsets into L2 (the array is consumed in order)
      if (et < 16) {
        const long long kp = kb + 2 * kEpiThreads + 16 * et;
        if (kp <= p.nseg) ptx::prefetch_l2(p.offs + kp);
      }
      // the counts are complete (popc barrier): the exclusive prefix over
      // rows = the warp's inclusive scan + the rows of the lower warps, read
      // straight from smem (no further barrier)
      const long long tile_starts = kb - kc;  // uniform
      tk0 = kc;
      tk1 = kb;
      if (tile_starts == 0 || !kRowsNeeded) {
        lo = hi = kc;
        kc = kb;
        return tile_starts;
      }
      const int cr = cnt[rit];
      int incl = cr;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int u = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += u;
      }
      int woff = 0;
#pragma unroll
      for (int k = 0; k < 3; ++k)
        if (k < qd) woff += cnt[32 * k + lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) woff += __shfl_xor_sync(kFull, woff, o);
      lo = kc + woff + (incl - cr);
      hi = lo + cr;
      kc = kb;
      return tile_starts;
    };
    // IRREG: the row's in-row inclusive prefix from TMEM; the ragged last
    // row (outside the TMA view) is recomputed from HBM
    auto irreg_load_row = [&](const auto& r, long long row, float (&vv)[64]) {
#pragma unroll
      for (int k = 0; k < 64; ++k) vv[k] = __uint_as_float(r[k]);
      if (row == p.rows_full) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < 64; ++k) {
          const long long e = row * kRow + k;
          s += (e < p.n) ? in_to_float(p.x, e, p.in_bf16 != 0) : 0.f;
          vv[k] = s;
        }
      }
    };
    // SPLIT: segment start column of this thread's row in tile tt (64 =
    // none; qm = the row's first element mod seg)
    auto split_start = [&](long long tt, long long qm) -> int {
      const long long rowpos = (tt * kTileRows + rit) * kRow;
      const long long r0 = qm == 0 ? 0 : p.m - qm;
      return (r0 < kRow && rowpos + r0 < p.n) ? static_cast<int>(r0) : kRow;
    };
    // position of an offset inside the row, clamped to [0, 64] (memory safety
    // for malformed offsets; exact for valid ones)
    auto irreg_pos = [](long long b) -> int {
      return static_cast<int>(b < 0 ? 0 : (b > kRow ? kRow : b));
    };

    // CHUNK: aggregate of the unit being reduced (P1), and of the last two
    // units, kept until their P2 (one-unit lag)
    double u_v = 0.0;
    int u_f = 0;
    // CHUNK, one granule per row: does tile t hold a segment start?
    // (rows < 2^31 since n < 2^37: 32-bit division, far cheaper than 64-bit)
    auto tile_has_start = [&](long long t) -> bool {
      const uint32_t r0 = static_cast<uint32_t>(t * kTileRows);
      const uint32_t m32 = static_cast<uint32_t>(p.m);
      long long fs = static_cast<long long>(r0 / m32) * m32;  // first start row >= r0
      if (fs < r0) fs += m32;
      if (fs == 0 && has_carry) fs = m32;  // row 0 continues the caller's segment
      return fs < static_cast<long long>(r0) + kTileRows && fs <= p.qlast;
    };
    // hand the unit's aggregate to the prefix warp, which publishes it (the
    // release store's fence would otherwise stall the TMA-issuing leader)
    auto save_unit = [&](long long uj) {
      if (leader) chunk_publish(p.u_word + 2 * (uj * Gc + cta), u_v, u_f, ep);
      u_v = 0.0;
      u_f = 0;
    };

    if constexpr (OP == OP_SCAN && MODE == MODE_CHUNK && GR == 1) {
      // ---- CHUNK, one granule per row: OUTPUT warps.  Tile s of this
      // CTA's sequence: wait for its X.U in TMEM, take the unit's entry value
      // from the prefix warp at the unit's first tile, then exactly the plain
      // row-scan epilogue (pair scans only in tiles holding a segment start).
      // The aggregate warps (6..9) read the same TMEM slots independently.
      const long long ntc =
          n_units ? (n_units - 1) * ck + (unit_t1(n_units - 1) - unit_t0(n_units - 1)) : 0;
      auto row_start = [&](long long row) -> int {
        return (static_cast<uint32_t>(row) % static_cast<uint32_t>(p.m) == 0) && row <= p.qlast &&
               !(row == 0 && has_carry);
      };
      const bool excl = p.exclusive != 0;
      long long jo = 0, ko = 0;
      static_assert(ACC == 8, "CHUNK epilogue assumes 8 TMEM tile slots");
      for (long long s2 = 0; s2 < ntc; ++s2) {
        const long long to = unit_t0(jo) + ko;
        const bool first_o = (ko == 0);
        const bool st_o = tile_has_start(to);
        const long long jo_c = jo;
        if (++ko == ck) {
          ko = 0;
          ++jo;
        }
        const int par = static_cast<int>(s2 & 1);
        const int sl = static_cast<int>(s2 & 7);
        uint32_t ro[64];
        ptx::mbar_wait_warp(&misc->tfull[sl], static_cast<uint32_t>((s2 >> 3) & 1));
        ptx::tc_fence_after();
        {
          uint32_t(&r0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&ro[0]);
          uint32_t(&r1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&ro[32]);
          ptx::tmem_ld_32x32b<32>(tmem + lane_base + sl * N, r0);
          ptx::tmem_ld_32x32b<32>(tmem + lane_base + sl * N + 32, r1);
        }
        ptx::tmem_wait_ld();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&misc->tempty[sl]);
        float vv[64];
#pragma unroll
        for (int k = 0; k < 64; ++k) vv[k] = __uint_as_float(ro[k]);
        const long long row_o = to * kTileRows + rit;
        if (row_o == p.rows_full) {  // ragged last row: recompute the row scan from HBM
          float acc = 0.f;
#pragma unroll
          for (int k = 0; k < 64; ++k) {
            const long long e = row_o * kRow + k;
            acc += (e < p.n) ? in_to_float(p.x, e, p.in_bf16 != 0) : 0.f;
            vv[k] = acc;
          }
        }
        if (first_o) {  // value entering the unit, from the prefix warp
          const int ps = static_cast<int>(jo_c & 3);
          ptx::mbar_wait_warp(&misc->pfull[ps], static_cast<uint32_t>((jo_c >> 2) & 1));
          carry = misc->entry[ps];
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&misc->pempty[ps]);
        }
        if (leader) ptx::bulk_wait_read<C::OUT_BUFS - 1>();  // staging buffer free
        __syncwarp();
        const float tot = vv[63];
        float o_ex = 0.f, o_ve = 0.f;
        int o_fe = 0;
        if (!st_o) {
          const float incl = warp_incl_scan(tot, lane);
          o_ex = __shfl_up_sync(kFull, incl, 1);
          if (lane == 0) o_ex = 0.f;
          if (lane == 31) misc->ov[par][qd] = incl;
        } else {
          float v = tot;
          int f = row_start(row_o);
          warp_pair_scan(v, f, lane);
          o_ve = __shfl_up_sync(kFull, v, 1);
          o_fe = __shfl_up_sync(kFull, f, 1);
          if (lane == 0) {
            o_ve = 0.f;
            o_fe = 0;
          }
          if (lane == 31) {
            misc->ov[par][qd] = v;
            misc->of[par][qd] = f;
          }
        }
        ptx::named_bar_sync(kEpiBar, kEpiThreads);
        float off;
        double offd;  // the same offset in fp64 (total_out)
        if (!st_o) {
          float woff = 0.f, ttot = 0.f;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float y = misc->ov[par][k];
            if (k < qd) woff += y;
            ttot += y;
          }
          offd = carry + static_cast<double>(o_ex + woff);
          off = static_cast<float>(offd);
          carry += static_cast<double>(ttot);
        } else {
          float wv = 0.f, tv = 0.f;
          int wf = 0, tf = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float yv = misc->ov[par][k];
            const int yf = misc->of[par][k];
            if (k < qd) compose(wv, wf, yv, yf);
            compose(tv, tf, yv, yf);
          }
          compose(wv, wf, o_ve, o_fe);
          offd = row_start(row_o) ? 0.0
                                  : (wf ? static_cast<double>(wv) : carry + static_cast<double>(wv));
          off = static_cast<float>(offd);
          carry = tf ? static_cast<double>(tv) : carry + static_cast<double>(tv);
        }
        auto outv = [&](int e) -> float {
          if (excl) return (e == 0) ? (off + 0.f) : (vv[e - 1] + off);
          return vv[e] + off;
        };
        if (p.total_out && row_o == (p.n - 1) / kRow) {
          // the open segment's inclusive sum, from the fp64 carry
          const int k = static_cast<int>((p.n - 1) % kRow);
          float in_row = 0.f;
#pragma unroll
          for (int e = 0; e < 64; ++e)
            if (e == k) in_row = vv[e];
          *p.total_out = static_cast<double>(in_row) + offd;
        }
        uint8_t* stg = smem + C::OFF_OUT + (C::OUT_BUFS == 2 ? par : 0) * C::OUT_BYTES;
        const uint32_t rb = static_cast<uint32_t>(rit) * 128u;
        const uint32_t sw = static_cast<uint32_t>(rit & 7);
        if constexpr (sizeof(OutT) == 2) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            uint4 w;
            __half2 h0 = __floats2half2_rn(outv(8 * c + 0), outv(8 * c + 1));
            __half2 h1 = __floats2half2_rn(outv(8 * c + 2), outv(8 * c + 3));
            __half2 h2 = __floats2half2_rn(outv(8 * c + 4), outv(8 * c + 5));
            __half2 h3 = __floats2half2_rn(outv(8 * c + 6), outv(8 * c + 7));
            w.x = *reinterpret_cast<uint32_t*>(&h0);
            w.y = *reinterpret_cast<uint32_t*>(&h1);
            w.z = *reinterpret_cast<uint32_t*>(&h2);
            w.w = *reinterpret_cast<uint32_t*>(&h3);
            *reinterpret_cast<uint4*>(stg + rb + ((c ^ sw) << 4)) = w;
          }
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              float4 w = make_float4(outv(32 * h + 4 * c + 0), outv(32 * h + 4 * c + 1),
                                     outv(32 * h + 4 * c + 2), outv(32 * h + 4 * c + 3));
              *reinterpret_cast<float4*>(stg + h * 16384 + rb + ((c ^ sw) << 4)) = w;
            }
          }
        }
        if (row_o == p.rows_full) {  // ragged last row: direct stores
          OutT* out = reinterpret_cast<OutT*>(p.out);
#pragma unroll
          for (int k = 0; k < 64; ++k) {
            const long long e = row_o * kRow + k;
            if (e < p.n) out[e] = cvt_out<OutT>(outv(k));
          }
        }
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(kEpiBar, kEpiThreads);
        if (leader) {
          const int32_t r0 = static_cast<int32_t>(to * kTileRows);
          ptx::tma_store_2d(&tout, stg, 0, r0);
          if constexpr (sizeof(OutT) == 4) ptx::tma_store_2d(&tout, stg + 16384, 32, r0);
          ptx::bulk_commit();
        }
      }
    } else {
      walk_epi([&](int i, int it, long long t, int pass, long long uj, bool first, bool last) {
        // TMEM slot of the tile.  CHUNK: the A pass waits for the MMA, the O
        // pass (a unit later) reads the same slot again and releases it.
        const int a = it % ACC;
        const uint32_t aph = (it / ACC) & 1;
        const int par = i & 1;
        const bool wait_full = C::CONTIG || pass == 0;
        const bool release = C::CONTIG || pass == 1;
        if constexpr (!C::CONTIG) {
          q0 = (t * kTileRows + rit) * GR;
        }
        // IRREG: segment starts of this row, [i_lo, i_hi) in offs (before the
        // TMEM wait, so the offset loads overlap the MMA)
        long long i_lo = 0, i_hi = 0, i_tn = 1;  // i_tn: segment starts in the tile (uniform)
        long long i_k0 = 0, i_k1 = 0;            // the tile's starts: offsets [i_k0, i_k1)
        if constexpr (C::IRREG) i_tn = irreg_rows(t, par, i_lo, i_hi, i_k0, i_k1);
        // SPLIT: the row's segment start (column sp_e, 64 = none); the raw 8
        // elements of the granule it splits come from the tile's SMEM stage
        // below (the stage is held until then)
        int sp_e = 64;
        uint4 sp_raw = make_uint4(0u, 0u, 0u, 0u);
        if constexpr (MODE == MODE_SPLIT) sp_e = split_start(t, qmod);
        // SPLITM: bit j of sm_mask = granule j holds a segment start, at
        // column 8 j + ((sm_k0 >> 4 j) & 15)
        uint32_t sm_mask = 0, sm_k0 = 0;
        if constexpr (MODE == MODE_SPLITM) {
          const long long rowpos = (t * kTileRows + rit) * kRow;
          const int s32 = static_cast<int>(p.m);
          const long long lim = p.n - rowpos;
          for (int e = qmod == 0 ? 0 : static_cast<int>(p.m - qmod); e < kRow && e < lim; e += s32) {
            sm_mask |= 1u << (e >> 3);
            sm_k0 |= static_cast<uint32_t>(e & 7) << (4 * (e >> 3));
          }
        }
        if (wait_full) ptx::mbar_wait_warp(&misc->tfull[a], aph);
        ptx::tc_fence_after();
        constexpr int LD = C::LD_COLS;
        uint32_t r[LD];
        if constexpr (LD <= 32) {
          ptx::tmem_ld_32x32b<LD>(tmem + lane_base + a * N, r);
        } else {
          uint32_t(&r0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[0]);
          uint32_t(&r1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[32]);
          ptx::tmem_ld_32x32b<32>(tmem + lane_base + a * N, r0);
          ptx::tmem_ld_32x32b<32>(tmem + lane_base + a * N + 32, r1);
        }
        ptx::tmem_wait_ld();
        if (release) {
          ptx::tc_fence_before();
          ptx::mbar_arrive(&misc->tempty[a]);
        }

        const long long row = t * kTileRows + rit;
        // SPLITM: granule j's 8 raw elements from the tile's SMEM stage (held
        // until the outputs are staged), or from HBM for the ragged last row
        [[maybe_unused]] auto raw8 = [&](int j, float (&xr)[8]) {
          uint4 w;
          if (row != p.rows_full) {
            const uint32_t off16 = static_cast<uint32_t>(rit) * 128u +
                                   ((static_cast<uint32_t>(j) ^ static_cast<uint32_t>(rit & 7)) << 4);
            w = *reinterpret_cast<const uint4*>(smem + (it % STAGES) * kTileBytes + off16);
          } else {
            const long long gpos = row * kRow + 8 * j;
            unsigned short hb[8];
  #pragma unroll
            for (int k = 0; k < 8; ++k)
              hb[k] = (gpos + k < p.n) ? __ldg(reinterpret_cast<const unsigned short*>(p.x) + gpos + k)
                                       : static_cast<unsigned short>(0);
            w = *reinterpret_cast<const uint4*>(hb);
          }
          const uint32_t* hw = reinterpret_cast<const uint32_t*>(&w);
  #pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t b = (hw[k >> 1] >> (16 * (k & 1))) & 0xffffu;
            xr[k] = p.in_bf16 ? __uint_as_float(b << 16)
                              : __half2float(__ushort_as_half(static_cast<unsigned short>(b)));
          }
        };
        if constexpr (MODE == MODE_SPLIT) {
          // the split granule's raw elements: one 16-B swizzled chunk of the
          // row in the tile's SMEM stage (the MMA has consumed it: tfull),
          // then the stage goes back to the producer (4 warp arrivals).  The
          // ragged last row is outside the TMA view: read from HBM.
          const int st = it % STAGES;
          if (sp_e < kRow) {
            if (row != p.rows_full) {
              const uint32_t off16 = static_cast<uint32_t>(rit) * 128u +
                                     ((static_cast<uint32_t>(sp_e >> 3) ^ static_cast<uint32_t>(rit & 7)) << 4);
              sp_raw = *reinterpret_cast<const uint4*>(smem + st * kTileBytes + off16);
            } else {
              const long long gpos = row * kRow + (sp_e & ~7);
              unsigned short hb[8];
  #pragma unroll
              for (int k = 0; k < 8; ++k)
                hb[k] = (gpos + k < p.n) ? __ldg(reinterpret_cast<const unsigned short*>(p.x) + gpos + k)
                                         : static_cast<unsigned short>(0);
              sp_raw = *reinterpret_cast<const uint4*>(hb);
            }
          }
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&misc->empty[st]);
        }

        if constexpr (C::IRREG && OP == OP_REDUCE) {
          // ================================================= irregular reduce
          // row pieces from the in-row prefix P (X.U): segment k starting in
          // this row is complete here iff the next start is in this row too;
          // the row's first start closes segment i_lo - 1 (head = P(start))
          float vv[64];
          irreg_load_row(r, row, vv);
          if (i_tn == 0) {
            // no segment starts in the tile: its sum joins the open segment
            const float ws = warp_sum(vv[63]);
            if (lane == 0) misc->pv[par][qd] = ws;
            ptx::named_bar_sync(kEpiBar, kEpiThreads);
            carry += static_cast<double>((misc->pv[par][0] + misc->pv[par][1]) +
                                         (misc->pv[par][2] + misc->pv[par][3]));
            return;
          }
          // segment-centric: the tile's row prefixes go to SMEM once, the
          // row totals get an fp64 tile-level exclusive prefix R, and then
          // thread i sums segments kc + i, kc + i + 128, ... that start and
          // end inside the tile (coalesced offset loads and output stores,
          // no per-row loops).  G(p) = R[p/64] + P_row(p%64) is the tile
          // prefix at position p; a segment inside one row is P(b) - P(a)
          // in fp32, a longer one (R[rb] - R[ra]) + P(b) - P(a) in fp64.
          OutT* out = reinterpret_cast<OutT*>(p.out);
          float* scr0 = reinterpret_cast<float*>(smem + C::OFF_SCR);
          {
            float* scr = scr0 + rit * 68;
  #pragma unroll
            for (int j = 0; j < 16; ++j)
              *reinterpret_cast<float4*>(scr + 4 * j) =
                  make_float4(vv[4 * j], vv[4 * j + 1], vv[4 * j + 2], vv[4 * j + 3]);
          }
          const double tr = static_cast<double>(vv[63]);
          double incl = tr;
  #pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const double u = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += u;
          }
          if (lane == 31) misc->irw[par][qd] = incl;
          ptx::named_bar_sync(kEpiBar, kEpiThreads);
          double woff = 0.0, wtot = 0.0;
  #pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double y = misc->irw[par][k];
            if (k < qd) woff += y;
            wtot += y;
          }
          misc->irs[rit] = woff + (incl - tr);
          if (et == kEpiThreads - 1) misc->irs[kTileRows] = wtot;
          ptx::named_bar_sync(kEpiBar, kEpiThreads);
          const long long tb = t * kTileElems;
          auto tpos = [&](long long o) -> int {  // position in the tile, clamped to [0, 8192]
            const long long q = o - tb;
            return static_cast<int>(q < 0 ? 0 : (q > kTileElems ? kTileElems : q));
          };
          auto prow = [&](int q) -> float {  // in-row prefix before position q
            const int c = q & 63;
            return c ? scr0[(q >> 6) * 68 + c - 1] : 0.f;
          };
          auto gpos = [&](int q) -> double { return misc->irs[q >> 6] + static_cast<double>(prow(q)); };
          for (long long k = i_k0 + et; k + 1 < i_k1; k += kEpiThreads) {
            const int qa = tpos(__ldg(p.offs + k)), qb = tpos(__ldg(p.offs + k + 1));
            if ((qa >> 6) == (qb >> 6)) {
              out[k] = cvt_out<OutT>(prow(qb) - prow(qa));
            } else {
              const double v = (misc->irs[qb >> 6] - misc->irs[qa >> 6]) +
                               (static_cast<double>(prow(qb)) - static_cast<double>(prow(qa)));
              out[k] = cvt_out_d<OutT>(v);
            }
          }
          // the tile's first start closes segment i_k0 - 1 (carry + head);
          // the segment of its last start stays open (carry = tail)
          const double head = gpos(tpos(__ldg(p.offs + i_k0)));
          const double tail = misc->irs[kTileRows] - gpos(tpos(__ldg(p.offs + i_k1 - 1)));
          const long long seg0 = i_k0 - 1;
          if (seg0 >= 0 && leader) {
            const double val = carry + head;
            if (seg0 < krange0) {
              misc->head_seg = seg0;  // partial: segment began in an earlier CTA's range
              misc->head_val = val;
            } else {
              out[seg0] = cvt_out_d<OutT>(val);
            }
          }
          carry = tail;
        } else if constexpr (OP == OP_REDUCE) {
          // ================================================= reduce
          float gs[GR];
  #pragma unroll
          for (int j = 0; j < GR; ++j) gs[j] = __uint_as_float(r[j]);
          if (row == p.rows_full) {  // ragged last row: beyond the TMA view, patch from HBM
            const long long e0 = row * kRow;
  #pragma unroll
            for (int j = 0; j < GR; ++j) {
              float s = 0.f;
              for (int k = 0; k < G; ++k) {
                const long long e = e0 + j * G + k;
                if (e < p.n) s += in_to_float(p.x, e, p.in_bf16 != 0);
              }
              gs[j] = s;
            }
          }
          OutT* out = reinterpret_cast<OutT*>(p.out);
          if constexpr (MODE == MODE_LOCAL) {
            store_run<OutT, GR>(out, q0, gs, p.qlast);
          } else if constexpr (MODE == MODE_ROWS) {
            // segments = aligned groups of 2^log2m rows inside the tile
            float v = gs[0];
            const int msz = 1 << p.log2m;
            if (msz <= 32) {
              for (int d = 1; d < msz; d <<= 1) v += __shfl_xor_sync(kFull, v, d);
              if ((lane & (msz - 1)) == 0) {
                const long long sg = row >> p.log2m;
                if (sg < p.nseg) out[sg] = cvt_out<OutT>(v);
              }
            } else {
              v = warp_sum(v);
              if (lane == 0) misc->pv[par][qd] = v;
              ptx::named_bar_sync(kEpiBar, kEpiThreads);
              if (lane == 0) {
                if (msz == 64 && (qd & 1) == 0) {
                  const long long sg = row >> 6;
                  if (sg < p.nseg)
                    out[sg] = cvt_out<OutT>(misc->pv[par][qd] + misc->pv[par][qd + 1]);
                } else if (msz == 128 && qd == 0) {
                  const float s4 = (misc->pv[par][0] + misc->pv[par][1]) +
                                   (misc->pv[par][2] + misc->pv[par][3]);
                  out[t] = cvt_out<OutT>(s4);
                }
              }
            }
          } else if constexpr (MODE == MODE_TILES) {
            // whole tiles belong to one segment of ktiles tiles
            const float v = warp_sum(gs[0]);
            if (lane == 0) misc->pv[par][qd] = v;
            ptx::named_bar_sync(kEpiBar, kEpiThreads);
            const float tsum = (misc->pv[par][0] + misc->pv[par][1]) +
                               (misc->pv[par][2] + misc->pv[par][3]);
            if (tpos == 0) carry = 0.0;
            carry += static_cast<double>(tsum);
            if ((tpos == p.ktiles - 1 || t == T - 1) && leader) {
              if (tseg * p.seg < range_first_elem) {
                misc->head_seg = tseg;  // began in an earlier CTA's range
                misc->head_val = carry;
              } else {
                out[tseg] = cvt_out_d<OutT>(carry);
              }
            }
            if (++tpos == p.ktiles) {
              tpos = 0;
              ++tseg;
            }
          } else {
            // MODE_GENERAL / MODE_GSCR: segmented (value, has_end) pair scan
            // over rows.  B is the granule INDICATOR, so gs[j] is the sum of
            // granule j's own elements, and every piece below is a forward
            // fp32 sum of whole granules of ONE segment: a segment's rounding
            // error scales with its own elements only (never with a
            // neighbour's, as a difference of row prefixes would).
            // Segment ends inside the row, in 32-bit granule offsets: the first
            // at p.m - 1 - qmod, then every p.m; the input's last granule ends
            // the ragged last segment.
            const long long rem0 = p.m - 1 - qmod;
            const long long dl = p.qlast - q0;
            const long long seg0 = qdiv;  // segment closed by the row's first end
            float run = 0.f, head = 0.f;
            int seen = 0;
            if constexpr (MODE == MODE_GSCR) {
              if (rit == 0) misc->tile_o[par] = qdiv;  // first segment ending in this tile (row 0)
            }
            if constexpr (MODE == MODE_SPLIT) {
              // MODE_SPLIT (s > 64, gcd(s, 64) <= 4): granules of 8 and at most
              // one segment end per row, at column rem0 (element granularity).
              // Whole granules go to the head or the tail; the granule the end
              // splits is re-summed from its 8 raw elements (sp_raw: the
              // tile's SMEM stage, read above), so head and tail stay forward
              // fp32 sums of their own segment's elements.
              const long long rowpos = row * kRow;
              const bool regular = rowpos + kRow < p.n;
              // warp-uniform: does any regular row of this warp hold an end?
              const bool any_end = __any_sync(kFull, regular && rem0 < kRow);
              if (regular) {
                const int ee = rem0 < kRow ? static_cast<int>(rem0) : kRow;  // end column (64: none)
                seen = ee < kRow ? 1 : 0;
                // pairwise trees (short dependency chains): the row total, and
                // only in warps holding an end the head / tail pieces
                const float total = ((gs[0] + gs[1]) + (gs[2] + gs[3])) + ((gs[4] + gs[5]) + (gs[6] + gs[7]));
                run = total;
                if (any_end) {
                  const int ge = (ee + 1) >> 3, o = (ee + 1) & 7;  // split granule, elements before the split
                  const int gt = o == 0 ? ge : ge + 1;            // first whole granule of the tail
                  float hv[8], tv8[8];
  #pragma unroll
                  for (int j = 0; j < GR; ++j) {
                    hv[j] = j < ge ? gs[j] : 0.f;
                    tv8[j] = j >= gt ? gs[j] : 0.f;
                  }
                  float hs = ((hv[0] + hv[1]) + (hv[2] + hv[3])) + ((hv[4] + hv[5]) + (hv[6] + hv[7]));
                  float ts = ((tv8[0] + tv8[1]) + (tv8[2] + tv8[3])) + ((tv8[4] + tv8[5]) + (tv8[6] + tv8[7]));
                  if (o != 0) {
                    const uint32_t* hw = reinterpret_cast<const uint32_t*>(&sp_raw);
                    float xh[8], xt[8];
  #pragma unroll
                    for (int k = 0; k < 8; ++k) {
                      const uint32_t bb = (hw[k >> 1] >> (16 * (k & 1))) & 0xffffu;
                      const float xk = p.in_bf16 ? __uint_as_float(bb << 16)
                                                 : __half2float(__ushort_as_half(static_cast<unsigned short>(bb)));
                      xh[k] = k < o ? xk : 0.f;
                      xt[k] = k < o ? 0.f : xk;
                    }
                    hs += ((xh[0] + xh[1]) + (xh[2] + xh[3])) + ((xh[4] + xh[5]) + (xh[6] + xh[7]));
                    ts = ((xt[0] + xt[1]) + (xt[2] + xt[3])) + ((xt[4] + xt[5]) + (xt[6] + xt[7])) + ts;
                  }
                  if (seen) {
                    head = hs;
                    run = ts;
                  }
                }
              } else {
                // the row holding the input's last element (or past it): walk
                // its elements from HBM; its ends are the regular one (column
                // rem0) and the input's last element
                const int ee = rem0 < kRow ? static_cast<int>(rem0) : kRow;
                long long sg = seg0;
                for (int k = 0; k < kRow && rowpos + k < p.n; ++k) {
                  const long long e = rowpos + k;
                  run += in_to_float(p.x, e, p.in_bf16 != 0);
                  if (k == ee || e == p.n - 1) {
                    if (!seen) {
                      head = run;
                      seen = 1;
                    } else {
                      out[sg] = cvt_out<OutT>(run);  // the ragged last segment, wholly in this row
                    }
                    ++sg;
                    run = 0.f;
                  }
                }
              }
            } else if (dl >= GR && row != p.rows_full) {
              // a full row that does not hold the input's last granule
              if constexpr (MODE == MODE_GSCR) {
                // many ends per row (2m < GR): ends at e0 < m, e0 + m, ...;
                // each end's value is staged in this row's SMEM slot j and the
                // tile's interior segments are stored coalesced below
                float* stg = reinterpret_cast<float*>(smem + C::OFF_SCR) + rit * (GR + 1);
                const int m32 = static_cast<int>(p.m);
                const int e0 = static_cast<int>(rem0);
                int nx = e0;
  #pragma unroll
                for (int j = 0; j < GR; ++j) {
                  const float v = run + gs[j];
                  const bool end = (j == nx);
                  if (end) {
                    stg[j] = v;
                    nx += m32;
                  }
                  run = end ? 0.f : v;
                }
                head = stg[e0];  // own row: program order, no barrier
                seen = 1;
              } else if (p.m >= GR) {
                // at most one end (granule e0; GR = none): head = granules
                // 0..e0, the open tail = the rest.  Eight interleaved
                // accumulators per piece (short dependency chains: the sums
                // are latency-, not issue-bound), then a fixed tree.
                const int e0 = rem0 < GR ? static_cast<int>(rem0) : GR;
                constexpr int NA = GR < 8 ? GR : 8;
                float ha[NA], ta[NA];
  #pragma unroll
                for (int q = 0; q < NA; ++q) ha[q] = ta[q] = 0.f;
  #pragma unroll
                for (int j = 0; j < GR; ++j) {
                  if (j <= e0)
                    ha[j % NA] += gs[j];
                  else
                    ta[j % NA] += gs[j];
                }
  #pragma unroll
                for (int w = NA / 2; w >= 1; w >>= 1)
  #pragma unroll
                  for (int q = 0; q < w; ++q) {
                    ha[q] += ha[q + w];
                    ta[q] += ta[q + w];
                  }
                seen = e0 < GR;
                head = ha[0];
                run = seen ? ta[0] : ha[0];
              } else {
                // at most two ends (2m >= GR): head, one interior segment, tail
                const int e0 = rem0 < GR ? static_cast<int>(rem0) : GR;
                const int e1 = (e0 < GR && e0 + p.m < GR) ? e0 + static_cast<int>(p.m) : GR;
                float a = 0.f, b = 0.f, c = 0.f;
  #pragma unroll
                for (int j = 0; j < GR; ++j) {
                  if (j <= e0)
                    a += gs[j];
                  else if (j <= e1)
                    b += gs[j];
                  else
                    c += gs[j];
                }
                seen = e0 < GR;
                head = a;
                if (e1 < GR) out[seg0 + 1] = cvt_out<OutT>(b);  // wholly inside this row
                run = !seen ? a : (e1 < GR ? c : b);
              }
            } else {
              // the row holding the input's last granule (or padding): walk
              const int lastj = dl < GR ? static_cast<int>(dl) : GR;
              const int m32 = p.m < (1LL << 20) ? static_cast<int>(p.m) : (1 << 20);
              int e = rem0 < GR ? static_cast<int>(rem0) : GR;
              long long sg = seg0;  // segment containing granule q0 + j
  #pragma unroll
              for (int j = 0; j < GR; ++j) {
                run += gs[j];
                if ((j == e && j <= lastj) || j == lastj) {
                  if (!seen) {
                    head = run;  // needs the carry from earlier rows / tiles
                    seen = 1;
                  } else {
                    out[sg] = cvt_out<OutT>(run);  // segment wholly inside this row
                  }
                  ++sg;
                  run = 0.f;
                  e += m32;
                }
              }
            }
            float v = run;
            int f = seen;
            warp_pair_scan(v, f, lane);
            float ve = __shfl_up_sync(kFull, v, 1);
            int fe = __shfl_up_sync(kFull, f, 1);
            if (lane == 0) {
              ve = 0.f;
              fe = 0;
            }
            if (lane == 31) {
              misc->pv[par][qd] = v;
              misc->pf[par][qd] = f;
            }
            ptx::named_bar_sync(kEpiBar, kEpiThreads);
            float wv = 0.f, tv = 0.f;
            int wf = 0, tf = 0;
  #pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float yv = misc->pv[par][k];
              const int yf = misc->pf[par][k];
              if (k < qd) compose(wv, wf, yv, yf);
              compose(tv, tf, yv, yf);
            }
            compose(wv, wf, ve, fe);
            if (seen) {
              const double val =
                  (static_cast<double>(wv) + static_cast<double>(head)) + (wf ? 0.0 : carry);
              if (seg0 * p.seg < range_first_elem) {
                misc->head_seg = seg0;  // partial: segment began in an earlier CTA's range
                misc->head_val = val;
              } else {
                out[seg0] = cvt_out_d<OutT>(val);
              }
            }
            carry = tf ? static_cast<double>(tv) : carry + static_cast<double>(tv);
            if constexpr (MODE == MODE_GSCR) {
              // the tile's interior segments (ending at a row's second, third,
              // ... end) from the SMEM staging slots, one output per thread per
              // round: coalesced stores instead of one scattered store per end.
              // Every row's walk is complete (pair-scan barrier above); the
              // row holding the input's last granule stored its own.
              const float* stg0 = reinterpret_cast<const float*>(smem + C::OFF_SCR);
              const long long g0 = t * static_cast<long long>(kTileRows) * GR;
              long long gend = g0 + static_cast<long long>(kTileRows) * GR;
              const long long glim = (p.qlast / GR) * GR;
              if (gend > glim) gend = glim;
              const long long m = p.m;
              for (long long o = misc->tile_o[par] + et;; o += kEpiThreads) {
                const long long ge = (o + 1) * m - 1;  // the segment's last granule
                if (ge >= gend) break;
                const int lg = static_cast<int>(ge - g0);
                const int jc = lg & (GR - 1);
                if (jc >= m) out[o] = cvt_out<OutT>(stg0[(lg / GR) * (GR + 1) + jc]);
              }
              // the next tile's walk rewrites the slots
              ptx::named_bar_sync(kEpiBar, kEpiThreads);
            }
            // advance to the next tile's row (contiguous ranges)
            qmod += p.step_mod;
            qdiv += p.step_div;
            if (qmod >= p.m) {
              qmod -= p.m;
              ++qdiv;
            }
          }
          q0 += static_cast<long long>(kTileRows) * GR;
        } else {
          // ================================================= scan
          float vv[64];
  #pragma unroll
          for (int k = 0; k < 64; ++k) vv[k] = __uint_as_float(r[k]);
          if (row == p.rows_full) {  // ragged last row: recompute in-granule scans from HBM
            const long long e0 = row * kRow;
            float s = 0.f;
  #pragma unroll
            for (int k = 0; k < 64; ++k) {
              if (k % G == 0) s = 0.f;
              const long long e = e0 + k;
              s += (e < p.n) ? in_to_float(p.x, e, p.in_bf16 != 0) : 0.f;
              vv[k] = s;
            }
          }
          if constexpr (MODE == MODE_SPLITM) {
            // every granule a segment start splits is re-summed from its raw
            // elements (the tile's SMEM stage) as two restarted prefixes:
            // columns < k0 from the granule start (the old segment), columns
            // >= k0 from k0 (the new one); then the stage is released
  #pragma unroll
            for (int j = 0; j < GR; ++j) {
              if (!((sm_mask >> j) & 1u)) continue;
              const int k0 = static_cast<int>((sm_k0 >> (4 * j)) & 15u);
              float xr[8];
              raw8(j, xr);
              float ao = 0.f, an = 0.f;
  #pragma unroll
              for (int k = 0; k < 8; ++k) {  // branch-free (a branch per column cost ~25 % of issue)
                const bool nw = k >= k0;
                ao = nw ? ao : ao + xr[k];
                an = nw ? an + xr[k] : an;
                vv[j * G + k] = nw ? an : ao;
              }
            }
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&misc->empty[it % STAGES]);
          }
          // SPLIT: the raw elements of the split granule, and the total of
          // its new part (columns k0..7: the new segment's first piece)
          [[maybe_unused]] float sp_x[8];
          [[maybe_unused]] float sp_tot = 0.f;
          if constexpr (MODE == MODE_SPLIT) {
            const uint32_t* hw = reinterpret_cast<const uint32_t*>(&sp_raw);
  #pragma unroll
            for (int k = 0; k < 8; ++k) {
              const uint32_t b = (hw[k >> 1] >> (16 * (k & 1))) & 0xffffu;
              sp_x[k] = p.in_bf16 ? __uint_as_float(b << 16)
                                  : __half2float(__ushort_as_half(static_cast<unsigned short>(b)));
              if (k >= (sp_e & 7)) sp_tot += sp_x[k];
            }
          }
          // staging buffer reuse: the TMA store that last used this buffer
          // must have finished reading it before anyone writes (barrier below).
          if (leader) ptx::bulk_wait_read<C::OUT_BUFS - 1>();
          float off[GR];  // per-granule offset to add (exclusive prefix within segment)
          double cinfd = 0.0;  // TILES / GENERAL / CHUNK: the carry part of off in fp64 (total_out)
          if constexpr (MODE == MODE_LOCAL) {
            ptx::named_bar_sync(kEpiBar, kEpiThreads);
  #pragma unroll
            for (int j = 0; j < GR; ++j) off[j] = 0.f;
          } else if constexpr (MODE == MODE_ROWS) {
            const float tot = vv[63];
            const int msz = 1 << p.log2m;
            float incl = tot;
            float excl;
            if (msz <= 32) {
              const int pos = lane & (msz - 1);
              for (int d = 1; d < msz; d <<= 1) {
                const float u = __shfl_up_sync(kFull, incl, d);
                if (pos >= d) incl += u;
              }
              excl = __shfl_up_sync(kFull, incl, 1);
              if (pos == 0) excl = 0.f;
              ptx::named_bar_sync(kEpiBar, kEpiThreads);
            } else {
              incl = warp_incl_scan(incl, lane);
              excl = __shfl_up_sync(kFull, incl, 1);
              if (lane == 0) excl = 0.f;
              if (lane == 31) misc->pv[par][qd] = incl;
              ptx::named_bar_sync(kEpiBar, kEpiThreads);
              float woff = 0.f;
              if (msz == 64) {
                if (qd & 1) woff = misc->pv[par][qd - 1];
              } else {
  #pragma unroll
                for (int k = 0; k < 3; ++k)
                  if (k < qd) woff += misc->pv[par][k];
              }
              excl += woff;
            }
            off[0] = excl;
          } else if constexpr (MODE == MODE_TILES) {
            const float tot = vv[63];
            float incl = warp_incl_scan(tot, lane);
            float excl = __shfl_up_sync(kFull, incl, 1);
            if (lane == 0) excl = 0.f;
            if (lane == 31) misc->pv[par][qd] = incl;
            ptx::named_bar_sync(kEpiBar, kEpiThreads);
            float woff = 0.f, ttot = 0.f;
  #pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float y = misc->pv[par][k];
              if (k < qd) woff += y;
              ttot += y;
            }
            if (tpos == 0) carry = 0.0;  // a segment starts at this tile
            cinfd = carry + static_cast<double>(excl + woff);
            off[0] = static_cast<float>(cinfd);
            carry += static_cast<double>(ttot);
            if (++tpos == p.ktiles) {
              tpos = 0;
              ++tseg;
            }
          } else if constexpr (C::IRREG) {
            // irregular segments: starts of this row as a 64-bit mask; the
            // row's (value, has-start) pair joins the same row/warp/tile
            // pair scan, then each output is the in-row prefix minus P(the
            // latest start at or before it), or plus the entering carry
            const long long rowbase = row * kRow;
            uint64_t msk = 0;
            float cinf;  // value of the open segment entering the row
            if (i_tn == 0) {
              // no segment starts in the tile: a plain row scan
              const float incl = warp_incl_scan(vv[63], lane);
              float ex = __shfl_up_sync(kFull, incl, 1);
              if (lane == 0) ex = 0.f;
              if (lane == 31) misc->pv[par][qd] = incl;
              ptx::named_bar_sync(kEpiBar, kEpiThreads);
              float woff = 0.f, ttot = 0.f;
  #pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float y = misc->pv[par][k];
                if (k < qd) woff += y;
                ttot += y;
              }
              cinf = static_cast<float>(carry + static_cast<double>(ex + woff));
              carry += static_cast<double>(ttot);
            } else {
              for (long long k = i_lo; k < i_hi && k < p.nseg; ++k) {
                const long long b = __ldg(p.offs + k) - rowbase;
                if (b >= 0 && b < kRow) msk |= 1ull << b;
              }
              float v = vv[63];
              int f = msk != 0;
              if (f) v = vv[63] - row_prefix(vv, 63 - __clzll(static_cast<long long>(msk)));
              warp_pair_scan(v, f, lane);
              float ve = __shfl_up_sync(kFull, v, 1);
              int fe = __shfl_up_sync(kFull, f, 1);
              if (lane == 0) {
                ve = 0.f;
                fe = 0;
              }
              if (lane == 31) {
                misc->pv[par][qd] = v;
                misc->pf[par][qd] = f;
              }
              ptx::named_bar_sync(kEpiBar, kEpiThreads);
              float wv = 0.f, tv = 0.f;
              int wf = 0, tf = 0;
  #pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float yv = misc->pv[par][k];
                const int yf = misc->pf[par][k];
                if (k < qd) compose(wv, wf, yv, yf);
                compose(tv, tf, yv, yf);
              }
              compose(wv, wf, ve, fe);
              const double tprefix = carry;
              carry = tf ? static_cast<double>(tv) : carry + static_cast<double>(tv);
              cinf = wf ? wv : static_cast<float>(tprefix + static_cast<double>(wv));
            }
            // final values in place, in element order (sub = P(latest start))
            float sub = -cinf, prev = 0.f;
            const bool excl = p.exclusive != 0;
            const uint32_t mlo = static_cast<uint32_t>(msk), mhi = static_cast<uint32_t>(msk >> 32);
            if (__any_sync(kFull, msk != 0)) {
  #pragma unroll
              for (int e = 0; e < 64; ++e) {
                const float cur = vv[e];
                const bool st = ((e < 32 ? mlo : mhi) >> (e & 31)) & 1u;
                if (st) sub = prev;
                vv[e] = excl ? (st ? 0.f : prev - sub) : cur - sub;
                prev = cur;
              }
            } else if (excl) {
  #pragma unroll
              for (int e = 63; e >= 0; --e) vv[e] = (e ? vv[e - 1] : 0.f) + cinf;
            } else {
  #pragma unroll
              for (int e = 0; e < 64; ++e) vv[e] += cinf;
            }
            off[0] = 0.f;
          } else {
            // MODE_GENERAL / MODE_CHUNK: pair scan with granule starts
            if constexpr (MODE == MODE_CHUNK) {
              if (pass == 1 && first) {
                // value entering the unit, composed by the prefix warp
                const int ps = static_cast<int>(uj & 3);
                ptx::mbar_wait_warp(&misc->pfull[ps], static_cast<uint32_t>((uj >> 2) & 1));
                carry = misc->entry[ps];
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&misc->pempty[ps]);
              }
            }
            int chain[GR];
            float run = 0.f;
            int seen = 0;
            if constexpr (MODE == MODE_SPLIT) {
              // granules of 8: before the split granule ge the open segment
              // continues (chained), the granule's columns from k0 on start
              // the new segment (their values come from the raw elements,
              // below), and the later granules continue it from the
              // new part's total.  Every value is a forward fp32 sum of its
              // own segment's elements.
              const int ge = sp_e >> 3;
  #pragma unroll
              for (int j = 0; j < GR; ++j) {
                off[j] = run;
                chain[j] = !seen;
                if (j == ge) {
                  run = sp_tot;
                  seen = 1;
                } else {
                  run += vv[j * G + G - 1];
                }
              }
            } else if constexpr (MODE == MODE_SPLITM) {
              // split granules hold restarted prefixes (above): their last
              // column is the new segment's first piece
  #pragma unroll
              for (int j = 0; j < GR; ++j) {
                off[j] = run;
                chain[j] = !seen;
                const bool sp = (sm_mask >> j) & 1u;
                run = sp ? vv[j * G + G - 1] : run + vv[j * G + G - 1];
                seen |= sp ? 1 : 0;
              }
            } else {
              // segment starts inside the row (32-bit granule offsets): the first
              // at (m - q0 % m) % m, then every m; none past the input's end,
              // and granule 0 continues the caller's segment when carried in
              const long long qm = (MODE == MODE_GENERAL) ? qmod : (q0 % p.m);
              const long long r0 = qm == 0 ? 0 : p.m - qm;
              const long long dl = p.qlast - q0;
              const int lastj = dl < GR ? static_cast<int>(dl) : GR;
              const int m32 = p.m < (1LL << 20) ? static_cast<int>(p.m) : (1 << 20);
              int nx = r0 < GR ? static_cast<int>(r0) : GR;
              const bool skip0 = (q0 == 0 && has_carry);
  #pragma unroll
              for (int j = 0; j < GR; ++j) {
                if (j == nx) {
                  if (j <= lastj && !(j == 0 && skip0)) {
                    run = 0.f;
                    seen = 1;
                  }
                  nx += m32;
                }
                off[j] = run;
                chain[j] = !seen;
                run += vv[j * G + G - 1];
              }
            }
            float v = run;
            int f = seen;
            warp_pair_scan(v, f, lane);
            float ve = __shfl_up_sync(kFull, v, 1);
            int fe = __shfl_up_sync(kFull, f, 1);
            if (lane == 0) {
              ve = 0.f;
              fe = 0;
            }
            if (lane == 31) {
              misc->pv[par][qd] = v;
              misc->pf[par][qd] = f;
            }
            ptx::named_bar_sync(kEpiBar, kEpiThreads);
            float wv = 0.f, tv = 0.f;
            int wf = 0, tf = 0;
  #pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float yv = misc->pv[par][k];
              const int yf = misc->pf[par][k];
              if (k < qd) compose(wv, wf, yv, yf);
              compose(tv, tf, yv, yf);
            }
            compose(wv, wf, ve, fe);
            double tprefix;
            if constexpr (MODE == MODE_GENERAL || MODE == MODE_SPLIT || MODE == MODE_SPLITM) {
              tprefix = carry;
              carry = tf ? static_cast<double>(tv) : carry + static_cast<double>(tv);
              qmod += p.step_mod;
              qdiv += p.step_div;
              if (qmod >= p.m) {
                qmod -= p.m;
                ++qdiv;
              }
            } else {
              // MODE_CHUNK
              if (pass == 0) {
                // P1: fold the tile aggregate into the unit's; publish at the unit's end
                u_v = tf ? static_cast<double>(tv) : u_v + static_cast<double>(tv);
                u_f |= tf;
                if (last) save_unit(uj);
                return;  // no output in the reduce pass
              }
              tprefix = carry;
              carry = tf ? static_cast<double>(tv) : carry + static_cast<double>(tv);
            }
            cinfd = wf ? static_cast<double>(wv) : tprefix + static_cast<double>(wv);
            if (p.total_out && row == (p.n - 1) / kRow) {
              // the open segment's inclusive sum: in-row part + the fp64 carry
              const int k = static_cast<int>((p.n - 1) % kRow);
              float in_g = 0.f, o = 0.f;
              int ch = 0;
  #pragma unroll
              for (int e = 0; e < 64; ++e)
                if (e == k) {
                  in_g = vv[e];
                  o = off[e / G];
                  ch = chain[e / G];
                }
              *p.total_out = static_cast<double>(in_g) + static_cast<double>(o) + (ch ? cinfd : 0.0);
            }
            const float cinf = static_cast<float>(cinfd);
  #pragma unroll
            for (int j = 0; j < GR; ++j)
              if (chain[j]) off[j] += cinf;
          }
          // outputs: in-granule scan + granule offset (exclusive: shifted),
          // produced chunk by chunk straight into the swizzled staging tile.
          constexpr bool ONE_OFF = (MODE == MODE_ROWS || MODE == MODE_TILES);
          const bool excl = p.exclusive != 0;
          [[maybe_unused]] int sm_cut[GR];  // SPLITM: restart column per granule (8: none)
          if constexpr (MODE == MODE_SPLITM) {
  #pragma unroll
            for (int j = 0; j < GR; ++j)
              sm_cut[j] = ((sm_mask >> j) & 1u) ? static_cast<int>((sm_k0 >> (4 * j)) & 15u) : 8;
          }
          auto outv = [&](int e) -> float {
            if constexpr (C::IRREG) return vv[e];  // already final
            if constexpr (MODE == MODE_SPLITM) {
              // columns from the split point on restart (offset 0; exclusive: 0 at the start)
              const int k = e & 7, cut = sm_cut[e >> 3];
              const float base = (k >= cut) ? 0.f : off[e >> 3];
              if (excl) return (k == 0 || k == cut) ? (base + 0.f) : (vv[e - 1] + base);
              return vv[e] + base;
            }
            const float base = off[ONE_OFF ? 0 : e / G];
            if (excl) return (e % G == 0) ? (base + 0.f) : (vv[e - 1] + base);
            return vv[e] + base;
          };
          if constexpr (MODE == MODE_LOCAL || MODE == MODE_ROWS || MODE == MODE_TILES) {
            if (p.total_out && row == (p.n - 1) / kRow) {
              // (GENERAL / CHUNK wrote it above, from their fp64 carry)
              const int k = static_cast<int>((p.n - 1) % kRow);
              float in_g = 0.f;
  #pragma unroll
              for (int e = 0; e < 64; ++e)
                if (e == k) in_g = vv[e];
              *p.total_out = static_cast<double>(in_g) + (MODE == MODE_TILES ? cinfd
                                                          : MODE == MODE_ROWS ? static_cast<double>(off[0])
                                                                              : 0.0);
            }
          }
          uint8_t* stg = smem + C::OFF_OUT + (C::OUT_BUFS == 2 ? par : 0) * C::OUT_BYTES;
          const uint32_t rb = static_cast<uint32_t>(rit) * 128u;
          const uint32_t sw = static_cast<uint32_t>(rit & 7);
          if constexpr (sizeof(OutT) == 2) {
  #pragma unroll
            for (int c = 0; c < 8; ++c) {
              uint4 w;
              __half2 h0 = __floats2half2_rn(outv(8 * c + 0), outv(8 * c + 1));
              __half2 h1 = __floats2half2_rn(outv(8 * c + 2), outv(8 * c + 3));
              __half2 h2 = __floats2half2_rn(outv(8 * c + 4), outv(8 * c + 5));
              __half2 h3 = __floats2half2_rn(outv(8 * c + 6), outv(8 * c + 7));
              w.x = *reinterpret_cast<uint32_t*>(&h0);
              w.y = *reinterpret_cast<uint32_t*>(&h1);
              w.z = *reinterpret_cast<uint32_t*>(&h2);
              w.w = *reinterpret_cast<uint32_t*>(&h3);
              *reinterpret_cast<uint4*>(stg + rb + ((c ^ sw) << 4)) = w;
            }
          } else {
  #pragma unroll
            for (int h = 0; h < 2; ++h) {
  #pragma unroll
              for (int c = 0; c < 8; ++c) {
                float4 w = make_float4(outv(32 * h + 4 * c + 0), outv(32 * h + 4 * c + 1),
                                       outv(32 * h + 4 * c + 2), outv(32 * h + 4 * c + 3));
                *reinterpret_cast<float4*>(stg + h * 16384 + rb + ((c ^ sw) << 4)) = w;
              }
            }
          }
          if (row == p.rows_full) {  // ragged last row is outside the TMA view: direct stores
            OutT* out = reinterpret_cast<OutT*>(p.out);
  #pragma unroll
            for (int k = 0; k < 64; ++k) {
              const long long e = row * kRow + k;
              if (e < p.n) out[e] = cvt_out<OutT>(outv(k));
            }
          }
          if constexpr (MODE == MODE_SPLIT) {
            // the split granule, rewritten in place from its raw elements:
            // columns < k0 continue the old segment from off[ge] (carry
            // included), columns >= k0 restart -- forward fp32 sums of each
            // segment's own elements, no per-column selects elsewhere
            if (sp_e < kRow) {
              const int ge = sp_e >> 3, k0 = sp_e & 7;
              float ro = off[0];
  #pragma unroll
              for (int j = 1; j < GR; ++j)
                if (j == ge) ro = off[j];
              float rn = 0.f;
              float gv[8];
  #pragma unroll
              for (int k = 0; k < 8; ++k) {
                const bool nw = k >= k0;
                if (excl) gv[k] = nw ? rn : ro;
                if (nw)
                  rn += sp_x[k];
                else
                  ro += sp_x[k];
                if (!excl) gv[k] = nw ? rn : ro;
              }
              if constexpr (sizeof(OutT) == 2) {
                uint4 w;
                __half2 h0 = __floats2half2_rn(gv[0], gv[1]);
                __half2 h1 = __floats2half2_rn(gv[2], gv[3]);
                __half2 h2 = __floats2half2_rn(gv[4], gv[5]);
                __half2 h3 = __floats2half2_rn(gv[6], gv[7]);
                w.x = *reinterpret_cast<uint32_t*>(&h0);
                w.y = *reinterpret_cast<uint32_t*>(&h1);
                w.z = *reinterpret_cast<uint32_t*>(&h2);
                w.w = *reinterpret_cast<uint32_t*>(&h3);
                *reinterpret_cast<uint4*>(stg + rb + ((static_cast<uint32_t>(ge) ^ sw) << 4)) = w;
              } else {
                const uint32_t c0 = 2u * static_cast<uint32_t>(ge & 3);
                uint8_t* hb = stg + (ge >> 2) * 16384 + rb;
                *reinterpret_cast<float4*>(hb + ((c0 ^ sw) << 4)) = make_float4(gv[0], gv[1], gv[2], gv[3]);
                *reinterpret_cast<float4*>(hb + (((c0 + 1) ^ sw) << 4)) =
                    make_float4(gv[4], gv[5], gv[6], gv[7]);
              }
              if (row == p.rows_full) {
                OutT* out = reinterpret_cast<OutT*>(p.out);
  #pragma unroll
                for (int k = 0; k < 8; ++k) {
                  const long long e = row * kRow + 8 * ge + k;
                  if (e < p.n) out[e] = cvt_out<OutT>(gv[k]);
                }
              }
            }
          }
          ptx::fence_proxy_async_smem();
          ptx::named_bar_sync(kEpiBar, kEpiThreads);
          if (leader) {
            const int32_t r0 = static_cast<int32_t>(t * kTileRows);
            if constexpr (sizeof(OutT) == 2) {
              ptx::tma_store_2d(&tout, stg, 0, r0);
            } else {
              ptx::tma_store_2d(&tout, stg, 0, r0);
              ptx::tma_store_2d(&tout, stg + 16384, 32, r0);
            }
            ptx::bulk_commit();
          }
          q0 += static_cast<long long>(kTileRows) * GR;
        }
      });  // tile loop
    }

    if constexpr (OP == OP_SCAN) {
      if (leader) ptx::bulk_wait<0>();
    }
    // ---- cross-CTA completion: reduce partial fixup / look-back epoch bump
    const bool need_ticket = (OP == OP_REDUCE) ? (p.need_fixup != 0) : (MODE == MODE_CHUNK);
    if (need_ticket) {
      ptx::named_bar_sync(kEpiBar, kEpiThreads);
      if (leader) {
        if constexpr (OP == OP_REDUCE) {
          // open segment at the end of the range -> tail partial
          Entry e0{misc->head_seg, misc->head_val};
          Entry e1{-1LL, carry};
          if constexpr (C::IRREG) {
            // kc - 1 = the last start before the range end; it is never
            // closed inside the range (the row holding its end offset
            // closes it), and it is the end offset itself in the last range
            e1.seg = (kc - 1 < p.nseg) ? kc - 1 : -1LL;
          } else if constexpr (MODE == MODE_SPLIT) {
            // element granularity (p.m = seg)
            const long long le = (t_end * kTileElems < p.n ? t_end * kTileElems : p.n) - 1;
            const bool closed = ((le + 1) % p.m == 0) || (le == p.n - 1);
            e1.seg = closed ? -1LL : le / p.m;
          } else {
            const long long lg_end = t_end * static_cast<long long>(kTileRows) * GR;
            const long long lg = (lg_end < p.qlast + 1 ? lg_end : p.qlast + 1) - 1;
            const bool closed = ((lg + 1) % p.m == 0) || (lg == p.qlast);
            e1.seg = closed ? -1LL : lg / p.m;
          }
          p.entries[2 * cta] = e0;
          p.entries[2 * cta + 1] = e1;
        }
        __threadfence();
        const unsigned tk = atomicAdd(&p.hdr->ticket, 1u);
        misc->is_last = (tk == static_cast<unsigned>(Gc - 1));
      }
      ptx::named_bar_sync(kEpiBar, kEpiThreads);
      if (misc->is_last) {
        __threadfence();
        if constexpr (OP == OP_REDUCE) {
          // deterministic combine of partials in CTA order (the paper's grid
          // pass 2, reduce.py:365-369, done by the last CTA instead of a
          // second launch).  Stage entries through the now idle input ring.
          Entry* se = reinterpret_cast<Entry*>(smem);
          const int ne = 2 * Gc;
          for (int k = et; k < ne; k += kEpiThreads) {
            Entry e;
            e.seg = __ldcg(&p.entries[k].seg);
            e.val = __ldcg(&p.entries[k].val);
            se[k] = e;
          }
          ptx::named_bar_sync(kEpiBar, kEpiThreads);
          // each run of equal segment ids is summed by the thread owning its first entry
          OutT* out = reinterpret_cast<OutT*>(p.out);
          for (int k = et; k < ne; k += kEpiThreads) {
            const long long sg = se[k].seg;
            if (sg < 0) continue;
            int pk = k - 1;
            while (pk >= 0 && se[pk].seg < 0) --pk;
            if (pk >= 0 && se[pk].seg == sg) continue;  // not the first entry of its run
            double acc = 0.0;
            for (int kk = k; kk < ne; ++kk) {
              const long long s2 = se[kk].seg;
              if (s2 < 0) continue;
              if (s2 != sg) break;
              acc += se[kk].val;
            }
            out[sg] = cvt_out_d<OutT>(acc);
          }
        }
        if (leader) {
          p.hdr->epoch = ep;
          p.hdr->ticket = 0u;
          __threadfence();
        }
      }
    }
  } else if (C::AGG && warp < 10) {
    // ================= aggregate warps (CHUNK, one granule per row) =========
    // Tile s: read only the row totals (TMEM column 63), fold start-free
    // tiles into a per-thread fp64 sum, compose (value, has-start) pairs in
    // tiles holding a segment start; at the unit's last tile publish the
    // unit aggregate as one fence-free 64-bit word.  Runs ahead of the output
    // warps by up to the 8 TMEM slots, which is the slack that hides the
    // publish -> observe latency from the other CTAs' prefix warps.
    if constexpr (C::AGG) {
      const int qa = warp & 3;
      const int ra = qa * 32 + lane;
      const int ea = threadIdx.x - 192;
      const bool has_carry = (p.carry_in != nullptr);
      const uint32_t ep = (p.hdr->epoch + 1u) & 0x3FFFFFFFu;
      const uint32_t lb = static_cast<uint32_t>(qa * 32) << 16;
      constexpr uint32_t kAggBar = 2;
      const long long ntc =
          n_units ? (n_units - 1) * ck + (unit_t1(n_units - 1) - unit_t0(n_units - 1)) : 0;
      double pacc = 0.0, u_v = 0.0;
      int u_f = 0, bpar = 0;
      long long ja = 0, ka = 0;
      for (long long s2 = 0; s2 < ntc; ++s2) {
        const long long ta = unit_t0(ja) + ka;
        const bool last_a = (ka == ck - 1) || (ta == T - 1);
        const long long ja_c = ja;
        if (++ka == ck) {
          ka = 0;
          ++ja;
        }
        const long long r0 = ta * kTileRows;
        bool st_a;
        {
          const uint32_t m32 = static_cast<uint32_t>(p.m);
          long long fs = static_cast<long long>(static_cast<uint32_t>(r0) / m32) * m32;
          if (fs < r0) fs += m32;
          if (fs == 0 && has_carry) fs = m32;
          st_a = fs < r0 + kTileRows && fs <= p.qlast;
        }
        const int sl = static_cast<int>(s2 & 7);
        uint32_t r1[1];
        ptx::mbar_wait_warp(&misc->tfull[sl], static_cast<uint32_t>((s2 >> 3) & 1));
        ptx::tc_fence_after();
        ptx::tmem_ld_32x32b<1>(tmem + lb + sl * N + 63, r1);
        ptx::tmem_wait_ld();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&misc->tempty[sl]);
        const long long row = r0 + ra;
        float tot = __uint_as_float(r1[0]);
        if (row == p.rows_full) {  // ragged last row: outside the TMA view
          float acc = 0.f;
#pragma unroll
          for (int k = 0; k < kRow; ++k) {
            const long long e = row * kRow + k;
            if (e < p.n) acc += in_to_float(p.x, e, p.in_bf16 != 0);
          }
          tot = acc;
        }
        __syncwarp();
        if (!st_a) pacc += static_cast<double>(tot);
        if (!(st_a || last_a)) continue;  // uniform
        if (st_a) {
          float v = tot;
          int f = (static_cast<uint32_t>(row) % static_cast<uint32_t>(p.m) == 0) &&
                  row <= p.qlast && !(row == 0 && has_carry);
          warp_pair_scan(v, f, lane);
          if (lane == 31) {
            misc->apv[bpar][qa] = v;
            misc->apf[bpar][qa] = f;
          }
        }
        const double pw = warp_sum_d(pacc);
        if (lane == 0) misc->apd[bpar][qa] = pw;
        ptx::named_bar_sync(kAggBar, kEpiThreads);
        u_v += ((misc->apd[bpar][0] + misc->apd[bpar][1]) + misc->apd[bpar][2]) +
               misc->apd[bpar][3];
        pacc = 0.0;
        if (st_a) {
          float tv = 0.f;
          int tf = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) compose(tv, tf, misc->apv[bpar][k], misc->apf[bpar][k]);
          u_v = tf ? static_cast<double>(tv) : u_v + static_cast<double>(tv);
          u_f |= tf;
        }
        if (last_a) {
          if (ea == 0) chunk_publish(p.u_word + 2 * (ja_c * Gc + cta), u_v, u_f, ep);
          u_v = 0.0;
          u_f = 0;
        }
        bpar ^= 1;
      }
    }
  } else {
    // ================= prefix warp (CHUNK only) =================
    if constexpr (MODE == MODE_CHUNK)
      prefix_warp(p, misc, n_units, cta, Gc, ck, T, lane, (p.hdr->epoch + 1u) & 0x3FFFFFFFu,
                  p.carry_in != nullptr);
  }

  // ---- teardown
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// =====================================================================
// MODE_ROWSEG reduce: whole segments per TMA row.
//
// For a segment size s with few factors of two (g = gcd(s, 64) <= 8, i.e.
// 8 or more granules per 64-element row), the granule formulation leaves
// many segment ends inside every row and a per-element walk in the
// epilogue.  Instead the input is viewed as a matrix X[R x L] whose rows
// hold k WHOLE segments, L = k s with 2L a multiple of 16 bytes (k a
// multiple of 8 / gcd(s, 8)) -- the paper's strided Reduction16n, where
// column c of the loaded tile is segment c, with the stride chosen so TMA
// can walk it.  A row is ceil(L / 64) SW128 chunks of 64 columns (TMA
// zero-fills the columns past L); the MMA accumulates every chunk c of a
// 128-row block against its own indicator B_c[k'][j] = [(64c + k') / s ==
// j] into one TMEM accumulator, so column j of row r is exactly the sum of
// segment r k + j, computed from that segment's elements only.  No segment
// crosses a row, so there is no carry chain and no cross-CTA fixup: the
// epilogue stores k consecutive outputs per row.  The tail of n - R L < L
// elements (< k + 1 segments, the last possibly ragged) is summed in fp64
// by the last CTA.
constexpr int kRsStages = 4;
constexpr int kRsAcc = 4;
constexpr uint32_t kRsMaxB = 24 * 1024;  // B matrices (ring 64 KB + B + staging 16 KB: 2 CTAs / SM)
constexpr int kRsMaxRowBytes = 64;       // k * sizeof(out) <= 64: one staging buffer <= 8 KB

struct RsParams {
  const __half* x;
  int in_bf16;
  void* out;
  long long n, s, L, R, nblk;  // elements, segment, row length, rows, 128-row blocks
  int k, nchunk;               // segments per row, 64-column chunks per row
  int evict_normal;            // L2 policy of the input loads (0: evict-first)
};

struct RsMisc {
  uint64_t full[kRsStages];
  uint64_t empty[kRsStages];
  uint64_t tfull[kRsAcc];
  uint64_t tempty[kRsAcc];
  uint32_t tmem_base;
};

__host__ __device__ constexpr int rs_n(int ks) { return ks < 16 ? 16 : ks; }  // UMMA N (a multiple of 16)
constexpr uint32_t kRsOffB = kRsStages * kTileBytes;
// dynamic shared memory of a launch: ring + nchunk B matrices + 2 output
// staging buffers (128 rows x row_bytes) + misc
__host__ __device__ inline uint32_t rs_off_stg(int nch, int n) {
  return kRsOffB + ((static_cast<uint32_t>(nch) * n * 128 + 1023) / 1024) * 1024;
}
__host__ __device__ inline uint32_t rs_off_misc(int nch, int n, int row_bytes) {
  return rs_off_stg(nch, n) + 2 * kTileRows * static_cast<uint32_t>(row_bytes);
}
constexpr uint32_t kRsSmemMax =
    kRsOffB + kRsMaxB + 2 * kTileRows * kRsMaxRowBytes + sizeof(RsMisc) + 2048;

template <typename OutT, int KS>
__global__ void __launch_bounds__(kThreads, 2)
    rowseg_reduce_kernel(const __grid_constant__ CUtensorMap tin,
                         const __grid_constant__ CUtensorMap tout, const RsParams p) {
  constexpr int kRsN = rs_n(KS);
  constexpr uint32_t kRsBBytes = kRsN * 128;  // one chunk's B: N rows of 128 B
  // rows of >= 16 output bytes go through SMEM and one TMA store per block
  // (a contiguous 128 * KS-output region): direct per-lane stores would
  // scatter 16-byte pieces over 32 lines per instruction
  constexpr int kRowBytes = KS * static_cast<int>(sizeof(OutT));
  constexpr bool kStage = kRowBytes >= 16;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  RsMisc* misc =
      reinterpret_cast<RsMisc*>(smem + rs_off_misc(p.nchunk, kRsN, kStage ? kRowBytes : 0));
  uint8_t* stg_base = smem + rs_off_stg(p.nchunk, kRsN);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const long long b_begin = p.nblk * blockIdx.x / gridDim.x;
  const long long b_end = p.nblk * (blockIdx.x + 1) / gridDim.x;
  const int nch = p.nchunk;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tin);
    if (kStage) ptx::prefetch_tmap(&tout);
    for (int i = 0; i < kRsStages; ++i) {
      ptx::mbar_init(&misc->full[i], 1);
      ptx::mbar_init(&misc->empty[i], 1);
    }
    for (int a = 0; a < kRsAcc; ++a) {
      ptx::mbar_init(&misc->tfull[a], 1);
      ptx::mbar_init(&misc->tempty[a], kEpiThreads);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(&misc->tmem_base, kRsAcc * kRsN < 32 ? 32 : kRsAcc * kRsN);
    ptx::tmem_relinquish();
  }
  // the per-chunk indicator matrices, K-major, 128-B swizzled (row j = B[.][j])
  const uint16_t one = p.in_bf16 ? 0x3F80 : 0x3C00;
  for (int idx = threadIdx.x; idx < nch * kRsN * 8; idx += blockDim.x) {
    const int c = idx / (kRsN * 8), rem = idx % (kRsN * 8);
    const int j = rem >> 3, pos = rem & 7;
    const int lc = pos ^ (j & 7);
    __align__(16) uint16_t h[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const long long col = 64LL * c + lc * 8 + e;  // column of the row
      h[e] = (j < p.k && col < p.L && col / p.s == j) ? one : 0;
    }
    *reinterpret_cast<uint4*>(smem + kRsOffB + c * kRsBBytes + j * 128 + pos * 16) =
        *reinterpret_cast<uint4*>(h);
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = misc->tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = p.evict_normal ? ptx::policy_evict_normal() : ptx::policy_evict_first();
      int i = 0;
      for (long long b = b_begin; b < b_end; ++b)
        for (int c = 0; c < nch; ++c, ++i) {
          const int st = i % kRsStages;
          ptx::mbar_wait(&misc->empty[st], ((i / kRsStages) & 1) ^ 1u);
          ptx::mbar_arrive_expect_tx(&misc->full[st], kTileBytes);
          ptx::tma_load_2d(&tin, smem + st * kTileBytes, &misc->full[st], 64 * c,
                           static_cast<int32_t>(b * kTileRows), pol);
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc =
          ptx::idesc_f16_f32(128, kRsN) | (p.in_bf16 ? ((1u << 7) | (1u << 10)) : 0u);
      int i = 0, blk = 0;
      for (long long b = b_begin; b < b_end; ++b, ++blk) {
        const int a = blk % kRsAcc;
        ptx::mbar_wait(&misc->tempty[a], ((blk / kRsAcc) & 1) ^ 1u);
        for (int c = 0; c < nch; ++c, ++i) {
          const int st = i % kRsStages;
          ptx::mbar_wait(&misc->full[st], (i / kRsStages) & 1);
          ptx::tc_fence_after();
          const uint64_t adesc = ptx::smem_desc_sw128(smem + st * kTileBytes);
          const uint64_t bdesc = ptx::smem_desc_sw128(smem + kRsOffB + c * kRsBBytes);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            ptx::mma_f16_ss(tmem + a * kRsN, adesc + 2 * kk, bdesc + 2 * kk, idesc,
                            (c > 0 || kk > 0) ? 1u : 0u);
          ptx::mma_commit(&misc->empty[st]);
        }
        ptx::mma_commit(&misc->tfull[a]);
      }
    }
    __syncwarp();
  } else {
    const int qd = warp & 3;
    const int rit = qd * 32 + lane;
    const int et = threadIdx.x - 64;
    const uint32_t lane_base = static_cast<uint32_t>(qd * 32) << 16;
    OutT* out = reinterpret_cast<OutT*>(p.out);
    int blk = 0;
    for (long long b = b_begin; b < b_end; ++b, ++blk) {
      const int a = blk % kRsAcc;
      ptx::mbar_wait_warp(&misc->tfull[a], (blk / kRsAcc) & 1);
      ptx::tc_fence_after();
      uint32_t r[KS];
      if constexpr (KS <= 32) {
        ptx::tmem_ld_32x32b<KS>(tmem + lane_base + a * kRsN, r);
      } else {
        uint32_t(&r0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[0]);
        uint32_t(&r1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[32]);
        ptx::tmem_ld_32x32b<32>(tmem + lane_base + a * kRsN, r0);
        ptx::tmem_ld_32x32b<32>(tmem + lane_base + a * kRsN + 32, r1);
      }
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&misc->tempty[a]);
      const long long row = b * kTileRows + rit;
      float v[KS];
#pragma unroll
      for (int j = 0; j < KS; ++j) v[j] = __uint_as_float(r[j]) + 0.f;  // -0 -> +0
      if constexpr (kStage) {
        uint8_t* stg = stg_base + (blk & 1) * (kTileRows * kRowBytes);
        if (et == 0) ptx::bulk_wait_read<1>();  // the store that used this buffer has read it
        ptx::named_bar_sync(kEpiBar, kEpiThreads);
        uint8_t* dst = stg + rit * kRowBytes;
        if constexpr (sizeof(OutT) == 2) {
#pragma unroll
          for (int q = 0; q < KS / 8; ++q) {
            uint4 w;
            __half2 h0 = __floats2half2_rn(v[8 * q + 0], v[8 * q + 1]);
            __half2 h1 = __floats2half2_rn(v[8 * q + 2], v[8 * q + 3]);
            __half2 h2 = __floats2half2_rn(v[8 * q + 4], v[8 * q + 5]);
            __half2 h3 = __floats2half2_rn(v[8 * q + 6], v[8 * q + 7]);
            w.x = *reinterpret_cast<uint32_t*>(&h0);
            w.y = *reinterpret_cast<uint32_t*>(&h1);
            w.z = *reinterpret_cast<uint32_t*>(&h2);
            w.w = *reinterpret_cast<uint32_t*>(&h3);
            reinterpret_cast<uint4*>(dst)[q] = w;
          }
        } else if constexpr (sizeof(OutT) == 4) {
#pragma unroll
          for (int q = 0; q < KS / 4; ++q)
            reinterpret_cast<float4*>(dst)[q] =
                make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else {
#pragma unroll
          for (int q = 0; q < KS / 2; ++q)
            reinterpret_cast<double2*>(dst)[q] =
                make_double2(static_cast<double>(v[2 * q]), static_cast<double>(v[2 * q + 1]));
        }
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(kEpiBar, kEpiThreads);
        if (et == 0) {
          ptx::tma_store_2d(&tout, stg, 0, static_cast<int32_t>(b * kTileRows));
          ptx::bulk_commit();
        }
      } else if (row < p.R) {
        store_run<OutT, KS>(out, row * KS, v, row * KS + KS - 1);
      }
    }
    if (kStage && et == 0) ptx::bulk_wait<0>();
    // the tail past R rows: < k + 1 segments, summed in fp64 by the last CTA
    if (blockIdx.x == gridDim.x - 1) {
      const long long base = p.R * p.L;
      const long long ntail = (p.n - base + p.s - 1) / p.s;
      for (long long j = et; j < ntail; j += kEpiThreads) {
        const long long lo = base + j * p.s;
        const long long hi = lo + p.s < p.n ? lo + p.s : p.n;
        double acc = 0.0;
        for (long long e = lo; e < hi; ++e) acc += in_to_float(p.x, e, p.in_bf16 != 0);
        out[p.R * KS + j] = cvt_out_d<OutT>(acc + 0.0);
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kRsAcc * kRsN < 32 ? 32 : kRsAcc * kRsN);
  }
}

// =====================================================================
// MODE_ROWSEG scan: the same whole-segments-per-row view for the scan.
//
// X[R x L], L = k s, k whole segments per row, ceil(L / 64) chunks per row.
// Chunk c of a 128-row block is multiplied by U_c[k'][j] = [seg(64c + k')
// == seg(64c + j) and k' <= j] (the block-diagonal upper-triangular ones of
// the paper's A.U row scan, with blocks = the segment pieces inside the
// chunk), so TMEM holds the inclusive in-segment prefix of every piece.  A
// segment that started in an earlier chunk of the same row continues with
// that chunk's last inclusive value (one carry per thread, added to the
// leading columns below the chunk's first segment start -- a position
// shared by every row).  Exclusive outputs are the inclusive ones shifted
// by one column inside each segment.  No segment crosses a row: no
// carries between rows, tiles or CTAs.  Outputs go through swizzled SMEM
// staging and TMA bulk-tensor stores into the same [R x L] view; the tail
// of n - R L < L elements is scanned in fp64 by the last CTA.
constexpr int kRssStages = 4;
constexpr int kRssAcc = 8;  // 8 x 64 TMEM columns: 1 CTA / SM
// chunks per row: B matrices of 8 KB each between the input ring and the
// output staging (fp16 output: 16 fit the 227-KB budget, fp32: 10)
constexpr int kRssMaxChunks = 16;
__host__ __device__ constexpr int rss_max_chunks(int out_esize) { return out_esize == 2 ? 16 : 10; }
constexpr uint32_t kRssOffB = kRssStages * kTileBytes;
template <typename OutT>
__host__ __device__ constexpr uint32_t rss_off_out() {
  return kRssOffB + rss_max_chunks(static_cast<int>(sizeof(OutT))) * 8192;
}

struct RssMisc {
  uint64_t full[kRssStages];
  uint64_t empty[kRssStages];
  uint64_t tfull[kRssAcc];
  uint64_t tempty[kRssAcc];
  uint64_t smask[kRssMaxChunks];  // segment starts in chunk c (bit j = column 64c + j)
  int fs[kRssMaxChunks];          // first start column in chunk c (64: none)
  int cont[kRssMaxChunks];        // chunk c's last segment continues into chunk c + 1
  uint32_t tmem_base;
};

template <typename OutT>
constexpr uint32_t rss_smem() {
  return rss_off_out<OutT>() + 2 * kTileElems * sizeof(OutT) + sizeof(RssMisc) + 1024;
}

struct RssParams {
  const __half* x;
  int in_bf16;
  void* out;
  long long n, s, L, R, nblk;
  int nchunk, exclusive;
  int evict_normal;  // L2 policy of the input loads (0: evict-first)
};

template <typename OutT>
__global__ void __launch_bounds__(kThreads, 1)
    rowseg_scan_kernel(const __grid_constant__ CUtensorMap tin,
                       const __grid_constant__ CUtensorMap tout, const RssParams p) {
  constexpr uint32_t kOutBytes = kTileElems * sizeof(OutT);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  RssMisc* misc = reinterpret_cast<RssMisc*>(smem + rss_off_out<OutT>() + 2 * kOutBytes);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const long long b_begin = p.nblk * blockIdx.x / gridDim.x;
  const long long b_end = p.nblk * (blockIdx.x + 1) / gridDim.x;
  const int nch = p.nchunk;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tin);
    ptx::prefetch_tmap(&tout);
    for (int i = 0; i < kRssStages; ++i) {
      ptx::mbar_init(&misc->full[i], 1);
      ptx::mbar_init(&misc->empty[i], 1);
    }
    for (int a = 0; a < kRssAcc; ++a) {
      ptx::mbar_init(&misc->tfull[a], 1);
      ptx::mbar_init(&misc->tempty[a], kEpiThreads);
    }
    // the chunk geometry is the same for every row
    for (int c = 0; c < nch; ++c) {
      const long long c0 = 64LL * c;
      const long long first = ((c0 + p.s - 1) / p.s) * p.s;
      uint64_t m = 0;
      for (long long q = first; q < c0 + 64 && q < p.L; q += p.s) m |= 1ull << (q - c0);
      misc->smask[c] = m;
      misc->fs[c] = first - c0 < 64 ? static_cast<int>(first - c0) : 64;
      misc->cont[c] = (c + 1 < nch) && ((c0 + 64) % p.s != 0);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(&misc->tmem_base, kRssAcc * 64);
    ptx::tmem_relinquish();
  }
  // U_c, K-major, 128-B swizzled: row j (output column) holds U_c[k'][j]
  const uint16_t one = p.in_bf16 ? 0x3F80 : 0x3C00;
  for (int idx = threadIdx.x; idx < nch * 64 * 8; idx += blockDim.x) {
    const int c = idx >> 9, rem = idx & 511;
    const int j = rem >> 3, pos = rem & 7;
    const int lc = pos ^ (j & 7);
    const long long cj = 64LL * c + j;
    __align__(16) uint16_t h[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int kk = lc * 8 + e;
      const long long ck = 64LL * c + kk;
      h[e] = (ck < p.L && cj < p.L && kk <= j && ck / p.s == cj / p.s) ? one : 0;
    }
    *reinterpret_cast<uint4*>(smem + kRssOffB + c * 8192 + j * 128 + pos * 16) =
        *reinterpret_cast<uint4*>(h);
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = misc->tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = p.evict_normal ? ptx::policy_evict_normal() : ptx::policy_evict_first();
      int i = 0;
      for (long long b = b_begin; b < b_end; ++b)
        for (int c = 0; c < nch; ++c, ++i) {
          const int st = i % kRssStages;
          ptx::mbar_wait(&misc->empty[st], ((i / kRssStages) & 1) ^ 1u);
          ptx::mbar_arrive_expect_tx(&misc->full[st], kTileBytes);
          ptx::tma_load_2d(&tin, smem + st * kTileBytes, &misc->full[st], 64 * c,
                           static_cast<int32_t>(b * kTileRows), pol);
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc =
          ptx::idesc_f16_f32(128, 64) | (p.in_bf16 ? ((1u << 7) | (1u << 10)) : 0u);
      int i = 0;
      for (long long b = b_begin; b < b_end; ++b)
        for (int c = 0; c < nch; ++c, ++i) {
          const int st = i % kRssStages;
          const int a = i % kRssAcc;
          ptx::mbar_wait(&misc->tempty[a], ((i / kRssAcc) & 1) ^ 1u);
          ptx::mbar_wait(&misc->full[st], (i / kRssStages) & 1);
          ptx::tc_fence_after();
          const uint64_t adesc = ptx::smem_desc_sw128(smem + st * kTileBytes);
          const uint64_t bdesc = ptx::smem_desc_sw128(smem + kRssOffB + c * 8192);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            ptx::mma_f16_ss(tmem + a * 64, adesc + 2 * kk, bdesc + 2 * kk, idesc,
                            kk > 0 ? 1u : 0u);
          ptx::mma_commit(&misc->empty[st]);
          ptx::mma_commit(&misc->tfull[a]);
        }
    }
    __syncwarp();
  } else {
    const int qd = warp & 3;
    const int rit = qd * 32 + lane;
    const int et = threadIdx.x - 64;
    const bool leader = (et == 0);
    const uint32_t lane_base = static_cast<uint32_t>(qd * 32) << 16;
    const bool excl = p.exclusive != 0;
    int i = 0;
    for (long long b = b_begin; b < b_end; ++b) {
      float carry = 0.f;  // inclusive value of the segment continuing into chunk c
      for (int c = 0; c < nch; ++c, ++i) {
        const int a = i % kRssAcc;
        const int par = i & 1;
        ptx::mbar_wait_warp(&misc->tfull[a], (i / kRssAcc) & 1);
        ptx::tc_fence_after();
        uint32_t r[64];
        {
          uint32_t(&r0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[0]);
          uint32_t(&r1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[32]);
          ptx::tmem_ld_32x32b<32>(tmem + lane_base + a * 64, r0);
          ptx::tmem_ld_32x32b<32>(tmem + lane_base + a * 64 + 32, r1);
        }
        ptx::tmem_wait_ld();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&misc->tempty[a]);
        // uniform chunk geometry: the first segment start at or after column
        // 64c (fs, 64 = none in this chunk), segment starts as a bit mask,
        // and whether the chunk's last segment continues into chunk c + 1
        const long long c0 = 64LL * c;
        const int fs = misc->fs[c];
        const uint64_t smask = misc->smask[c];
        const bool cont = misc->cont[c] != 0;
        float v[64];
#pragma unroll
        for (int j = 0; j < 64; ++j) v[j] = __uint_as_float(r[j]) + (j < fs ? carry : 0.f);
        const float last = v[63];
        if (excl) {
          const uint32_t mlo = static_cast<uint32_t>(smask), mhi = static_cast<uint32_t>(smask >> 32);
#pragma unroll
          for (int j = 63; j >= 0; --j) {
            const bool st = ((j < 32 ? mlo : mhi) >> (j & 31)) & 1u;
            v[j] = st ? 0.f : (j ? v[j - 1] : carry);
          }
        }
        carry = cont ? last : 0.f;
        // stage (swizzled, as the output tensor map's SW128 box) and store
        if (leader) ptx::bulk_wait_read<1>();
        ptx::named_bar_sync(kEpiBar, kEpiThreads);
        uint8_t* stg = smem + rss_off_out<OutT>() + par * kOutBytes;
        const uint32_t rb = static_cast<uint32_t>(rit) * 128u;
        const uint32_t sw = static_cast<uint32_t>(rit & 7);
        if constexpr (sizeof(OutT) == 2) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            uint4 w;
            __half2 h0 = __floats2half2_rn(v[8 * q + 0] + 0.f, v[8 * q + 1] + 0.f);
            __half2 h1 = __floats2half2_rn(v[8 * q + 2] + 0.f, v[8 * q + 3] + 0.f);
            __half2 h2 = __floats2half2_rn(v[8 * q + 4] + 0.f, v[8 * q + 5] + 0.f);
            __half2 h3 = __floats2half2_rn(v[8 * q + 6] + 0.f, v[8 * q + 7] + 0.f);
            w.x = *reinterpret_cast<uint32_t*>(&h0);
            w.y = *reinterpret_cast<uint32_t*>(&h1);
            w.z = *reinterpret_cast<uint32_t*>(&h2);
            w.w = *reinterpret_cast<uint32_t*>(&h3);
            *reinterpret_cast<uint4*>(stg + rb + ((q ^ sw) << 4)) = w;
          }
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              float4 w = make_float4(v[32 * h + 4 * q] + 0.f, v[32 * h + 4 * q + 1] + 0.f,
                                     v[32 * h + 4 * q + 2] + 0.f, v[32 * h + 4 * q + 3] + 0.f);
              *reinterpret_cast<float4*>(stg + h * 16384 + rb + ((q ^ sw) << 4)) = w;
            }
          }
        }
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(kEpiBar, kEpiThreads);
        if (leader) {
          const int32_t r0 = static_cast<int32_t>(b * kTileRows);
          if constexpr (sizeof(OutT) == 2) {
            ptx::tma_store_2d(&tout, stg, static_cast<int32_t>(c0), r0);
          } else {
            ptx::tma_store_2d(&tout, stg, static_cast<int32_t>(c0), r0);
            if (c0 + 32 < p.L) ptx::tma_store_2d(&tout, stg + 16384, static_cast<int32_t>(c0 + 32), r0);
          }
          ptx::bulk_commit();
        }
      }
    }
    if (leader) ptx::bulk_wait<0>();
    // the tail past R rows (< L elements): scanned in fp64 by the last CTA
    if (blockIdx.x == gridDim.x - 1) {
      const long long base = p.R * p.L;
      const long long ntail = (p.n - base + p.s - 1) / p.s;
      OutT* out = reinterpret_cast<OutT*>(p.out);
      for (long long j = et; j < ntail; j += kEpiThreads) {
        const long long lo = base + j * p.s;
        const long long hi = lo + p.s < p.n ? lo + p.s : p.n;
        double run = 0.0;
        for (long long e = lo; e < hi; ++e) {
          const double y = in_to_float(p.x, e, p.in_bf16 != 0);
          if (excl) {
            out[e] = cvt_out_d<OutT>(run + 0.0);
            run += y;
          } else {
            run += y;
            out[e] = cvt_out_d<OutT>(run + 0.0);
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kRssAcc * 64);
  }
}


// =====================================================================
// Irregular (CSR) segmented reduce, tile-parallel epilogue.
//
// The MMA is the scan's X.U64 (in-row inclusive prefixes in TMEM), as in
// MODE_IRREG; what changes is how the epilogue finds and closes segments:
//
//  * a small pre-pass (irreg_k0_kernel, one coalesced read of the offsets)
//    writes k0[t] = lower_bound(offsets, 8192 t) for every tile, so each
//    tile knows its start range [k0[t], k0[t+1]) without searching;
//  * kIrNG independent epilogue GROUPS (4 warps each, one per TMEM lane
//    quadrant) take the CTA's tiles round-robin, each with its own SMEM
//    staging of the in-row prefixes, offsets and named barrier, so kIrNG
//    tiles are in the epilogue at once (the single group's per-tile latency
//    bounded the previous design at ~50 % of copy bandwidth);
//  * nothing flows between tiles inside the epilogue: a tile writes the
//    segments that start and end in it, plus a record (head = value before
//    its first start, tail = value after its last start, or its total), and
//    after the range one warp composes the records in tile order
//    (a segmented pair scan) to close the segments that cross tiles.  The
//    range-crossing segments use the deterministic last-CTA fixup of the
//    regular reduce.
//
// Numerics are those of MODE_IRREG: a segment inside one row is
// P(b) - P(a) of fp32 in-row prefixes, a longer one adds an fp64 prefix of
// row totals; tile and range carries are fp64.  The pre-pass table and the
// records are re-zeroed after use (the workspace region is shared with the
// CHUNK scan's epoch-tagged look-back words).
#ifndef TC_IR_NG
#define TC_IR_NG 3
#endif
constexpr int kIrNG = TC_IR_NG;  // epilogue groups (build-time: 3 measured best with 4 stages)
constexpr int kIrStages = 4;
constexpr int kIrAcc = 8;       // TMEM slots (64 columns each)
constexpr int kIrThreads = 64 + kIrNG * kEpiThreads;
constexpr int kIrCap = 256;     // offsets staged in SMEM per tile (more: read from L2)
constexpr uint32_t kIrOffB = kIrStages * kTileBytes;
constexpr uint32_t kIrOffScr = kIrOffB + 64 * 128;
constexpr int kIrRowF = 68;     // staging row stride in floats (conflict-free 16-B stores)
constexpr uint32_t kIrScrBytes = kTileRows * kIrRowF * 4;
constexpr uint32_t kIrOffMisc = kIrOffScr + kIrNG * kIrScrBytes;
constexpr uint32_t kIrFinalBar = 1 + kIrNG;  // named barrier of all epilogue groups

struct IrRec {  // one tile's carry record
  double h;       // sum before the first start (closes segment seg0)
  double v;       // sum after the last start, or the whole tile (f == 0)
  long long seg0; // k0[t] - 1
  long long f;    // the tile holds a start
};
struct IrMisc {
  uint64_t full[kIrStages];
  uint64_t empty[kIrStages];
  uint64_t tfull[kIrAcc];
  uint64_t tempty[kIrAcc];
  uint32_t tmem_base;
  int is_last;
  float wsum[kIrNG][2][4];
  double wtot[kIrNG][2][4];
  double rex[kIrNG][kTileRows];  // exclusive fp64 prefix of row totals within the row's warp
  long long so[kIrNG][kIrCap];
};
constexpr uint32_t kIrSmem = kIrOffMisc + sizeof(IrMisc) + 1024;
#ifdef TC_IRREG_TRACE
// phase timestamps of CTA 0's group leaders (debug builds: -DTC_IRREG_TRACE)
__device__ long long g_irtrace[kIrNG][64][8];
#define IR_TRACE(ph) \
  if (cta == 0 && leader && it < 64) g_irtrace[g][it][ph] = clock64();
#else
#define IR_TRACE(ph)
#endif

__global__ void irreg_k0_kernel(const long long* __restrict__ offs, long long nseg, long long T,
                                long long* __restrict__ k0) {
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k > nseg) return;
  const long long o = __ldg(offs + k);
  long long tlo = 0;
  if (k > 0) {
    const long long op = __ldg(offs + k - 1);
    tlo = (op < 0 ? -1 : op / kTileElems) + 1;
  }
  long long thi = o < 0 ? -1 : o / kTileElems;
  if (thi > T - 1) thi = T - 1;
  for (long long t = tlo; t <= thi; ++t) k0[t] = k;
  if (k == nseg) k0[T] = nseg + 1;
}

template <typename OutT>
__global__ void __launch_bounds__(kIrThreads, 1)
    irreg_reduce_kernel(const __grid_constant__ CUtensorMap tin, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  IrMisc* misc = reinterpret_cast<IrMisc*>(smem + kIrOffMisc);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const long long T = p.num_tiles;
  const int Gc = gridDim.x;
  const int cta = blockIdx.x;
  const long long t_begin = T * cta / Gc, t_end = T * (cta + 1) / Gc;
  const int ntl = static_cast<int>(t_end - t_begin);
  IrRec* rec = reinterpret_cast<IrRec*>(p.trec);

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tin);
    for (int s = 0; s < kIrStages; ++s) {
      ptx::mbar_init(&misc->full[s], 1);
      ptx::mbar_init(&misc->empty[s], 1);
    }
    for (int a = 0; a < kIrAcc; ++a) {
      ptx::mbar_init(&misc->tfull[a], 1);
      ptx::mbar_init(&misc->tempty[a], 4);  // lane 0 of the group's 4 warps
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(&misc->tmem_base, 512);
    ptx::tmem_relinquish();
  }
  build_b<OP_SCAN, 1, 64>(smem + kIrOffB, p.in_bf16 ? 0x3F80 : 0x3C00);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = misc->tmem_base;

  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0) {
      const uint64_t pol = ptx::policy_evict_first();
      for (int i = 0; i < ntl; ++i) {
        const int s = i % kIrStages;
        ptx::mbar_wait(&misc->empty[s], ((i / kIrStages) & 1) ^ 1u);
        ptx::mbar_arrive_expect_tx(&misc->full[s], kTileBytes);
        ptx::tma_load_2d(&tin, smem + s * kTileBytes, &misc->full[s], 0,
                         static_cast<int32_t>((t_begin + i) * kTileRows), pol);
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer: X.U64 per tile =================
    if (lane == 0) {
      const uint32_t idesc = ptx::idesc_f16_f32(128, 64) | (p.in_bf16 ? ((1u << 7) | (1u << 10)) : 0u);
      const uint64_t bdesc = ptx::smem_desc_sw128(smem + kIrOffB);
      for (int i = 0; i < ntl; ++i) {
        const int s = i % kIrStages;
        const int a = i % kIrAcc;
        ptx::mbar_wait(&misc->tempty[a], ((i / kIrAcc) & 1) ^ 1u);
        ptx::mbar_wait(&misc->full[s], (i / kIrStages) & 1);
        ptx::tc_fence_after();
        const uint64_t adesc = ptx::smem_desc_sw128(smem + s * kTileBytes);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          ptx::mma_f16_ss(tmem + a * 64, adesc + 2 * k, bdesc + 2 * k, idesc, k > 0 ? 1u : 0u);
        ptx::mma_commit(&misc->empty[s]);
        ptx::mma_commit(&misc->tfull[a]);
      }
    }
    __syncwarp();
  } else {
    // ================= epilogue groups =================
    const int g = (warp - 2) >> 2;
    const int qd = warp & 3;           // TMEM lane quadrant
    const int rit = qd * 32 + lane;    // row in tile
    const int et = threadIdx.x - 64 - g * kEpiThreads;
    const bool leader = (et == 0);
    const uint32_t bar = 1 + g;
    const uint32_t lane_base = static_cast<uint32_t>(qd * 32) << 16;
    float* scr = reinterpret_cast<float*>(smem + kIrOffScr + g * kIrScrBytes);
    long long* so = misc->so[g];
    double* rex = misc->rex[g];
    OutT* out = reinterpret_cast<OutT*>(p.out);
    constexpr long long kNoStart = 1LL << 62;
    const long long kmax = p.nseg + 1;
    auto ldk0 = [&](int i) -> long long {  // k0 of local tile i (i <= ntl); clamped at use
      return __ldg(p.tk0 + t_begin + i);
    };
    auto clampk = [&](long long v) -> long long { return v < 0 ? 0 : (v > kmax ? kmax : v); };
    auto ldoff = [&](long long k, long long lim) -> long long {
      return k < lim ? __ldg(p.offs + k) : kNoStart;
    };
    // pipeline: this tile's range and first offsets, the next tile's range
    // (k0 only: its offsets are loaded one tile ahead)
    int i = g;
    long long kA = 0, kB = 0, o0 = kNoStart, o1 = kNoStart, nA = 0, nB = 0;
    if (i < ntl) {
      kA = clampk(ldk0(i));
      kB = clampk(ldk0(i + 1));
      if (kB < kA) kB = kA;
      o0 = ldoff(kA + et, kB);
      o1 = ldoff(kA + et + kEpiThreads, kB);
      if (i + kIrNG < ntl) {
        nA = ldk0(i + kIrNG);  // raw: clamped when used, a tile later (no wait here)
        nB = ldk0(i + kIrNG + 1);
      }
    }
    for (int it = 0; i < ntl; i += kIrNG, ++it) {
      const long long t = t_begin + i;
      // prefetch: the next tile's offsets, the tile after's range
      long long n0 = kNoStart, n1 = kNoStart, mA = 0, mB = 0;
      if (i + kIrNG < ntl) {
        nA = clampk(nA);
        nB = clampk(nB);
        if (nB < nA) nB = nA;
        n0 = ldoff(nA + et, nB);
        n1 = ldoff(nA + et + kEpiThreads, nB);
        if (i + 2 * kIrNG < ntl) {  // raw loads: clamped a tile later
          mA = ldk0(i + 2 * kIrNG);
          mB = ldk0(i + 2 * kIrNG + 1);
        }
      }
      const int a = i % kIrAcc;
      const int par = it & 1;
      IR_TRACE(0)
      ptx::mbar_wait_warp(&misc->tfull[a], static_cast<uint32_t>((i / kIrAcc) & 1));
      ptx::tc_fence_after();
      IR_TRACE(1)
      uint32_t r[64];
      {
        uint32_t(&r0)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[0]);
        uint32_t(&r1)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[32]);
        ptx::tmem_ld_32x32b<32>(tmem + lane_base + a * 64, r0);
        ptx::tmem_ld_32x32b<32>(tmem + lane_base + a * 64 + 32, r1);
      }
      ptx::tmem_wait_ld();
      IR_TRACE(2)
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&misc->tempty[a]);
      float vv[64];
#pragma unroll
      for (int k = 0; k < 64; ++k) vv[k] = __uint_as_float(r[k]);
      const long long row = t * kTileRows + rit;
      if (row == p.rows_full) {  // ragged last row: outside the TMA view, recompute from HBM
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < 64; ++k) {
          const long long e = row * kRow + k;
          s += (e < p.n) ? in_to_float(p.x, e, p.in_bf16 != 0) : 0.f;
          vv[k] = s;
        }
      }
      const long long starts = kB - kA;
      if (starts == 0) {
        // no start in the tile: its total continues the open segment
        const float ws = warp_sum(vv[63]);
        if (lane == 0) misc->wsum[g][par][qd] = ws;
        ptx::named_bar_sync(bar, kEpiThreads);
        if (leader) {
          const float* w = misc->wsum[g][par];
          IrRec q;
          q.h = 0.0;
          q.v = static_cast<double>((w[0] + w[1]) + (w[2] + w[3]));
          q.seg0 = kA - 1;
          q.f = 0;
          rec[t] = q;
        }
      } else {
        // stage the row prefixes, the row totals' fp64 prefix and the offsets
        float* srow = scr + rit * kIrRowF;
#pragma unroll
        for (int j = 0; j < 16; ++j)
          *reinterpret_cast<float4*>(srow + 4 * j) =
              make_float4(vv[4 * j], vv[4 * j + 1], vv[4 * j + 2], vv[4 * j + 3]);
        IR_TRACE(7)
        const double tr = static_cast<double>(vv[63]);
        double incl = tr;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const double u = __shfl_up_sync(kFull, incl, d);
          if (lane >= d) incl += u;
        }
        rex[rit] = incl - tr;
        if (lane == 31) misc->wtot[g][par][qd] = incl;
        so[et] = o0;
        so[et + kEpiThreads] = o1;
        IR_TRACE(3)
        ptx::named_bar_sync(bar, kEpiThreads);
        IR_TRACE(4)
        const double* wt = misc->wtot[g][par];
        const double wo1 = wt[0], wo2 = wo1 + wt[1], wo3 = wo2 + wt[2], tot = wo3 + wt[3];
        const long long tb = t * kTileElems;
        auto tpos = [&](long long o) -> int {  // position in the tile, clamped to [0, 8192]
          const long long q = o - tb;
          return static_cast<int>(q < 0 ? 0 : (q > kTileElems ? kTileElems : q));
        };
        auto prow = [&](int q) -> float {  // in-row prefix before position q
          const int c = q & 63;
          return c ? scr[(q >> 6) * kIrRowF + c - 1] : 0.f;
        };
        auto rpre = [&](int rr) -> double {  // tile prefix of row totals before row rr (0..128)
          const int w = rr >> 5;
          const double wo = w == 0 ? 0.0 : w == 1 ? wo1 : w == 2 ? wo2 : w == 3 ? wo3 : tot;
          return rr >= kTileRows ? tot : wo + rex[rr];
        };
        auto offk = [&](long long j) -> long long {  // offset kA + j
          return j < kIrCap ? so[j] : __ldg(p.offs + kA + j);
        };
        // segments that start and end in the tile: same row -> P(b) - P(a) in
        // fp32, else the fp64 tile prefix of row totals joins in
        for (long long j = et; j + 1 < starts; j += kEpiThreads) {
          const int qa = tpos(offk(j)), qb = tpos(offk(j + 1));
          if ((qa >> 6) == (qb >> 6)) {
            out[kA + j] = cvt_out<OutT>(prow(qb) - prow(qa));
          } else {
            const double v = (rpre(qb >> 6) - rpre(qa >> 6)) +
                             (static_cast<double>(prow(qb)) - static_cast<double>(prow(qa)));
            out[kA + j] = cvt_out_d<OutT>(v);
          }
        }
        if (et == kEpiThreads / 2) {  // the record: off the segment-0 thread's path
          const int qf = tpos(offk(0)), ql = tpos(offk(starts - 1));
          IrRec q;
          q.h = rpre(qf >> 6) + static_cast<double>(prow(qf));
          q.v = tot - (rpre(ql >> 6) + static_cast<double>(prow(ql)));
          q.seg0 = kA - 1;
          q.f = 1;
          rec[t] = q;
        }
        IR_TRACE(5)
        ptx::named_bar_sync(bar, kEpiThreads);  // staging, offsets and rex are rewritten next tile
        IR_TRACE(6)
      }
      kA = nA;
      kB = nB;
      o0 = n0;
      o1 = n1;
      nA = mA;
      nB = mB;
    }

    // ---- compose the records in tile order: close the segments that cross
    // tiles, and hand the range's first / last open segment to the fixup
    ptx::named_bar_sync(kIrFinalBar, kIrNG * kEpiThreads);
    const long long krange0 = ntl > 0 ? ldk0(0) : 0;
    const long long kend = ntl > 0 ? ldk0(ntl) : 0;
    if (warp == 2) {
      double carry = 0.0;
      long long hseg = -1;
      double hval = 0.0;
      for (int base = 0; base < ntl; base += 32) {
        const int j = base + lane;
        IrRec q{0.0, 0.0, -1, 0};
        if (j < ntl) {
          q.h = __ldcg(&rec[t_begin + j].h);
          q.v = __ldcg(&rec[t_begin + j].v);
          q.seg0 = __ldcg(&rec[t_begin + j].seg0);
          q.f = __ldcg(&rec[t_begin + j].f);
          rec[t_begin + j] = IrRec{0.0, 0.0, 0, 0};
        }
        // inclusive segmented pair scan of (v, f) over the lanes
        double v = q.v;
        int f = static_cast<int>(q.f);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const double pv = __shfl_up_sync(kFull, v, d);
          const int pf = __shfl_up_sync(kFull, f, d);
          if (lane >= d) {
            if (!f) v = pv + v;
            f |= pf;
          }
        }
        double ve = __shfl_up_sync(kFull, v, 1);
        int fe = __shfl_up_sync(kFull, f, 1);
        const double cin = (lane == 0) ? carry : (fe ? ve : carry + ve);
        if (j < ntl && q.f && q.seg0 >= 0) {
          const double val = cin + q.h;
          if (q.seg0 < krange0) {  // began in an earlier CTA's range: a partial
            hseg = q.seg0;
            hval = val;
          } else {
            out[q.seg0] = cvt_out_d<OutT>(val);
          }
        }
        const double vl = __shfl_sync(kFull, v, 31);
        const int fl = __shfl_sync(kFull, f, 31);
        carry = fl ? vl : carry + vl;
      }
      // at most one lane saw the range's head segment
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const long long hs2 = __shfl_xor_sync(kFull, hseg, o);
        const double hv2 = __shfl_xor_sync(kFull, hval, o);
        if (hs2 >= 0) {
          hseg = hs2;
          hval = hv2;
        }
      }
      if (lane == 0) {
        Entry e0{hseg, hval};
        // the range's last start (kend - 1) stays open (its end offset is in a
        // later range); in the last range it is the end offset itself
        Entry e1{(kend - 1 >= 0 && kend - 1 < p.nseg) ? kend - 1 : -1LL, carry};
        p.entries[2 * cta] = e0;
        p.entries[2 * cta + 1] = e1;
        __threadfence();
        const unsigned tk = atomicAdd(&p.hdr->ticket, 1u);
        misc->is_last = (tk == static_cast<unsigned>(Gc - 1));
      }
    }
    // re-zero this range's interior k0 entries (the boundaries are shared
    // with the neighbouring ranges: the last CTA clears them)
    const int ft = threadIdx.x - 64;
    for (long long tt = t_begin + 1 + ft; tt < t_end; tt += kIrNG * kEpiThreads) p.tk0[tt] = 0;
    ptx::named_bar_sync(kIrFinalBar, kIrNG * kEpiThreads);
    if (misc->is_last) {
      __threadfence();
      // deterministic combine of the range partials in CTA order (as the
      // regular reduce's fixup), staged through the idle input ring
      Entry* se = reinterpret_cast<Entry*>(smem);
      const int ne = 2 * Gc;
      for (int k = ft; k < ne; k += kIrNG * kEpiThreads) {
        Entry e;
        e.seg = __ldcg(&p.entries[k].seg);
        e.val = __ldcg(&p.entries[k].val);
        se[k] = e;
      }
      for (int c = ft; c <= Gc; c += kIrNG * kEpiThreads)
        p.tk0[c == Gc ? T : T * c / Gc] = 0;
      ptx::named_bar_sync(kIrFinalBar, kIrNG * kEpiThreads);
      for (int k = ft; k < ne; k += kIrNG * kEpiThreads) {
        const long long sg = se[k].seg;
        if (sg < 0) continue;
        int pk = k - 1;
        while (pk >= 0 && se[pk].seg < 0) --pk;
        if (pk >= 0 && se[pk].seg == sg) continue;  // not the first entry of its run
        double acc = 0.0;
        for (int kk = k; kk < ne; ++kk) {
          const long long s2 = se[kk].seg;
          if (s2 < 0) continue;
          if (s2 != sg) break;
          acc += se[kk].val;
        }
        out[sg] = cvt_out_d<OutT>(acc);
      }
      if (ft == 0) {
        p.hdr->epoch = (p.hdr->epoch + 1u) & 0x3FFFFFFFu;
        p.hdr->ticket = 0u;
        __threadfence();
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// =====================================================================
// host side
// =====================================================================

static thread_local char g_err[512] = "";
static thread_local uint64_t g_launches = 0;

static void set_err(const char* fmt, const char* a = "", long long b = 0) {
  snprintf(g_err, sizeof(g_err), fmt, a, b);
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

struct DevInfo {
  int sms = 0;
  int major = 0;
  bool ok = false;
};
static DevInfo dev_info(int dev) {
  static DevInfo cache[64];
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0 || dev >= 64) return DevInfo{};
  if (!cache[dev].ok) {
    int sms = 0, major = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess)
      return DevInfo{};
    cache[dev].sms = sms;
    cache[dev].major = major;
    cache[dev].ok = true;
  }
  return cache[dev];
}

static bool make_map(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* base,
                     long long rows, int box_cols, long long row_len = kRow,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B,
                     CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(row_len), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_len) * esize};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(kTileRows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// L2 handling of the strided [R x L] row-segment input view.  With more than
// one 64-column chunk per row, each box reads 128 rows of 128 B at a 2L-byte
// pitch, and a pitch that is not a multiple of 128 B makes every piece
// straddle two 128-B lines whose other half belongs to the row's next chunk,
// loaded a few boxes later: evict-first loads drop those halves and they are
// read from HBM twice.  Measured on B200 (2^30 fp16, % of copy bandwidth;
// tools/probe_modes.py with PROBE_AB_R=multi, profiles/r02/rowseg_l2/):
//   (promotion, policy)          (256 B, first) (none, first) (256 B, normal)
//   reduce s = 9 / 17 / 33 f16        79 / 82 / 82   84 / 86 / 82   98 / 97 / 94
//   reduce s = 3 / 7 (one chunk)      88 / 80        91 / 82        59 / 51
//   reduce s = 49 / 100 / 300 f16     92 / 98 / 94   87 / 91 / 86   80 / 96 / 82
//   scan f16 s = 3 / 17 / 33          81 / 69 / 67   86 / 72 / 71   89 / 82 / 82
//   reduce s = 49 / 63 / 65 f32 (twice)  74 / 78 / 77   76 / 78 / 77   82 / 88 / 86
// so: one chunk per row (contiguous boxes) -> no promotion, evict-first;
// scans, reduces with s < 48 and fp32 / fp64-output reduces -> 256-B
// promotion, evict-normal; fp16-output reduces with s >= 48 -> 256-B
// promotion, evict-first.  TC_RS_PROMO (0 / 64 / 128 /
// 256) and TC_RS_EVICT (0 / 1) override (A/B switches).
struct RsL2 {
  CUtensorMapL2promotion promo;
  int evict_normal;
};
static RsL2 rs_l2(bool scan, long long s, int nchunk, int out_esize = 2) {
  int promo = 256, normal = 0;
  if (nchunk <= 1) {
    promo = 0;
  } else if (scan || s < 48 || out_esize >= 4) {
    normal = 1;
  }
  if (const char* e = getenv("TC_RS_PROMO")) promo = atoi(e);
  if (const char* e = getenv("TC_RS_EVICT")) normal = atoi(e) == 1 ? 1 : 0;
  RsL2 r;
  r.promo = promo == 0     ? CU_TENSOR_MAP_L2_PROMOTION_NONE
            : promo == 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
            : promo == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                           : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  r.evict_normal = normal;
  return r;
}

static long long gcd_ll(long long a, long long b) {
  while (b) {
    long long t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// Segments per row for MODE_ROWSEG (0 = not applicable).  k is a power of
// two times 8 / gcd(s, 8) (row pitch a multiple of 16 B), k outputs of at
// most kRsMaxRowBytes per row (measured: 64 outputs per row ran at 54-63 %), with
// the per-chunk B matrices within kRsMaxB; among those, the k with the
// fewest 64-column chunks per element (a partly filled last chunk costs a
// whole chunk's pipeline slot; measured on B200: rows of 40 elements run at
// ~42 % of copy bandwidth, whole 64-column chunks at ~90 %).
// TC_RS_TIE=1: among equally filled layouts take the longest rows (A/B switch)
static bool rs_tie_longer() {
  const char* e = getenv("TC_RS_TIE");
  return e && atoi(e) == 1;
}
static int rowseg_k(long long s, long long n, int out_esize) {
  if (s < 2 || s >= n) return 0;
  if (gcd_ll(s, 64) > 8) return 0;  // >= 16-element granules: the GENERAL kernel is as fast
  int best = 0;
  double best_cost = 0.0;
  for (long long k = 8 / gcd_ll(s, 8); k * out_esize <= kRsMaxRowBytes; k *= 2) {
    const long long L = k * s;
    const long long nch = (L + kRow - 1) / kRow;
    const long long nn = k < 16 ? 16 : k;
    if (nch * nn * 128 > static_cast<long long>(kRsMaxB)) break;
    const double cost = static_cast<double>(nch) / static_cast<double>(L);
    if (best == 0 || cost < best_cost * (1.0 - 1e-9) ||
        (rs_tie_longer() && cost < best_cost * (1.0 + 1e-9))) {
      best = static_cast<int>(k);
      best_cost = cost;
    }
  }
  return best;
}

// Segments per row for the MODE_ROWSEG scan (0 = not applicable): rows of
// L = k s <= 64 rss_max_chunks elements, k a power of two times 8 / gcd(s, 8),
// the fewest chunks per element.  Only where it beats the granule scan
// (measured on B200, 2^30 fp16, % of copy bandwidth): s < 64 (larger s run
// as MODE_SPLIT), gcd(s, 64) <= 2 (gcd 4: GENERAL 88 % vs 61-83 %); with
// fp32 output GENERAL wins for gcd 2 (88 vs 71-80 %) and for odd s > 9
// (73 vs 67-71 %).
static bool split_enabled();
static bool splitm_wins(long long s, int out_esize);
constexpr long long kSplitMMin = 9;  // >= 9: at most one start per granule of 8
static int rowseg_scan_k(long long s, long long n, int out_esize) {
  if (s < 2 || s >= n || s >= kRow) return 0;
  const char* all = getenv("TC_RSS_ALL");  // probe switch: ROWSEG for every s < 64 with gcd <= 2
  const bool force = all && atoi(all) == 1;
  if (!force && split_enabled() && splitm_wins(s, out_esize)) return 0;  // MODE_SPLITM
  const long long g = gcd_ll(s, 64);
  if (g > 2) return 0;
  if (!force && out_esize == 4 && (g == 2 || s > 9)) return 0;
  int best = 0;
  double best_cost = 0.0;
  // among layouts of equal cost, rows of whole 32-B sectors (L % 16 == 0):
  // a row pitch ending mid-sector makes every strided box write partial
  // sectors (measured, fp16 out: s = 23 / 29 / 31 / 39 80 / 77 / 80 / 78 ->
  // 85 / 82 / 82 / 79 %); TC_RSS_ALIGN32=0 turns the preference off
  const char* al = getenv("TC_RSS_ALIGN32");
  const bool prefer_aligned = !(al && al[0] == '0');
  const long long lmax = 64LL * rss_max_chunks(out_esize);
  bool best_al = false;
  for (long long k = 8 / gcd_ll(s, 8); k * s <= lmax; k *= 2) {
    const long long L = k * s;
    const double cost = static_cast<double>((L + kRow - 1) / kRow) / static_cast<double>(L);
    const bool aligned = prefer_aligned && (L % 16 == 0);
    if (best == 0 || cost < best_cost * (1.0 - 1e-9) ||
        (aligned && !best_al && cost < best_cost * (1.0 + 1e-9))) {
      best = static_cast<int>(k);
      best_cost = cost;
      best_al = aligned;
    }
  }
  return best;
}

// CHUNK arrays: units u = j*Gc + c < T + kMaxCtas, chunks j < T
static long long chunk_slots(long long n) { return (n + kTileElems - 1) / kTileElems + kMaxCtas; }

// IRREG reduce scratch after the look-back region start: the per-tile k0
// table (T + 1 entries) and the per-tile carry records
static size_t irreg_k0_bytes(long long n) {
  const long long T = (n + kTileElems - 1) / kTileElems;
  return ((static_cast<size_t>(T + 1) * sizeof(long long)) + 255) & ~size_t(255);
}
static size_t ws_need(int op, long long n, long long seg) {
  size_t b = kWsLookback;
  if (op == TC_OP_REDUCE)  // (irregular segments; small next to the data: 40 B per 16-KB tile)
    b += irreg_k0_bytes(n) + sizeof(IrRec) * static_cast<size_t>((n + kTileElems - 1) / kTileElems) + 256;
  if (op == TC_OP_SCAN)
    b += static_cast<size_t>(chunk_slots(n)) * 2 * sizeof(uint64_t) + 64;
  if (op == TC_OP_BN_STATS)  // per-(n, c) shifted moments (S1, S2) + per-channel tickets, cleared after use
    b += (2 * sizeof(double) + sizeof(unsigned)) * static_cast<size_t>((n + seg - 1) / (seg > 0 ? seg : 1)) + 512;
  return (b + 255) & ~size_t(255);
}

// CHUNK unit size: K tiles per CTA per chunk.  A unit's tiles stay in TMEM
// from its A pass to its O pass, one unit later, so two units must fit the
// 8 TMEM tile slots: K <= 4 (K = 2 leaves a third unit for the MMA to fill
// meanwhile).  TC_CHUNK_TILES overrides (tuning).
static long long chunk_tiles(long long T, long long grid) {
  const char* e = getenv("TC_CHUNK_TILES");
  long long k = (e && atoll(e) > 0) ? atoll(e) : 2;
  if (k > 4) k = 4;
  const long long fair = T / (grid > 0 ? grid : 1);
  if (k > fair) k = fair;
  return k < 1 ? 1 : k;
}

// CHUNK lag L: O(j) runs after A(j+L), so the cross-CTA wait for unit j's
// entry value has L units of slack.  Units j..j+L must all be resident in
// the 8 TMEM tile slots, (L + 1) * K <= 8 (else A(j+L) would wait for a slot
// only O(j) frees: deadlock).  Measured on B200 (2^30, fp32 out): K = 2,
// L = 3 is best; L = 1 leaves the ~5 us publish-to-observe latency under
// full HBM load exposed.
static long long chunk_lag(long long k) {
  const long long lmax = 8 / k - 1;
  const char* e = getenv("TC_CHUNK_LAG");
  long long l = (e && atoll(e) > 0) ? atoll(e) : lmax;
  if (l > lmax) l = lmax;
  return l < 1 ? 1 : l;
}

template <int OP, int GR, int MODE, typename OutT>
static int launch(const Params& p0, int out_esize, cudaStream_t st) {
  constexpr uint32_t smem = smem_bytes<OP, GR, MODE, OutT>();
  static_assert(smem <= 232448, "shared memory budget");
  auto kern = seg_kernel<OP, GR, MODE, OutT>;
  int dev = 0;
  cudaGetDevice(&dev);
  // function attributes are per device: set them once on each device used
  static std::atomic<uint64_t> attr_done{0};
  const uint64_t dev_bit = 1ull << (dev & 63);
  if (!(attr_done.load() & dev_bit)) {
    // max shared-memory carveout, so MINB = 2 kernels really get 2 CTAs/SM
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
        cudaSuccess) {
      set_err("cudaFuncSetAttribute failed: %s%lld", cudaGetErrorString(cudaGetLastError()), 0);
      return TC_CUDA_ERROR;
    }
    attr_done.fetch_or(dev_bit);
  }
  DevInfo di = dev_info(dev);
  if (!di.ok || di.major < 10) {
    set_err("no sm_100 device (compute capability major %s%lld)", "", di.major);
    return TC_NO_DEVICE;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg<OP, GR, MODE, OutT>::THREADS, smem) !=
          cudaSuccess ||
      per_sm < 1) {
    set_err("occupancy query failed: %s%lld", cudaGetErrorString(cudaGetLastError()), 0);
    return TC_CUDA_ERROR;
  }
  // CTAs per SM.  The occupancy API reports 1 for these kernels (it appears
  // to budget a full TMEM allocation per CTA), but two CTAs do co-reside,
  // and measured on B200 (2^30 fp16) a second epilogue per SM pays off where
  // the per-tile epilogue is latency-heavy: the cross-row-group combine of
  // reduce ROWS with >= 16 rows per segment (s = 1024/4096: 92-93 % -> 99 %
  // of copy bandwidth) and the pair scans of GENERAL (s = 300: reduce 26 ->
  // 47 %, scan 70 -> 85 %; GENERAL reduce with 8..32 granules per row takes
  // 3, see Cfg::MINB), and fp32-output scans of tiny segments (85 ->
  // 89 %).  Elsewhere one CTA/SM is as fast or faster (reduce TILES 100 vs
  // 97 %, fp16 scans 93-95 vs 91-92 %); cooperative launches (CHUNK) must
  // match the API.
  if (MODE != MODE_CHUNK) {
    per_sm = (MODE == MODE_GSCR) ? 2
             : (MODE == MODE_GENERAL || MODE == MODE_IRREG || MODE == MODE_SPLIT ||
                MODE == MODE_SPLITM)
                 ? Cfg<OP, GR, MODE, OutT>::MINB
             : ((OP == OP_REDUCE && MODE == MODE_ROWS && p0.log2m >= 4 && p0.log2m < 7) ||
                (OP == OP_SCAN && MODE == MODE_LOCAL && sizeof(OutT) == 4))
                 ? 2
                 : 1;
    if (per_sm > Cfg<OP, GR, MODE, OutT>::MINB) per_sm = Cfg<OP, GR, MODE, OutT>::MINB;
  } else if (per_sm > 1) {
    per_sm = 1;
  }
  if (const char* e = getenv("TC_CTAS_PER_SM")) {  // tuning override
    const int want = atoi(e);
    if (want >= 1 && want <= Cfg<OP, GR, MODE, OutT>::MINB && MODE != MODE_CHUNK) per_sm = want;
  }
  long long grid = static_cast<long long>(di.sms) * per_sm;
  if (grid > p0.num_tiles) grid = p0.num_tiles;
  if (grid > kMaxCtas) grid = kMaxCtas;
  if (MODE == MODE_CHUNK && grid > 256) grid = 256;  // prefix warp reads <= 8 units per lane
  if (grid < 1) grid = 1;

  Params p = p0;
  if (MODE == MODE_CHUNK) {
    p.ck = chunk_tiles(p.num_tiles, grid);
    p.lag = chunk_lag(p.ck);
  }
  CUtensorMap tin, tout;
  const char* wsb = reinterpret_cast<const char*>(p.hdr);
  const void* in_base = p.rows_full > 0 ? static_cast<const void*>(p.x)
                                        : static_cast<const void*>(wsb + kWsZeroRow);
  if (!make_map(&tin, p.in_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                2, in_base,
                p.rows_full > 0 ? p.rows_full : 1, kRow)) {
    set_err("cuTensorMapEncodeTiled (input) failed%s%lld", "", 0);
    return TC_CUDA_ERROR;
  }
  if (OP == OP_SCAN) {
    const void* ob = p.rows_full > 0 ? p.out : static_cast<const void*>(wsb + kWsDummyOut);
    const bool ok = (out_esize == 2)
                        ? make_map(&tout, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, ob,
                                   p.rows_full > 0 ? p.rows_full : 1, kRow)
                        : make_map(&tout, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, ob,
                                   p.rows_full > 0 ? p.rows_full : 1, 32);
    if (!ok) {
      set_err("cuTensorMapEncodeTiled (output) failed%s%lld", "", 0);
      return TC_CUDA_ERROR;
    }
  } else {
    tout = tin;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(Cfg<OP, GR, MODE, OutT>::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  int na = 0;
  if (MODE == MODE_CHUNK) {
    // the cross-CTA spin-waits need every CTA resident: cooperative launch
    // guarantees co-residency (or fails loudly instead of deadlocking).
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    na = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (MODE == MODE_IRREG && OP == OP_SCAN) {
    // pass 1: the carry each CTA range hands on (same range split as below)
    irreg_tail_kernel<<<static_cast<unsigned>(grid), kTailThreads, 0, st>>>(p.x, p.in_bf16, p.n, p.offs,
                                                                  p.nseg, p.num_tiles, p.entries);
    const cudaError_t e1 = cudaGetLastError();
    if (e1 != cudaSuccess) {
      set_err("kernel launch failed: %s%lld", cudaGetErrorString(e1), 0);
      return TC_CUDA_ERROR;
    }
    ++g_launches;
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tin, tout, p);
  if (e != cudaSuccess) {
    set_err("kernel launch failed: %s%lld", cudaGetErrorString(e), 0);
    return TC_CUDA_ERROR;
  }
  ++g_launches;
  return TC_OK;
}

template <typename OutT, int KS>
static int launch_rowseg_k(const RsParams& p0, void* ws, cudaStream_t st) {
  auto kern = rowseg_reduce_kernel<OutT, KS>;
  int dev = 0;
  cudaGetDevice(&dev);
  static std::atomic<uint64_t> attr_done{0};
  const uint64_t dev_bit = 1ull << (dev & 63);
  if (!(attr_done.load() & dev_bit)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kRsSmemMax) !=
        cudaSuccess) {
      set_err("cudaFuncSetAttribute failed: %s%lld", cudaGetErrorString(cudaGetLastError()), 0);
      return TC_CUDA_ERROR;
    }
    attr_done.fetch_or(dev_bit);
  }
  const DevInfo di = dev_info(dev);
  if (!di.ok || di.major < 10) {
    set_err("no sm_100 device (compute capability major %s%lld)", "", di.major);
    return TC_NO_DEVICE;
  }
  RsParams p = p0;
  long long grid = 2LL * di.sms;  // 2 CTAs / SM (4-stage ring + B matrices)
  if (grid > p.nblk) grid = p.nblk;
  if (grid < 1) grid = 1;
  CUtensorMap tin;
  const char* wsb = reinterpret_cast<const char*>(ws);
  const bool ok = p.R > 0
      ? make_map(&tin, p.in_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                 2, p.x, p.R, kRow, p.L, CU_TENSOR_MAP_SWIZZLE_128B, rs_l2(false, p.s, p.nchunk).promo)
      : make_map(&tin, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, wsb + kWsZeroRow, 1, kRow);
  if (!ok) {
    set_err("cuTensorMapEncodeTiled (row-segment input) failed%s%lld", "", 0);
    return TC_CUDA_ERROR;
  }
  constexpr int kRowBytes = KS * static_cast<int>(sizeof(OutT));
  CUtensorMap tout = tin;
  if (kRowBytes >= 16 && p.R > 0) {
    const CUtensorMapDataType dt = sizeof(OutT) == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                   : sizeof(OutT) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                       : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
    if (!make_map(&tout, dt, static_cast<int>(sizeof(OutT)), p.out, p.R, KS, KS,
                  CU_TENSOR_MAP_SWIZZLE_NONE)) {
      set_err("cuTensorMapEncodeTiled (row-segment output) failed%s%lld", "", 0);
      return TC_CUDA_ERROR;
    }
  }
  const uint32_t smem =
      rs_off_misc(p.nchunk, rs_n(KS), kRowBytes >= 16 ? kRowBytes : 0) + sizeof(RsMisc) + 1024;
  kern<<<static_cast<unsigned>(grid), kThreads, smem, st>>>(tin, tout, p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_err("kernel launch failed: %s%lld", cudaGetErrorString(e), 0);
    return TC_CUDA_ERROR;
  }
  ++g_launches;
  return TC_OK;
}

template <typename OutT>
static int launch_rowseg(const RsParams& p, void* ws, cudaStream_t st) {
  switch (p.k) {
    case 1: return launch_rowseg_k<OutT, 1>(p, ws, st);
    case 2: return launch_rowseg_k<OutT, 2>(p, ws, st);
    case 4: return launch_rowseg_k<OutT, 4>(p, ws, st);
    case 8: return launch_rowseg_k<OutT, 8>(p, ws, st);
    case 16: return launch_rowseg_k<OutT, 16>(p, ws, st);
    case 32: return launch_rowseg_k<OutT, 32>(p, ws, st);
  }
  set_err("no row-segment kernel for %s%lld segments per row", "", p.k);
  return TC_BAD_CONFIG;
}

template <typename OutT>
static int launch_rowseg_scan(const RssParams& p0, void* ws, cudaStream_t st) {
  auto kern = rowseg_scan_kernel<OutT>;
  constexpr uint32_t smem = rss_smem<OutT>();
  static_assert(smem <= 232448, "shared memory budget");
  int dev = 0;
  cudaGetDevice(&dev);
  static std::atomic<uint64_t> attr_done{0};
  const uint64_t dev_bit = 1ull << (dev & 63);
  if (!(attr_done.load() & dev_bit)) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
        cudaSuccess) {
      set_err("cudaFuncSetAttribute failed: %s%lld", cudaGetErrorString(cudaGetLastError()), 0);
      return TC_CUDA_ERROR;
    }
    attr_done.fetch_or(dev_bit);
  }
  const DevInfo di = dev_info(dev);
  if (!di.ok || di.major < 10) {
    set_err("no sm_100 device (compute capability major %s%lld)", "", di.major);
    return TC_NO_DEVICE;
  }
  RssParams p = p0;
  long long grid = di.sms;
  if (grid > p.nblk) grid = p.nblk;
  if (grid < 1) grid = 1;
  CUtensorMap tin, tout;
  const char* wsb = reinterpret_cast<const char*>(ws);
  const bool fp16 = sizeof(OutT) == 2;
  bool ok;
  if (p.R > 0) {
    ok = make_map(&tin, p.in_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                  2, p.x, p.R, kRow, p.L, CU_TENSOR_MAP_SWIZZLE_128B, rs_l2(true, p.s, p.nchunk).promo) &&
         (fp16 ? make_map(&tout, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, p.out, p.R, kRow, p.L)
               : make_map(&tout, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, p.out, p.R, 32, p.L));
  } else {
    ok = make_map(&tin, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, wsb + kWsZeroRow, 1, kRow) &&
         make_map(&tout, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, wsb + kWsDummyOut, 1, kRow);
  }
  if (!ok) {
    set_err("cuTensorMapEncodeTiled (row-segment scan) failed%s%lld", "", 0);
    return TC_CUDA_ERROR;
  }
  kern<<<static_cast<unsigned>(grid), kThreads, smem, st>>>(tin, tout, p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_err("kernel launch failed: %s%lld", cudaGetErrorString(e), 0);
    return TC_CUDA_ERROR;
  }
  ++g_launches;
  return TC_OK;
}


template <typename OutT>
static int launch_irreg2(const Params& p0, cudaStream_t st) {
  auto kern = irreg_reduce_kernel<OutT>;
  int dev = 0;
  cudaGetDevice(&dev);
  static std::atomic<uint64_t> attr_done{0};
  const uint64_t dev_bit = 1ull << (dev & 63);
  if (!(attr_done.load() & dev_bit)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kIrSmem) !=
        cudaSuccess) {
      set_err("cudaFuncSetAttribute failed: %s%lld", cudaGetErrorString(cudaGetLastError()), 0);
      return TC_CUDA_ERROR;
    }
    attr_done.fetch_or(dev_bit);
  }
  const DevInfo di = dev_info(dev);
  if (!di.ok || di.major < 10) {
    set_err("no sm_100 device (compute capability major %s%lld)", "", di.major);
    return TC_NO_DEVICE;
  }
  Params p = p0;
  char* wsb = reinterpret_cast<char*>(p.hdr);
  p.tk0 = reinterpret_cast<long long*>(wsb + kWsLookback);
  p.trec = wsb + kWsLookback + irreg_k0_bytes(p.n);
  long long grid = di.sms;  // one CTA per SM: kIrNG epilogue groups each
  if (grid > p.num_tiles) grid = p.num_tiles;
  if (grid > kMaxCtas) grid = kMaxCtas;
  if (grid < 1) grid = 1;
  CUtensorMap tin;
  const void* in_base = p.rows_full > 0 ? static_cast<const void*>(p.x)
                                        : static_cast<const void*>(wsb + kWsZeroRow);
  if (!make_map(&tin, p.in_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                2, in_base, p.rows_full > 0 ? p.rows_full : 1, kRow)) {
    set_err("cuTensorMapEncodeTiled (input) failed%s%lld", "", 0);
    return TC_CUDA_ERROR;
  }
  const long long nk = p.nseg + 1;
  irreg_k0_kernel<<<static_cast<unsigned>((nk + 255) / 256), 256, 0, st>>>(p.offs, p.nseg,
                                                                          p.num_tiles, p.tk0);
  kern<<<static_cast<unsigned>(grid), kIrThreads, kIrSmem, st>>>(tin, p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_err("kernel launch failed: %s%lld", cudaGetErrorString(e), 0);
    return TC_CUDA_ERROR;
  }
  g_launches += 2;
  return TC_OK;
}

static bool rowseg_enabled() {
  const char* e = getenv("TC_ROWSEG");  // tuning / A-B switch
  return !(e && e[0] == '0');
}

using LaunchFn = int (*)(const Params&, int, cudaStream_t);

template <int OP, int MODE, typename OutT>
static LaunchFn pick_gr(int gr) {
  switch (gr) {
    case 1: return &launch<OP, 1, MODE, OutT>;
    case 2: return &launch<OP, 2, MODE, OutT>;
    case 4: return &launch<OP, 4, MODE, OutT>;
    case 8: return &launch<OP, 8, MODE, OutT>;
    case 16: return &launch<OP, 16, MODE, OutT>;
    case 32: return &launch<OP, 32, MODE, OutT>;
    case 64: return &launch<OP, 64, MODE, OutT>;
  }
  return nullptr;
}

template <int OP, typename OutT>
static LaunchFn pick(int gr, int mode) {
  switch (mode) {
    case MODE_LOCAL: return pick_gr<OP, MODE_LOCAL, OutT>(gr);
    case MODE_ROWS: return gr == 1 ? &launch<OP, 1, MODE_ROWS, OutT> : nullptr;
    case MODE_TILES: return gr == 1 ? &launch<OP, 1, MODE_TILES, OutT> : nullptr;
    case MODE_GENERAL: return pick_gr<OP, MODE_GENERAL, OutT>(gr);
    case MODE_CHUNK:
      if constexpr (OP == OP_SCAN) return pick_gr<OP, MODE_CHUNK, OutT>(gr);
      return nullptr;
    case MODE_IRREG: return gr == 1 ? &launch<OP, 1, MODE_IRREG, OutT> : nullptr;
    case MODE_SPLIT:
      return gr == 8 ? &launch<OP, 8, MODE_SPLIT, OutT> : nullptr;
    case MODE_SPLITM:
      if constexpr (OP == OP_SCAN) return gr == 8 ? &launch<OP, 8, MODE_SPLITM, OutT> : nullptr;
      return nullptr;
    case MODE_GSCR:
      if constexpr (OP == OP_REDUCE) {
        switch (gr) {
          case 8: return &launch<OP, 8, MODE_GSCR, OutT>;
          case 16: return &launch<OP, 16, MODE_GSCR, OutT>;
          case 32: return &launch<OP, 32, MODE_GSCR, OutT>;
          case 64: return &launch<OP, 64, MODE_GSCR, OutT>;
        }
      }
      return nullptr;
  }
  return nullptr;
}

static int common_checks(const void* x, long long n, long long seg, const void* out, int out_dtype,
                         bool scan, void* ws, size_t ws_bytes, int op) {
  if (n < 1 || n >= (1LL << 37)) {
    set_err("input length %s%lld outside [1, 2^37)", "", n);
    return TC_BAD_LENGTH;
  }
  if (seg < 1) {
    set_err("segment size must be positive, got %s%lld", "", seg);
    return TC_BAD_LENGTH;
  }
  if (!x || !out || !ws) {
    set_err("null pointer argument%s%lld", "", 0);
    return TC_BAD_CONFIG;
  }
  if (out_dtype != TC_F16 && out_dtype != TC_F32 && !(out_dtype == TC_F64 && !scan)) {
    set_err("unsupported output dtype %s%lld", "", out_dtype);
    return TC_BAD_CONFIG;
  }
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(out) & 15) ||
      (reinterpret_cast<uintptr_t>(ws) & 255)) {
    set_err("x/out must be 16-byte aligned and ws 256-byte aligned%s%lld", "", 0);
    return TC_BAD_ALIGNMENT;
  }
  if (ws_bytes < ws_need(op, n, seg)) {
    set_err("workspace too small: need %s%lld bytes", "", (long long)ws_need(op, n, seg));
    return TC_WORKSPACE_TOO_SMALL;
  }
  return TC_OK;
}

// Segment geometry -> granules, carry mode and per-mode constants.
static bool split_enabled() {
  const char* e = getenv("TC_SPLIT");  // tuning / A-B switch
  return !(e && e[0] == '0');
}
constexpr long long kSplitReduceMin = kTileElems + kTileElems / 2;  // SPLIT reduce from here on
static bool split_reduce_enabled() {
  const char* e = getenv("TC_SPLIT_REDUCE");  // A/B switch: 0 = GENERAL (one-element granules) instead
  return !(e && e[0] == '0');
}
static bool split_reduce_forced() {
  const char* e = getenv("TC_SPLIT_REDUCE");  // probe switch: 2 = SPLIT for every s > 64
  return e && e[0] == '2';
}
static bool splitm_enabled() {
  const char* e = getenv("TC_SPLITM");  // tuning / A-B switch
  return !(e && e[0] == '0');
}
// MODE_SPLITM only where it measured faster (B200, 2^30, % of copy): fp32
// output, odd s in [11, 64) (s = 17 / 33 / 63: 79 / 80 / 93 % vs GENERAL
// 75 %); fp16 output keeps ROWSEG (SPLITM 44-52 %), gcd 2 / 4 keep GENERAL
// (87 % vs 76-80 %)
static bool splitm_wins(long long s, int out_esize) {
  const char* e = getenv("TC_SPLITM");
  if (e && e[0] == '2') return s >= kSplitMMin && s < kRow && gcd_ll(s, 64) <= 4;  // probe: always
  return splitm_enabled() && out_esize == 4 && (s & 1) && s >= 11 && s < kRow;
}
// largest segment whose range-entry carry a bounded scan recomputes (above:
// CHUNK).  GR = 1 keeps 2^18 (its CHUNK kernel streams at copy speed); the
// multi-granule CHUNK epilogue is slow, so those scans re-read up to 2^21.
static long long prepass_max(int gr) {
  if (const char* e = getenv("TC_PREPASS_MAX")) return atoll(e);  // tuning / A-B switch
  return gr == 1 ? kScanPrepassMax : (1LL << 21);
}

static Params make_params(const void* x, long long n, long long seg, void* out, void* ws, int op,
                          bool has_carry, int* gr_out, int* mode_out, bool allow_split = false,
                          int out_esize = 2) {
  if (seg > n) seg = n;  // one segment spanning everything: same result, smaller m
  Params p{};
  const long long g = gcd_ll(seg, kRow);
  int gr = static_cast<int>(kRow / g);
  p.x = reinterpret_cast<const __half*>(x);
  p.out = out;
  p.n = n;
  p.seg = seg;
  p.m = seg / g;
  p.rows_full = n / kRow;
  p.num_tiles = (n + kTileElems - 1) / kTileElems;
  p.qlast = (n - 1) / g;
  p.nseg = (n + seg - 1) / seg;
  const long long step = static_cast<long long>(kTileRows) * gr;
  p.step_div = step / p.m;
  p.step_mod = step % p.m;
  const bool scan_carry = (op == TC_OP_SCAN && has_carry);
  int mode;
  const bool pow2m = (p.m & (p.m - 1)) == 0;
  if (p.m == 1 && !scan_carry) {
    mode = MODE_LOCAL;
  } else if (gr == 1 && pow2m && p.m <= kTileRows && !scan_carry) {
    mode = MODE_ROWS;
    int l = 0;
    while ((1LL << l) < p.m) ++l;
    p.log2m = l;
  } else if (gr == 1 && p.m % kTileRows == 0 && !scan_carry) {
    mode = MODE_TILES;
    p.ktiles = p.m / kTileRows;
  } else {
    mode = MODE_GENERAL;
  }
  if (op == TC_OP_SCAN && mode == MODE_GENERAL && allow_split && !scan_carry && g <= 4 &&
      seg >= kSplitMMin && seg <= prepass_max(gr) && split_enabled() &&
      (seg >= kRow || splitm_wins(seg, out_esize))) {
    // few factors of two: granules of 8, each granule a segment start
    // splits recomputed from its raw elements (one start per row: MODE_SPLIT;
    // several: MODE_SPLITM)
    mode = seg >= kRow ? MODE_SPLIT : MODE_SPLITM;
    gr = 8;
    p.m = seg;  // element granularity for the start bookkeeping
    p.step_div = kTileElems / seg;
    p.step_mod = kTileElems % seg;
  }
  if (op == TC_OP_REDUCE && mode == MODE_GENERAL && g <= 4 && seg > kRow &&
      (seg >= kSplitReduceMin || split_reduce_forced()) && split_enabled() &&
      split_reduce_enabled()) {
    // the same for reduces: granules of 8, at most one end per row, the
    // granule it splits re-summed from its raw elements.  Measured on B200
    // (2^30 fp16, % of copy, SPLIT vs GENERAL with one-element granules):
    // s = 127 77 / 82, 4097 78 / 81, 8193 79 / 82, 12289 93 / 83,
    // 32769 101 / 84, 100001 93 / 85 -- with one or more ends per tile the
    // split rows' extra pass holds the tile's pair-scan barrier
    mode = MODE_SPLIT;
    gr = 8;
    p.m = seg;
    p.step_div = kTileElems / seg;
    p.step_mod = kTileElems % seg;
  }
  if (op == TC_OP_SCAN && (mode == MODE_TILES || mode == MODE_GENERAL) &&
      (seg > prepass_max(gr) || scan_carry))
    mode = MODE_CHUNK;
  *gr_out = gr;
  *mode_out = mode;
  char* w = reinterpret_cast<char*>(ws);
  p.hdr = reinterpret_cast<WsHeader*>(w);
  p.entries = reinterpret_cast<Entry*>(w + kWsEntries);
  const size_t slots = static_cast<size_t>(chunk_slots(n));
  size_t off = kWsLookback;
  p.u_word = reinterpret_cast<uint64_t*>(w + off);
  p.ck = 1;
  // GENERAL reduce with many segment ends per row (2m < GR; m is odd, so
  // GR >= 8): its own mode, the walk's end values staged in SMEM and the
  // interior segments stored coalesced (the other GENERAL kernels keep their
  // deeper rings and no staging buffer)
  if (op == TC_OP_REDUCE && mode == MODE_GENERAL && 2 * p.m < gr) mode = MODE_GSCR;
  *mode_out = mode;
  p.need_fixup = (op == TC_OP_REDUCE &&
                  (mode == MODE_TILES || mode == MODE_GENERAL || mode == MODE_GSCR ||
                   mode == MODE_SPLIT) &&
                  (kTileElems % seg != 0))
                     ? 1
                     : 0;
  return p;
}

}  // namespace tc

// =====================================================================
// C ABI
// =====================================================================
using namespace tc;

extern "C" {

size_t tc_workspace_bytes(int op, int64_t n, int64_t seg) {
  if (n < 1) n = 1;
  return ws_need(op, n, seg);
}

int tc_seg_reduce_ex(const void* x, int in_dtype, int64_t n, int64_t seg, void* out, int out_dtype,
                     void* ws, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  int rc = common_checks(x, n, seg, out, out_dtype, false, ws, ws_bytes, TC_OP_REDUCE);
  if (rc) return rc;
  if (in_dtype != TC_F16 && in_dtype != TC_BF16) {
    set_err("unsupported input dtype %s%lld", "", in_dtype);
    return TC_BAD_CONFIG;
  }
  const int out_es = out_dtype == TC_F16 ? 2 : out_dtype == TC_F32 ? 4 : 8;
  if (const int k = rowseg_enabled() ? rowseg_k(seg, n, out_es) : 0) {
    // whole segments per TMA row (MODE_ROWSEG): no carries at all
    RsParams rp{};
    rp.x = reinterpret_cast<const __half*>(x);
    rp.in_bf16 = (in_dtype == TC_BF16) ? 1 : 0;
    rp.out = out;
    rp.n = n;
    rp.s = seg;
    rp.k = k;
    rp.L = static_cast<long long>(k) * seg;
    rp.R = n / rp.L;
    rp.nblk = (rp.R + kTileRows - 1) / kTileRows;
    rp.nchunk = static_cast<int>((rp.L + kRow - 1) / kRow);
    rp.evict_normal = rs_l2(false, seg, rp.nchunk, out_es).evict_normal;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    return out_dtype == TC_F16   ? launch_rowseg<__half>(rp, ws, st)
           : out_dtype == TC_F32 ? launch_rowseg<float>(rp, ws, st)
                                 : launch_rowseg<double>(rp, ws, st);
  }
  int gr = 0, mode = 0;
  Params p = make_params(x, n, seg, out, ws, TC_OP_REDUCE, false, &gr, &mode);
  p.in_bf16 = (in_dtype == TC_BF16) ? 1 : 0;
  LaunchFn fn = nullptr;
  int es = 2;
  if (out_dtype == TC_F16) {
    fn = pick<OP_REDUCE, __half>(gr, mode);
    es = 2;
  } else if (out_dtype == TC_F32) {
    fn = pick<OP_REDUCE, float>(gr, mode);
    es = 4;
  } else {
    fn = pick<OP_REDUCE, double>(gr, mode);
    es = 8;
  }
  if (!fn) {
    set_err("no kernel for granules-per-row %s%lld", "", gr);
    return TC_BAD_CONFIG;
  }
  return fn(p, es, reinterpret_cast<cudaStream_t>(stream));
}

int tc_seg_reduce(const void* x, int64_t n, int64_t seg, void* out, int out_dtype, void* ws,
                  size_t ws_bytes, void* stream) {
  return tc_seg_reduce_ex(x, TC_F16, n, seg, out, out_dtype, ws, ws_bytes, stream);
}

int tc_full_reduce(const void* x, int64_t n, void* out, int out_dtype, void* ws, size_t ws_bytes,
                   void* stream) {
  return tc_seg_reduce(x, n, n < 1 ? 1 : n, out, out_dtype, ws, ws_bytes, stream);
}

int tc_seg_scan_ex(const void* x, int in_dtype, int64_t n, int64_t seg, void* out, int out_dtype,
                   int exclusive, const double* carry_in, double* total_out, void* ws,
                   size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  int rc = common_checks(x, n, seg, out, out_dtype, true, ws, ws_bytes, TC_OP_SCAN);
  if (rc) return rc;
  if (in_dtype != TC_F16 && in_dtype != TC_BF16) {
    set_err("unsupported input dtype %s%lld", "", in_dtype);
    return TC_BAD_CONFIG;
  }
  if (carry_in == nullptr && total_out == nullptr) {
    if (const int k = rowseg_enabled() ? rowseg_scan_k(seg, n, out_dtype == TC_F16 ? 2 : 4) : 0) {
      // whole segments per TMA row (MODE_ROWSEG): no carries between rows
      RssParams rp{};
      rp.x = reinterpret_cast<const __half*>(x);
      rp.in_bf16 = (in_dtype == TC_BF16) ? 1 : 0;
      rp.out = out;
      rp.n = n;
      rp.s = seg;
      rp.L = static_cast<long long>(k) * seg;
      rp.R = n / rp.L;
      rp.nblk = (rp.R + kTileRows - 1) / kTileRows;
      rp.nchunk = static_cast<int>((rp.L + kRow - 1) / kRow);
      rp.exclusive = exclusive ? 1 : 0;
      rp.evict_normal = rs_l2(true, seg, rp.nchunk).evict_normal;
      cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
      return out_dtype == TC_F16 ? launch_rowseg_scan<__half>(rp, ws, st)
                                 : launch_rowseg_scan<float>(rp, ws, st);
    }
  }
  int gr = 0, mode = 0;
  Params p = make_params(x, n, seg, out, ws, TC_OP_SCAN, carry_in != nullptr, &gr, &mode,
                         carry_in == nullptr && total_out == nullptr, out_dtype == TC_F16 ? 2 : 4);
  p.exclusive = exclusive ? 1 : 0;
  p.in_bf16 = (in_dtype == TC_BF16) ? 1 : 0;
  p.carry_in = carry_in;
  p.total_out = total_out;
  LaunchFn fn =
      (out_dtype == TC_F16) ? pick<OP_SCAN, __half>(gr, mode) : pick<OP_SCAN, float>(gr, mode);
  if (!fn) {
    set_err("no kernel for granules-per-row %s%lld", "", gr);
    return TC_BAD_CONFIG;
  }
  return fn(p, out_dtype == TC_F16 ? 2 : 4, reinterpret_cast<cudaStream_t>(stream));
}

int tc_seg_scan(const void* x, int64_t n, int64_t seg, void* out, int out_dtype, int exclusive,
                const double* carry_in, double* total_out, void* ws, size_t ws_bytes,
                void* stream) {
  return tc_seg_scan_ex(x, TC_F16, n, seg, out, out_dtype, exclusive, carry_in, total_out, ws,
                        ws_bytes, stream);
}

int tc_full_scan(const void* x, int64_t n, void* out, int out_dtype, int exclusive,
                 const double* carry_in, double* total_out, void* ws, size_t ws_bytes,
                 void* stream) {
  return tc_seg_scan(x, n, n < 1 ? 1 : n, out, out_dtype, exclusive, carry_in, total_out, ws,
                     ws_bytes, stream);
}

// Irregular (CSR-offset) segments: validation shared by reduce and scan.
static int irreg_checks(const void* x, int in_dtype, int64_t n, const int64_t* offsets,
                        int64_t nseg, const void* out, int out_dtype, bool scan, void* ws,
                        size_t ws_bytes) {
  g_err[0] = 0;
  int rc = common_checks(x, n, 1, out, out_dtype, scan, ws, ws_bytes,
                         scan ? TC_OP_SCAN : TC_OP_REDUCE);
  if (rc) return rc;
  if (in_dtype != TC_F16 && in_dtype != TC_BF16) {
    set_err("unsupported input dtype %s%lld", "", in_dtype);
    return TC_BAD_CONFIG;
  }
  if (nseg < 1 || nseg > n + (1LL << 31)) {
    set_err("segment count %s%lld outside [1, n + 2^31]", "", nseg);
    return TC_BAD_LENGTH;
  }
  if (!offsets || (reinterpret_cast<uintptr_t>(offsets) & 7)) {
    set_err("offsets must be a non-null, 8-byte aligned device pointer%s%lld", "", 0);
    return TC_BAD_ALIGNMENT;
  }
  return TC_OK;
}

static Params irreg_params(const void* x, int in_dtype, int64_t n, const int64_t* offsets,
                           int64_t nseg, void* out, void* ws, int op) {
  int gr = 0, mode = 0;
  Params p = make_params(x, n, n, out, ws, op, false, &gr, &mode);
  p.in_bf16 = (in_dtype == TC_BF16) ? 1 : 0;
  p.offs = reinterpret_cast<const long long*>(offsets);
  p.nseg = nseg;
  p.need_fixup = (op == TC_OP_REDUCE) ? 1 : 0;
  return p;
}

int tc_irreg_reduce(const void* x, int in_dtype, int64_t n, const int64_t* offsets, int64_t nseg,
                    void* out, int out_dtype, void* ws, size_t ws_bytes, void* stream) {
  int rc = irreg_checks(x, in_dtype, n, offsets, nseg, out, out_dtype, false, ws, ws_bytes);
  if (rc) return rc;
  Params p = irreg_params(x, in_dtype, n, offsets, nseg, out, ws, TC_OP_REDUCE);
  const char* v1 = getenv("TC_IRREG_V1");  // A/B switch: the single-group MODE_IRREG kernel
  if (!(v1 && v1[0] == '1')) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    return out_dtype == TC_F16   ? launch_irreg2<__half>(p, st)
           : out_dtype == TC_F32 ? launch_irreg2<float>(p, st)
                                 : launch_irreg2<double>(p, st);
  }
  LaunchFn fn = (out_dtype == TC_F16)   ? pick<OP_REDUCE, __half>(1, MODE_IRREG)
                : (out_dtype == TC_F32) ? pick<OP_REDUCE, float>(1, MODE_IRREG)
                                        : pick<OP_REDUCE, double>(1, MODE_IRREG);
  const int es = (out_dtype == TC_F16) ? 2 : (out_dtype == TC_F32) ? 4 : 8;
  return fn(p, es, reinterpret_cast<cudaStream_t>(stream));
}

int tc_irreg_scan(const void* x, int in_dtype, int64_t n, const int64_t* offsets, int64_t nseg,
                  void* out, int out_dtype, int exclusive, void* ws, size_t ws_bytes,
                  void* stream) {
  int rc = irreg_checks(x, in_dtype, n, offsets, nseg, out, out_dtype, true, ws, ws_bytes);
  if (rc) return rc;
  Params p = irreg_params(x, in_dtype, n, offsets, nseg, out, ws, TC_OP_SCAN);
  p.exclusive = exclusive ? 1 : 0;
  LaunchFn fn = (out_dtype == TC_F16) ? pick<OP_SCAN, __half>(1, MODE_IRREG)
                                      : pick<OP_SCAN, float>(1, MODE_IRREG);
  return fn(p, out_dtype == TC_F16 ? 2 : 4, reinterpret_cast<cudaStream_t>(stream));
}

int tc_bn_stats(const void* x, int in_dtype, int64_t N, int64_t C, int64_t HW, void* mean,
                void* var, int out_dtype, void* ws, size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  if (N < 1 || C < 1 || HW < 1 || N > (1LL << 37) / C / HW) {
    set_err("batch-norm shape outside 1 <= N*C*HW < 2^37 (N*C = %s%lld)", "", N * C);
    return TC_BAD_LENGTH;
  }
  if (!mean || !var) {
    set_err("null pointer argument%s%lld", "", 0);
    return TC_BAD_CONFIG;
  }
  if (out_dtype != TC_F32 && out_dtype != TC_F64) {
    set_err("batch-norm statistics are F32 or F64, got %s%lld", "", out_dtype);
    return TC_BAD_CONFIG;
  }
  const long long n = N * C * HW;
  if (ws_bytes < ws_need(TC_OP_BN_STATS, n, HW)) {
    set_err("workspace too small: need %s%lld bytes", "", (long long)ws_need(TC_OP_BN_STATS, n, HW));
    return TC_WORKSPACE_TOO_SMALL;
  }
  if (!x || (reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(ws) & 255)) {
    set_err("x must be non-null and 16-byte aligned, ws 256-byte aligned%s%lld", "", 0);
    return TC_BAD_ALIGNMENT;
  }
  if (in_dtype != TC_F16 && in_dtype != TC_BF16) {
    set_err("unsupported input dtype %s%lld", "", in_dtype);
    return TC_BAD_CONFIG;
  }
  // scratch: the per-(n, c) moments, at the start of the look-back region
  // (bn_finish_kernel clears every entry it read, so the region stays zero)
  double2* mom = reinterpret_cast<double2*>(reinterpret_cast<char*>(ws) + kWsLookback);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0;
  cudaGetDevice(&dev);
  const DevInfo di = dev_info(dev);
  if (!di.ok || di.major < 10) {
    set_err("no sm_100 device (compute capability major %s%lld)", "", di.major);
    return TC_NO_DEVICE;
  }
  const long long nsegs = N * C;
  const __half* xh = reinterpret_cast<const __half*>(x);
  const int bf = in_dtype == TC_BF16 ? 1 : 0;
  long long groups = N;
  const int V = (HW % 8 == 0) ? 8 : (HW % 4 == 0) ? 4 : (HW % 2 == 0) ? 2 : 1;
  long long chan_min = kBnChanMin;
  if (const char* e = getenv("TC_BN_CHAN_MIN")) chan_min = atoll(e);  // tuning / A-B switch
  if (HW >= chan_min && N * (HW / V) < (1LL << 31)) {
    // per-channel blocks over sample ranges, ~2 full waves of 8 blocks / SM
    // (a partial second wave cost ~10 % at C = 256; more, shorter blocks
    // lose to their start-up and combine)
    const long long wave = 8LL * di.sms;
    long long waves = 2;  // measured (256x256x56x56): 2 waves 84 %, 4 waves 79 %, 8 waves 68 %
    int bn_unroll = 4;
    if (const char* e = getenv("TC_BN_WAVES")) waves = atoll(e);  // tuning / A-B switches
    if (const char* e = getenv("TC_BN_UNROLL")) bn_unroll = atoi(e);
    long long splits = (waves * wave) / C;
    if (splits < 1) splits = 1;
    if (splits > N) splits = N;
    if (splits > 65535) splits = 65535;
    groups = splits;
    const FastDiv fd = make_fastdiv(static_cast<uint32_t>(HW / V));
    const dim3 grid(static_cast<unsigned>(C), static_cast<unsigned>(splits));
    // per-channel arrival tickets: the dedicated always-zero region for
    // C <= kBnMaxTicketC; otherwise after the moments, where other ops'
    // scratch (the CHUNK scan's epoch-tagged look-back words) may linger,
    // so they are zeroed first, stream-ordered
    unsigned* ticket = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(ws) + kWsBnTickets);
    if (C > kBnMaxTicketC) {
      ticket = reinterpret_cast<unsigned*>(mom + N * C);
      if (cudaMemsetAsync(ticket, 0, sizeof(unsigned) * static_cast<size_t>(C), st) != cudaSuccess) {
        set_err("cudaMemsetAsync failed: %s%lld", cudaGetErrorString(cudaGetLastError()), 0);
        return TC_CUDA_ERROR;
      }
    }
    auto go = [&](auto out_tag) {
      using OutT = decltype(out_tag);
      OutT* mo = reinterpret_cast<OutT*>(mean);
      OutT* vo = reinterpret_cast<OutT*>(var);
      auto launch_v = [&](auto u_tag) {
        constexpr int U = decltype(u_tag)::value;
        switch (V) {
          case 8: bn_chan_kernel<8, U, OutT><<<grid, kBnThreads, 0, st>>>(xh, bf, N, C, HW, fd, mom, ticket, mo, vo); break;
          case 4: bn_chan_kernel<4, U, OutT><<<grid, kBnThreads, 0, st>>>(xh, bf, N, C, HW, fd, mom, ticket, mo, vo); break;
          case 2: bn_chan_kernel<2, U, OutT><<<grid, kBnThreads, 0, st>>>(xh, bf, N, C, HW, fd, mom, ticket, mo, vo); break;
          default: bn_chan_kernel<1, U, OutT><<<grid, kBnThreads, 0, st>>>(xh, bf, N, C, HW, fd, mom, ticket, mo, vo); break;
        }
      };
      if (bn_unroll == 8)
        launch_v(std::integral_constant<int, 8>{});
      else
        launch_v(std::integral_constant<int, 4>{});
    };
    if (out_dtype == TC_F32)
      go(0.f);
    else
      go(0.0);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      set_err("kernel launch failed: %s%lld", cudaGetErrorString(e), 0);
      return TC_CUDA_ERROR;
    }
    g_launches += 1;
    return TC_OK;
  } else {
    const long long per_block = HW < kBnWarpMin ? kBnThreads : kBnThreads / 32;  // segments
    long long blocks = (nsegs + per_block - 1) / per_block;
    const long long cap = static_cast<long long>(di.sms) * (2048 / kBnThreads);  // one wave
    if (blocks > cap) blocks = cap;
    bn_moments_kernel<<<static_cast<unsigned>(blocks), kBnThreads, 0, st>>>(xh, bf, N, C, HW, mom);
  }
  if (out_dtype == TC_F32)
    bn_finish_kernel<float><<<static_cast<unsigned>(C), kBnThreads, 0, st>>>(
        xh, bf, N, C, HW, mom, groups, reinterpret_cast<float*>(mean), reinterpret_cast<float*>(var));
  else
    bn_finish_kernel<double><<<static_cast<unsigned>(C), kBnThreads, 0, st>>>(
        xh, bf, N, C, HW, mom, groups, reinterpret_cast<double*>(mean),
        reinterpret_cast<double*>(var));
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_err("kernel launch failed: %s%lld", cudaGetErrorString(e), 0);
    return TC_CUDA_ERROR;
  }
  g_launches += 2;
  return TC_OK;
}

int tc_plan_info(int op, int64_t n, int64_t seg, int out_dtype, int has_carry, int has_total,
                 int* mode, int64_t* row_len) {
  if (n < 1 || seg < 1 || (op != TC_OP_REDUCE && op != TC_OP_SCAN) || !mode || !row_len)
    return TC_BAD_CONFIG;
  const int es = out_dtype == TC_F16 ? 2 : out_dtype == TC_F32 ? 4 : 8;
  int k = 0;
  if (rowseg_enabled()) {
    if (op == TC_OP_REDUCE)
      k = rowseg_k(seg, n, es);
    else if (!has_carry && !has_total)
      k = rowseg_scan_k(seg, n, es);
  }
  if (k) {
    *mode = MODE_ROWSEG;
    *row_len = static_cast<int64_t>(k) * seg;
    return TC_OK;
  }
  static char dummy[1024];
  int gr = 0, md = 0;
  make_params(dummy, n, seg, dummy, dummy, op, op == TC_OP_SCAN && has_carry, &gr, &md,
              !has_carry && !has_total, es);
  *mode = md;
  *row_len = kRow;
  return TC_OK;
}

const char* tc_status_string(int s) {
  switch (s) {
    case TC_OK: return "ok";
    case TC_BAD_LENGTH: return "bad length";
    case TC_BAD_CONFIG: return "bad config";
    case TC_BAD_ALIGNMENT: return "bad alignment";
    case TC_WORKSPACE_TOO_SMALL: return "workspace too small";
    case TC_CUDA_ERROR: return "cuda error";
    case TC_NO_DEVICE: return "no sm_100 device";
  }
  return "unknown status";
}

const char* tc_last_error(void) { return g_err; }

uint64_t tc_launch_count(void) { return g_launches; }
void tc_reset_launch_count(void) { g_launches = 0; }

#ifdef TC_IRREG_TRACE
int tc_debug_irreg_trace(void* host_out) {
  return cudaMemcpyFromSymbol(host_out, g_irtrace, sizeof(g_irtrace)) == cudaSuccess ? 0 : -1;
}
#endif

int tc_abi_version(void) { return (1 << 16) | 5; }

}  // extern "C"
