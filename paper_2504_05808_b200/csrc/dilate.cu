#include <cstdio>
#include <cstdlib>
// K5 (default path): exact ball dilation LT^2(p) = max{ D(q) : |p-q|^2 < D(q) }
// by "exact-order cover", fused with the shell test and the per-label reductions.
//
// Work organisation.  A CTA of 4 warps owns a group of 4 output tiles (3D: 1x2x2 tiles of
// 32x8x8, 2D: 2x2 tiles of 32x64; a tile = 64 rows of 32 elements); each warp owns one tile
// (values, coverage masks), while the candidate gather and sort are shared by the 4 tiles.
//   1. gather : the CTA collects every kept maximal ball (K4 output) whose ball reaches the
//               group's box into a shared list (packed centre + D) and a histogram of a
//               monotone bucket of D.  K4's lists are sorted by bucket, so a home tile is
//               abandoned as soon as its remaining balls are too small to reach the group.
//   2. sort   : an exact counting sort of the list by D, descending (a round covers at most
//               kCap candidates and a D range of at most kHist values; larger gathers run in
//               several D-descending rounds).
//   3. cover  : each warp walks the sorted list: lanes screen 32 balls at a time (the ball
//               reaches the tile, and its bounding rows hold still-uncovered foreground within
//               its x-extent, tracked as four 64-bit row masks, one per 8-column chunk); each
//               surviving ball is painted with the lanes over the tile's rows: per row the
//               interval |x-qx| <= isqrt(D-1-dy^2-dz^2), restricted to uncovered foreground.
//               Exactness: balls arrive in exactly descending D, so the first ball covering a
//               cell carries the max D over all kept balls containing it; each cell is written
//               once and marked covered at once.  A warp stops when nothing is left uncovered.
//   4. epilogue : LT^2 per element, shell (D == 1), per-label reductions (shared with the
//               fallback kernel in lt.cu).
// The pathological case (a single bucket exceeding the list or the sort range) hands the
// group to the atomic sparse-table kernel k_dilate_atomic (lt.cu), which also handles
// Dmax > 65535 (FASTRS_FORCE_FALLBACK sends every tile there: a GPU-internal cross-check).
#include "common.cuh"
#include "dilate_common.cuh"

namespace fastrs {
namespace {

constexpr int kWarps = 4;  // warps per CTA = tiles per group
constexpr int kCap = 1536;   // candidate list capacity per round (3D single pass: 2 * kCap compact entries)
constexpr int kIdx = 2048;   // sort indices (rounds path) / gather scratch (record prefix sums and z offsets)
constexpr int kBuckets = 128;
constexpr int kHist = 1536;  // exact-D counting-sort bins per round
#ifndef FASTRS_KPOINT
#define FASTRS_KPOINT 64
#endif
// uncovered cells at which a warp switches to point tests (a multiple of 32).  Round-2 sweep
// (C4, dot-product point tests, K5a + K5b, tools/sweep_define.sh): 32 -> 14.68 ms, 64 -> 14.51,
// 96 -> 14.99, 128 -> 16.71, 192 -> 20.22, 256 -> 23.10
constexpr int kPoint = FASTRS_KPOINT;
static_assert(kPoint % 32 == 0 && kPoint <= 1024, "point-mode list: whole warps of entries");
constexpr int kPointW = kPoint / 32;
// gcount[group]: (wave << 29) | list length, or one of the two sentinels
constexpr uint32_t kGroupFallback = 0xFFFFFFFFu;  // left to the atomic fallback (k_dilate_atomic)
constexpr uint32_t kGroupDeferred = 0xFFFFFFFEu;  // the pool was full: the next wave gathers it
constexpr uint32_t kGroupCountMask = (1u << 29) - 1u;
constexpr int kOff = 16384;  // coordinate bias of packed candidates

constexpr int kStgChunks = 8;  // record chunks a group may stage list overflow for

struct Smem;
static_assert(3 * 512 <= 1536 && 2 * (512 + 8) + 512 <= 2048, "gather scratch fits S.hist / S.idx");

struct Smem {  // K5a (gather + sort)
  union {
    unsigned long long list[kCap];   // gathered candidates (centre relative to the group), gather order
    uint32_t list32[2 * kCap];       // the same, compact (3D single-pass path, see pack32)
  };
  uint32_t hist[kHist];              // exact-D counting sort: bin Dhi - D (rounds path; gather scratch)
  uint16_t idx[kIdx];                // indices into list, sorted by D (descending)
  uint32_t dh[kHist];                // exact-D histogram / cursors of the single-pass path
  uint32_t bhist[kBuckets];
  unsigned long long base;           // the group's offset in the global candidate pool
  uint32_t wsum[kWarps];
  uint32_t count, total, nrec;
  int round_lo, round_hi, round_top, next_hi, fallback, rounds, bigbucket;
  int bb[6];                         // bounding box of the group's foreground (group coordinates)
  // single-pass list overflow staged in the pool's top half, one block per record chunk:
  // list position pos >= stg_lo[k] of chunk k lives at stage[stg_off[k] + pos]
  unsigned long long stg_off[kStgChunks];
  uint32_t stg_lo[kStgChunks];
  int nstg, stg_fail;
  int defer;                         // the pool is full: defer the group to the next wave
  unsigned long long topkey;         // cover cut: (max D << 32) | home tile of the largest reaching ball
  int qstar[4];                      // its centre (group coordinates) and D
};

// K5b CTAs hold NW of a group's kWarps tiles (one warp each).  The warps share
// nothing, so one warp per CTA lets every tile retire on its own: no warp slot idles while a
// sibling tile of the same CTA is still painting.
// K5b launch shape: warps per CTA and resident CTAs per SM (sets the register cap: 64 here, 32
// resident warps; the fused reductions spill at 56).  C4 sweep (persistent, round 1, LT plane):
// (2,16) 10.63 ms, (2,18) 10.58, (2,20) 10.71, (2,24) 10.68, (1,32) 10.76, (4,10) 10.70; round 2
// (fused, K5a + K5b): (2,16) 16.40 ms, (2,14) 16.48, (2,12) 16.88, (2,10) 17.87; round 2b (straight-line
// per-ball rows, C4 K5a + K5b): (2,16) 11.80 ms, (2,14) 11.44, (2,12) 11.88.
#ifndef FASTRS_PAINT_MINB
#define FASTRS_PAINT_MINB 14
#endif
constexpr int kPaintNW = 2, kPaintMinB = FASTRS_PAINT_MINB;
// x chunks of the uncovered-row masks the K5b screen intersects with a ball's x-extent (4 chunks of
// 8 columns or 8 of 4)
#ifndef FASTRS_UC_CHUNKS
#define FASTRS_UC_CHUNKS 4
#endif
constexpr int kUcChunks = FASTRS_UC_CHUNKS, kUcW = 32 / kUcChunks;
constexpr uint32_t kUcBits = (1u << kUcW) - 1u;
template <int NW, bool FUSED>
struct PaintSmem {  // K5b (one tile per warp)
  uint16_t val[NW][FUSED ? 1 : kRows * 32];  // LT^2 per element of each warp's tile (D <= 65535 here)
  int4 sball[NW][32];             // survivors of a screened batch: centre (tile coords), D
  unsigned long long scand[NW][32];  // their candidate rows
  alignas(16) unsigned long long uc[NW][kUcChunks];  // rows with uncovered foreground per x chunk
  uint16_t ulist[NW][kPoint];     // point mode: the still-uncovered cells (row*32 + x)
  uint2 pcell[NW][kPoint];        // the same cells for the dot-product test: (2x, 2y, 2z) bytes, -|p|^2
  uint32_t qa[NW][32];            // fused: covering events, (cell offset | count << 16)
  uint32_t qb[NW][32];            //        and (D | shell count << 16)
};


struct GroupDivs {  // a flat group index -> (gx, gy, gz, item)
  FastDiv x, y, z;
};
__host__ inline GroupDivs group_divs(const Geom& g) {
  const int GX = g.ndim == 3 ? 1 : 2, GY = 2, GZ = g.ndim == 3 ? 2 : 1;
  GroupDivs d;
  d.x = FastDiv((uint32_t)((g.ntx + GX - 1) / GX));
  d.y = FastDiv((uint32_t)((g.nty + GY - 1) / GY));
  d.z = FastDiv((uint32_t)((g.tz_hi - g.tz_lo + GZ - 1) / GZ));
  return d;
}

template <bool IS3D>
struct Shape {
  static constexpr int TY = IS3D ? 8 : 64, TZ = IS3D ? 8 : 1;
  static constexpr int GX = IS3D ? 1 : 2, GY = 2, GZ = IS3D ? 2 : 1;  // tiles per group
};

__device__ __forceinline__ unsigned long long pack(int x, int y, int z, uint32_t D) {
  return (unsigned long long)D | ((unsigned long long)(uint16_t)(x + kOff) << 16) |
         ((unsigned long long)(uint16_t)(y + kOff) << 32) | ((unsigned long long)(uint16_t)(z + kOff) << 48);
}
// Compact 32-bit candidate of the 3D single-pass gather (Dmax <= kHist, so r <= 39): a centre
// that reaches the group lies within r of its 32x16x16 box, i.e. x in [-39, 70], y, z in
// [-39, 54]; biased by 40 they fit 7 bits each, D <= 1536 fits 11.  Twice the entries of the
// shared list in the same bytes, so fewer groups overflow into the regather.
constexpr int kB32 = 40;
__device__ __forceinline__ uint32_t pack32(int x, int y, int z, uint32_t D) {
  return (uint32_t)(x + kB32) | ((uint32_t)(y + kB32) << 7) | ((uint32_t)(z + kB32) << 14) | (D << 21);
}
__device__ __forceinline__ unsigned long long unpack32(uint32_t e) {
  return pack((int)(e & 127u) - kB32, (int)((e >> 7) & 127u) - kB32, (int)((e >> 14) & 127u) - kB32, e >> 21);
}

__device__ __forceinline__ int gap(int lo, int hi, int c) { return c < lo ? lo - c : (c > hi ? c - hi : 0); }

// floor(sqrt(h)) for 0 <= h < 2^16 via the hardware approximation (error << 1/512; integer
// inputs are never denormal, so the flush-to-zero form needs no input scaling)
__device__ __forceinline__ int isqrt16(int h) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"((float)h));
  return (int)(r + 1e-3f);
}

__device__ __forceinline__ uint32_t range_mask(int l, int r) {  // bits l..r (0 <= l <= r <= 31)
  uint32_t m;
  asm("bmsk.clamp.b32 %0, %1, %2;" : "=r"(m) : "r"(l), "r"(r - l + 1));  // r-l+1 bits from bit l
  return m;
}

// Gather the candidates reaching the group box with bucket in [blo, bhi] into S.list.
// HIST: also histogram them (the first pass of a round).  Flattened: the CTA first lists the
// home tiles whose balls can reach the group (records: neighbour index, first entry, count),
// reading per home tile only the prefix of its bucket-sorted list that can reach the group and
// lies in the bucket range (K4's octave counts), then every thread takes entries of any record
// (binary search over the record prefix sums), so all the entry loads are in flight at once.
// S.hist and S.idx serve as scratch (they are rebuilt by the sort afterwards).
constexpr int kRecCap = 512;  // records per chunk: 3 words each in S.hist, prefix sums in S.idx

// Exclusive prefix sum of a[0..n) (n <= kHist) in place by the whole CTA; returns the total.
// Ends with a barrier.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t* a, int n, uint32_t* wsum) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kPer = kHist / (kWarps * 32);
  const int base = tid * kPer;
  uint32_t loc[kPer], sum = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    loc[j] = base + j < n ? a[base + j] : 0u;
    sum += loc[j];
  }
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  uint32_t run = inc - sum, total = 0;
  for (int w = 0; w < kWarps; ++w) {
    if (w < warp) run += wsum[w];
    total += wsum[w];
  }
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    if (base + j < n) a[base + j] = run;
    run += loc[j];
  }
  __syncthreads();
  return total;
}

// gather modes: what happens to each candidate that reaches the group
enum { kListBucketHist = 0,  // append to S.list (up to kCap) and count its D bucket in S.bhist
       kListOnly = 1,        // append to S.list
       kListExactHist = 2,   // append to S.list and count its exact D in S.dh (bin dtop - D)
       kScatter = 3,         // store it at out[S.dh[dtop - D]++] (S.dh holds the sorted cursors)
       kExactCount = 4 };    // count its exact D in S.dh (bin dtop - D), no list

#ifdef FASTRS_GATHER_STATS
__device__ unsigned long long g_stats_ptr[3];  // examined, D-cut by the record's own gap, taken
#endif

template <bool IS3D, int MODE, bool COMPACT = false>
__device__ __forceinline__ void gather(Smem& S, const TileMeta* __restrict__ meta, const uint2* __restrict__ cent,
                                       const uint16_t* __restrict__ oct, const Geom& g, int64_t b, int64_t tx0,
                                       int64_t ty0, int64_t tz0, int nrx, int nry, int nrz, int blo, int bhi,
                                       uint32_t dtop = 0, unsigned long long* out = nullptr,
                                       unsigned long long* stage = nullptr, unsigned long long* stage_used = nullptr,
                                       unsigned long long stage_cap = 0, uint32_t dlo_f = 0u,
                                       uint32_t dhi_f = 0xFFFFFFFFu) {
  using P = Shape<IS3D>;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = P::GX + 2 * nrx, ny = P::GY + 2 * nry, nz = P::GZ + 2 * nrz;
  const int nneigh = nx * ny * nz;
  uint32_t* rec = S.hist;                                  // 3 words per record
  uint32_t* pre = reinterpret_cast<uint32_t*>(S.idx);      // kRecCap + 1 prefix sums
  int16_t* recz = reinterpret_cast<int16_t*>(S.idx) + 2 * (kRecCap + 8);  // home tile z offsets
  const int o_start = (bhi + 1 + 3) >> 2;                  // entries with bucket > bhi come first
  // n -> (ix, iy, iz) without integer divides: umulhi(n, floor((2^32-1)/d) + 1) = n / d
  // exactly whenever n * d < 2^32 (here n < 10^5, d < 100); d = 1 (the reciprocal would be
  // 2^32) is taken apart
  const uint32_t rx = 0xFFFFFFFFu / (uint32_t)nx + 1u, ry = 0xFFFFFFFFu / (uint32_t)ny + 1u;
  const int bb0 = S.bb[0], bb1 = S.bb[1], bb2 = S.bb[2], bb3 = S.bb[3], bb4 = S.bb[4], bb5 = S.bb[5];
  const bool full_range = blo <= 0 && bhi >= kBucketTop;
  for (int nb0 = 0; nb0 < nneigh; nb0 += kRecCap) {
    __syncthreads();
    if (tid == 0) S.nrec = 0;
    __syncthreads();
    const int nb1 = min(nneigh, nb0 + kRecCap);
    for (int n = nb0 + tid; n < nb1; n += kWarps * 32) {
      const int q1 = nx == 1 ? n : (int)__umulhi((uint32_t)n, rx);
      const int iz = ny == 1 ? q1 : (int)__umulhi((uint32_t)q1, ry);
      const int ix = n - q1 * nx, iy = q1 - iz * ny;
      const int64_t hx = tx0 + ix - nrx, hy = ty0 + iy - nry, hz = tz0 + iz - nrz;
      if (hx < 0 || hx >= g.ntx || hy < 0 || hy >= g.nty || hz < 0 || hz >= g.ntz) continue;
      const int64_t ht = ((b * g.ntz + hz) * g.nty + hy) * g.ntx + hx;
      const TileMeta hm = meta[ht];
      if (!hm.count) continue;
      const int hox = (ix - nrx) * kTX, hoy = (iy - nry) * P::TY, hoz = (iz - nrz) * P::TZ;
      // gap between the home tile box and the bounding box of the group's foreground
      const int gx = max(0, max(hox - bb1, bb0 - (hox + kTX - 1)));
      const int gy = max(0, max(hoy - bb3, bb2 - (hoy + P::TY - 1)));
      const int gz = max(0, max(hoz - bb5, bb4 - (hoz + P::TZ - 1)));
      const int g2 = gx * gx + gy * gy + gz * gz;
      if (g2 > (int)hm.maxD - 1 || dbucket(hm.maxD) < blo) continue;
      // lowest bucket whose largest D can still reach the gap: D - 1 >= g2 <=> D >= g2 + 1
      const int bmin = max(dbucket((uint32_t)g2 + 1u), blo);
      const uint16_t* oc = oct + ht * kOctPerTile;
      const uint32_t end = oc[bmin >> 2];
      const uint32_t start = o_start >= kOctPerTile ? 0u : oc[o_start];
      if (end <= start) continue;
      const uint32_t slot = atomicAdd(&S.nrec, 1u);
      rec[3 * slot] = (uint32_t)ht;  // tile index (< 2^32, checked in make_geom)
      rec[3 * slot + 1] = start | ((end - start) << 16);
      // home tile origin relative to the group, biased to stay non-negative (|offset| < 2^15)
      rec[3 * slot + 2] = (uint32_t)(hox + kOff) | ((uint32_t)(hoy + kOff) << 16);
      recz[slot] = (int16_t)hoz;
    }
    __syncthreads();
    const int nrec = (int)S.nrec;
    {  // exclusive prefix of the record counts (kRecCap / 128 = 5 records per thread)
      constexpr int kPer = (kRecCap + kWarps * 32 - 1) / (kWarps * 32);
      uint32_t loc[kPer], sum = 0;
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int r = tid * kPer + j;
        loc[j] = r < nrec ? rec[3 * r + 1] >> 16 : 0u;
        sum += loc[j];
      }
      uint32_t inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += v;
      }
      if (lane == 31) S.wsum[warp] = inc;
      __syncthreads();
      uint32_t run = inc - sum;
      for (int w = 0; w < warp; ++w) run += S.wsum[w];
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int r = tid * kPer + j;
        if (r < nrec) pre[r] = run;
        run += loc[j];
      }
      if (tid == kWarps * 32 - 1) pre[nrec] = run;
    }
    __syncthreads();
    const uint32_t total = pre[nrec];
    // list overflow of this chunk (kListExactHist with a staging area): positions beyond the
    // shared list go to a block of the staging area sized by the chunk's entry count
    constexpr uint32_t kLCap = COMPACT ? 2 * kCap : kCap;
    unsigned long long stg = 0;
    bool stg_ok = false;
    if (MODE == kListExactHist && stage) {
      if (tid == 0) {
        const uint32_t c0 = S.count, lo = max(c0, kLCap), hi = c0 + total;
        if (hi > lo && !S.stg_fail) {
          if (S.nstg >= kStgChunks) {
            S.stg_fail = 1;
          } else {
            const unsigned long long b0 = atomicAdd(stage_used, (unsigned long long)(hi - lo));
            if (b0 + (hi - lo) > stage_cap) {
              S.stg_fail = 1;
            } else {
              S.stg_lo[S.nstg] = lo;
              S.stg_off[S.nstg] = b0 - lo;
              ++S.nstg;
            }
          }
        }
      }
      __syncthreads();
      stg_ok = !S.stg_fail && S.nstg > 0;
      if (stg_ok) stg = S.stg_off[S.nstg - 1];
    }
    // every warp walks a contiguous quarter of the entries in batches of 32.  Records hold >= 1
    // entry, so at most 32 record starts fall in (e0, e0 + 32]: one load of the next 32 prefix
    // sums places every lane's entry in its record (no per-entry search)
    const uint32_t chunk = (total + kWarps * 32 - 1) / (kWarps * 32) * 32;
    const uint32_t wbeg = min(total, (uint32_t)warp * chunk), wend = min(total, wbeg + chunk);
    int cur = 0;  // record holding entry e0 (warp-uniform): pre[cur] <= e0 < pre[cur + 1]
    if (wbeg < wend) {
      int hi = nrec;
      while (hi - cur > 1) {
        const int mid = (cur + hi) >> 1;
        if (pre[mid] <= wbeg) cur = mid; else hi = mid;
      }
    }
    // batch e0: its record lo and centre entry; the next batch's entry is loaded before the
    // current one is processed (its latency overlaps the tests and list appends)
    auto locate = [&](uint32_t e0, int& lo, uint2& en) {
      const int j = cur + 1 + lane;
      const uint32_t off = (j <= nrec ? pre[j] : 0xFFFFFFFFu) - e0;  // record j starts at e0 + off
      const uint32_t starts = __reduce_or_sync(kFull, off - 1u < 31u ? 1u << off : 0u);
      lo = cur + __popc(starts & ((2u << lane) - 1u));
      cur += __popc(__ballot_sync(kFull, off - 1u < 32u));
      en = make_uint2(0u, 0u);
      if (e0 + lane < wend) {
        const uint32_t k = (rec[3 * lo + 1] & 0xFFFFu) + (e0 + lane - pre[lo]);
        en = __ldg(cent + (size_t)rec[3 * lo] * kTileVol + k);
      }
    };
    int lo_n = 0;
    uint2 en_n = make_uint2(0u, 0u);
    if (wbeg < wend) locate(wbeg, lo_n, en_n);
    for (uint32_t e0 = wbeg; e0 < wend; e0 += 32) {
      const uint32_t e = e0 + lane;
      const int lo = lo_n;
      const uint2 en = en_n;
      if (e0 + 32 < wend) locate(e0 + 32, lo_n, en_n);
      bool take = false;
      int bk = -1;
      unsigned long long pe = 0;
      uint32_t pe32 = 0;
      if (e < wend) {
        const uint32_t o = rec[3 * lo + 2];
        const uint32_t v = en.x;  // element index in the home tile (row * 32 + x)
        const int cx = (int)(o & 0xFFFFu) - kOff + (int)(v & 31u),
                  cy = (int)(o >> 16) - kOff + (int)((v >> 5) & (uint32_t)(P::TY - 1)),
                  cz = (int)recz[lo] + (int)(v / (32u * P::TY));
        const int ddx = gap(bb0, bb1, cx), ddy = gap(bb2, bb3, cy), ddz = gap(bb4, bb5, cz);
        // the bucket range test is void for a full-range pass (warp-uniform)
        bool inr = true;
        if (MODE == kListBucketHist || !full_range) {
          bk = dbucket(en.y);
          inr = bk >= blo && bk <= bhi;
        }
        if (dlo_f != 0u || dhi_f != 0xFFFFFFFFu)  // (warp-uniform) the cover cut / an exact-D sub-range
          inr = inr && en.y >= dlo_f && en.y <= dhi_f;
#ifdef FASTRS_GATHER_STATS
        {
          const int hox = (int)(o & 0xFFFFu) - kOff, hoy = (int)(o >> 16) - kOff, hoz = (int)recz[lo];
          const int gx = max(0, max(hox - bb1, bb0 - (hox + kTX - 1)));
          const int gy = max(0, max(hoy - bb3, bb2 - (hoy + P::TY - 1)));
          const int gz = max(0, max(hoz - bb5, bb4 - (hoz + P::TZ - 1)));
          const bool dcut = gx * gx + gy * gy + gz * gz > (int)en.y - 1;
          const bool tk = ddx * ddx + ddy * ddy + ddz * ddz <= (int)en.y - 1 && inr;
          atomicAdd(&g_stats_ptr[0], 1ull);
          if (dcut) atomicAdd(&g_stats_ptr[1], 1ull);
          if (tk) atomicAdd(&g_stats_ptr[2], 1ull);
        }
#endif
        if (ddx * ddx + ddy * ddy + ddz * ddz <= (int)en.y - 1 && inr) {
          take = true;
          pe = pack(cx, cy, cz, en.y);
          if (COMPACT) pe32 = pack32(cx, cy, cz, en.y);
        }
      }
      const uint32_t tm = __ballot_sync(kFull, take);
      if (tm) {
        if (MODE == kScatter) {
          if (take) out[atomicAdd(&S.dh[dtop - (uint32_t)(pe & 0xFFFFu)], 1u)] = pe;
        } else if (MODE == kExactCount) {
          if (take) atomicAdd(&S.dh[dtop - (uint32_t)(pe & 0xFFFFu)], 1u);
        } else {
          if (MODE == kListBucketHist) {
            const uint32_t grp = __match_any_sync(kFull, take ? bk : -1);
            if (take && lane == __ffs(grp) - 1) atomicAdd(&S.bhist[bk], (uint32_t)__popc(grp));
          }
          if (MODE == kListExactHist && take) atomicAdd(&S.dh[dtop - (uint32_t)(pe & 0xFFFFu)], 1u);
          uint32_t base = 0;
          if (lane == 0) base = atomicAdd(&S.count, (uint32_t)__popc(tm));
          base = __shfl_sync(kFull, base, 0);
          const uint32_t pos = base + __popc(tm & ((1u << lane) - 1u));
          if (COMPACT) {
            if (take && pos < 2 * kCap) S.list32[pos] = pe32;
          } else {
            if (take && pos < kCap) S.list[pos] = pe;
          }
          if (MODE == kListExactHist && take && pos >= kLCap && stg_ok) stage[stg + pos] = pe;
        }
      }
    }
  }
  __syncthreads();
}

// [lo, hi] = x range of the set bits of a row mask; an empty mask gives a range no ball reaches
__device__ __forceinline__ void uncovered_range(uint32_t u, int& lo, int& hi) {
  lo = u ? __ffs(u) - 1 : 1 << 14;
  hi = u ? 31 - __clz(u) : -(1 << 14);
}

// 64-bit mask of the tile rows (row = lz*TY + ly) inside [ya,yb] x [za,zb]
template <bool IS3D>
__device__ __forceinline__ unsigned long long row_box(int ya, int yb, int za, int zb) {
  if (IS3D) {
    const unsigned long long ym = (unsigned long long)range_mask(ya, yb) * 0x0101010101010101ull;
    const unsigned long long zhi = zb >= 7 ? ~0ull : ((1ull << (8 * (zb + 1))) - 1ull);
    return ym & zhi & (~0ull << (8 * za));
  } else {
    const unsigned long long hi = yb >= 63 ? ~0ull : ((1ull << (yb + 1)) - 1ull);
    return hi & (~0ull << ya);
  }
}

template <bool IS3D>
__device__ __forceinline__ void gather_group(const uint32_t group_id, Smem& S, const uint32_t* __restrict__ fgm,
                                             const TileMeta* __restrict__ meta, const uint2* __restrict__ cent,
                                             const uint16_t* __restrict__ oct, uint32_t* __restrict__ fbl,
                                             const Geom& g, int gather_mode, unsigned long long* __restrict__ pool,
                                             unsigned long long pool_cap, uint32_t* __restrict__ gcount,
                                             uint32_t* __restrict__ goff, WsHeader* __restrict__ hdr,
                                             const GroupDivs& gd, int wave, uint32_t* __restrict__ defer_out) {
  using P = Shape<IS3D>;
  constexpr int TY = P::TY, TZ = P::TZ;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t dmax = hdr->dmax;

  // ---- group / tile coordinates --------------------------------------------------------
  // groups tile the layers [tz_lo, tz_hi) (all layers except on the slab path)
  uint32_t t = group_id, rq;
  t = gd.x.divmod(t, rq);
  const int64_t gxi = rq;
  t = gd.y.divmod(t, rq);
  const int64_t gyi = rq;
  t = gd.z.divmod(t, rq);
  const int64_t gzi = rq;
  const int64_t b = t;
  const int64_t tx0 = gxi * P::GX, ty0 = gyi * P::GY, tz0 = g.tz_lo + gzi * P::GZ;
  const int wx = warp % P::GX, wy = (warp / P::GX) % P::GY, wz = warp / (P::GX * P::GY);
  const int64_t mtx = tx0 + wx, mty = ty0 + wy, mtz = tz0 + wz;
  const bool have_tile = mtx < g.ntx && mty < g.nty && mtz < g.tz_hi;
  const int64_t mtile = have_tile ? ((b * g.ntz + mtz) * g.nty + mty) * g.ntx + mtx : 0;
  const int mox = wx * kTX, moy = wy * TY, moz = wz * TZ;  // my tile origin within the group
  const bool active = have_tile && meta[mtile].nfg != 0;
  const int64_t group = group_id;
  if (__syncthreads_or(active) == 0) {  // the whole group is background
    if (tid == 0) gcount[group] = 0;
    return;
  }
  if (gather_mode & kGatherForceFallback) {
    if (lane == 0 && have_tile) fbl[atomicAdd(&hdr->n_fb, 1u)] = (uint32_t)mtile;
    if (tid == 0) gcount[group] = kGroupFallback;
    return;
  }
  // bounding box of the group's foreground (K4's row masks): candidates must reach it
  if (tid == 0) {
    S.bb[0] = S.bb[2] = S.bb[4] = 1 << 20;
    S.bb[1] = S.bb[3] = S.bb[5] = -(1 << 20);
  }
  __syncthreads();
  {
    uint32_t xm = 0;
    int y0 = 1 << 20, y1 = -(1 << 20), z0 = 1 << 20, z1 = -(1 << 20);
    if (active) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int row = lane + 32 * k;
        const uint32_t f = fgm[mtile * kRows + row];
        if (f) {
          xm |= f;
          const int ly = row % TY + moy, lz = row / TY + moz;
          y0 = min(y0, ly); y1 = max(y1, ly); z0 = min(z0, lz); z1 = max(z1, lz);
        }
      }
    }
    xm = __reduce_or_sync(kFull, xm);
    y0 = __reduce_min_sync(kFull, y0); y1 = __reduce_max_sync(kFull, y1);
    z0 = __reduce_min_sync(kFull, z0); z1 = __reduce_max_sync(kFull, z1);
    if (lane == 0 && xm) {
      atomicMin(&S.bb[0], mox + __ffs(xm) - 1);
      atomicMax(&S.bb[1], mox + 31 - __clz(xm));
      atomicMin(&S.bb[2], y0); atomicMax(&S.bb[3], y1);
      atomicMin(&S.bb[4], z0); atomicMax(&S.bb[5], z1);
    }
  }
  __syncthreads();
  const int rmax = dmax > 0 ? isqrt16((int)(dmax - 1)) : 0;
  const int nrx = (rmax + kTX - 1) / kTX, nry = (rmax + TY - 1) / TY, nrz = IS3D ? (rmax + TZ - 1) / TZ : 0;
  // ---- cover cut.  The largest kept ball that reaches the group: when it contains every
  // foreground cell of the group, no ball with a smaller D can carry the maximum at any of them
  // (LT^2 = max over the covering balls), so the gather keeps D >= its D only.  Exact, and it
  // turns the candidate lists of large objects (the centre ball of a big sphere covers whole
  // groups; thousands of nearly tangent balls reach them) into a handful of entries.
  // (only for Dmax > kHist, the D-bucket rounds path: below it the candidate lists are bounded by
  // the reach of balls of radius < 40 and the cut's extra dependent loads cost more than it saves
  // -- C4: k5 11.56 -> 12.64 ms with the cut on every group)
  uint32_t dcut = 0;
  if (!(gather_mode & kGatherNoCoverCut) && dmax > (uint32_t)kHist) {
    if (tid == 0) {
      S.topkey = 0ull;
      S.qstar[3] = 0;
    }
    __syncthreads();
    const int nx = P::GX + 2 * nrx, ny = P::GY + 2 * nry, nz = P::GZ + 2 * nrz;
    const int bb0 = S.bb[0], bb1 = S.bb[1], bb2 = S.bb[2], bb3 = S.bb[3], bb4 = S.bb[4], bb5 = S.bb[5];
    for (int n = tid; n < nx * ny * nz; n += kWarps * 32) {
      const int ix = n % nx, iy = (n / nx) % ny, iz = n / (nx * ny);
      const int64_t hx = tx0 + ix - nrx, hy = ty0 + iy - nry, hz = tz0 + iz - nrz;
      if (hx < 0 || hx >= g.ntx || hy < 0 || hy >= g.nty || hz < 0 || hz >= g.ntz) continue;
      const int64_t ht = ((b * g.ntz + hz) * g.nty + hy) * g.ntx + hx;
      const TileMeta hm = meta[ht];
      if (!hm.count) continue;
      const int hox = (ix - nrx) * kTX, hoy = (iy - nry) * TY, hoz = (iz - nrz) * TZ;
      const int gx = max(0, max(hox - bb1, bb0 - (hox + kTX - 1)));
      const int gy = max(0, max(hoy - bb3, bb2 - (hoy + TY - 1)));
      const int gz = max(0, max(hoz - bb5, bb4 - (hoz + TZ - 1)));
      if (gx * gx + gy * gy + gz * gz > (int)hm.maxD - 1) continue;
      atomicMax(&S.topkey, ((unsigned long long)hm.maxD << 32) | (unsigned long long)n);
    }
    __syncthreads();
    const unsigned long long key = S.topkey;
    if (key) {
      const uint32_t dstar = (uint32_t)(key >> 32);
      const int n = (int)(key & 0xFFFFFFFFu);
      const int ix = n % nx, iy = (n / nx) % ny, iz = n / (nx * ny);
      if (warp == 0) {  // an entry with D == dstar in the head of that tile's bucket-sorted list
        const int64_t ht = ((b * g.ntz + (tz0 + iz - nrz)) * g.nty + (ty0 + iy - nry)) * g.ntx + (tx0 + ix - nrx);
        const uint32_t cnt = meta[ht].count;
        const uint2* lst = cent + (size_t)ht * kTileVol;
        for (uint32_t k0 = 0; k0 < cnt; k0 += 32) {
          const uint2 en = k0 + lane < cnt ? lst[k0 + lane] : make_uint2(0u, 0u);
          const uint32_t hit = __ballot_sync(kFull, k0 + lane < cnt && en.y == dstar);
          if (hit) {
            if (lane == __ffs(hit) - 1) {
              const uint32_t v = en.x;
              S.qstar[0] = (ix - nrx) * kTX + (int)(v & 31u);
              S.qstar[1] = (iy - nry) * TY + (int)((v >> 5) & (uint32_t)(TY - 1));
              S.qstar[2] = (iz - nrz) * TZ + (int)(v / (32u * TY));
              S.qstar[3] = 1;
            }
            break;
          }
        }
      }
      __syncthreads();
      bool ok = S.qstar[3] != 0;
      if (ok && active) {  // every foreground row of my tile inside the chord of B(q*)
        const int qx = S.qstar[0] - mox;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int row = lane + 32 * k;
          const uint32_t f = fgm[mtile * kRows + row];
          if (!f) continue;
          const int dy = row % TY + moy - S.qstar[1], dz = row / TY + moz - S.qstar[2];
          const int h = (int)dstar - 1 - dy * dy - dz * dz;
          if (h < 0) {
            ok = false;
            continue;
          }
          const int w = isqrt16(h);
          const int l = qx - w, r = qx + w;
          const uint32_t allowed = (r < 0 || l > 31) ? 0u : range_mask(max(l, 0), min(r, 31));
          if (f & ~allowed) ok = false;
        }
      }
      if (__syncthreads_and(ok)) dcut = dstar;
    }
  }
  const int bcut = dcut ? dbucket(dcut) : 0;
  uint32_t written = 0;
  if (tid == 0) {
    S.fallback = 0;
    S.defer = 0;
    S.base = 0;
  }
  __syncthreads();
  if (dmax <= (uint32_t)kHist) {
    // ---- single pass: the exact-D histogram is built while gathering, the group's slice of
    // the global pool is allocated, and the list is scattered to its sorted (descending D)
    // positions; a list that overflowed the shared buffer is regathered straight to the pool
    const uint32_t dtop = dmax;
    for (int k = tid; k < (int)dtop; k += kWarps * 32) S.dh[k] = 0;
    if (tid == 0) {
      S.count = 0;
      S.nstg = 0;
      S.stg_fail = 0;
    }
    __syncthreads();
    // the pool's top half stages list overflow (the slices are allocated below it); a chunk
    // reserves room for all its examined entries, so the reservation is ~2x what is taken
    const unsigned long long main_cap = pool_cap - pool_cap / 2;
    unsigned long long* stage = (gather_mode & kGatherNoStaging) ? nullptr : pool + main_cap;
    // (no cover cut on this path: dmax <= kHist, see above; literal full-range arguments keep
    // the bucket and D-range tests out of the entry loop)
    gather<IS3D, kListExactHist, IS3D>(S, meta, cent, oct, g, b, tx0, ty0, tz0, nrx, nry, nrz, 0, kBuckets - 1, dtop,
                                       nullptr, stage, &hdr->stage_used, pool_cap / 2);
    const uint32_t total = S.count;
#ifdef FASTRS_DEBUG_GATHER
    if (tid == 0 && group < 4)
      printf("gather g%lld wave %d total %u dtop %u nrx %d nry %d nrz %d bb %d %d %d %d %d %d pool_cap %llu\n",
             (long long)group, wave, total, dtop, nrx, nry, nrz, S.bb[0], S.bb[1], S.bb[2], S.bb[3], S.bb[4], S.bb[5],
             pool_cap);
#endif
    constexpr uint32_t kListCap = IS3D ? 2 * kCap : kCap;  // 3D keeps compact entries
    if (tid == 0) {
      const unsigned long long b0 = atomicAdd(&hdr->pool_used, (unsigned long long)total);
      S.base = b0;
      if (b0 + total > main_cap) {  // the pool is full: the next wave (the last: the fallback)
        if (wave + 1 < kDilateWaves) S.defer = 1;
        else S.fallback = 1;
      }
    }
    block_exclusive_scan(S.dh, (int)dtop, S.wsum);
    if (!S.fallback && !S.defer) {
      unsigned long long* out = pool + S.base;
      if (total <= kListCap || (stage && !S.stg_fail)) {
        const int nstg = S.nstg;
        if (total > kListCap && tid == 0) atomicAdd(&hdr->n_staged, 1u);
        for (uint32_t i = tid; i < total; i += kWarps * 32) {
          unsigned long long pe;
          if (i < kListCap) {
            pe = IS3D ? unpack32(S.list32[i]) : S.list[i];
          } else {  // staged: the last chunk block whose range starts at or below i
            int k = nstg - 1;
            while (k > 0 && S.stg_lo[k] > i) --k;
            pe = stage[S.stg_off[k] + i];
          }
          out[atomicAdd(&S.dh[dtop - (uint32_t)(pe & 0xFFFFu)], 1u)] = pe;
        }
      } else {
        if (tid == 0) atomicAdd(&hdr->n_regathers, 1u);
        gather<IS3D, kScatter>(S, meta, cent, oct, g, b, tx0, ty0, tz0, nrx, nry, nrz, 0, kBuckets - 1, dtop, out);
      }
      written = total;
    }
    __syncthreads();
  } else {
  // ---- rounds over D-bucket ranges (Dmax > kHist): each round an exactly sorted chunk
  unsigned long long* out = nullptr;
  if (tid == 0) {
    S.round_hi = kBuckets - 1;
    S.rounds = 0;
  }
  __syncthreads();
  for (;;) {
    const int rhi = S.round_hi;
    for (int i = tid; i < kBuckets; i += kWarps * 32) S.bhist[i] = 0;
    if (tid == 0) S.count = 0;
    __syncthreads();
    gather<IS3D, kListBucketHist>(S, meta, cent, oct, g, b, tx0, ty0, tz0, nrx, nry, nrz, bcut, rhi, 0, nullptr,
                                  nullptr, nullptr, 0, dcut);
    __syncthreads();
    // --- this round's bucket range [rlo, rhi]: as many buckets as fit the list and the sort
    // range (warp 0: descending inclusive scan of the histogram, 4 buckets per lane)
    if (warp == 0) {
      uint32_t h[4], sum = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // lane l holds buckets 127-4l .. 124-4l (descending order)
        const int k = kBuckets - 1 - 4 * lane - q;
        h[q] = k <= rhi ? S.bhist[k] : 0u;
        sum += h[q];
      }
      uint32_t inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += v;
      }
      uint32_t run = inc - sum;
      // the highest non-empty bucket bounds the round's D range from above
      int top_l = -1;
#pragma unroll
      for (int q = 3; q >= 0; --q) {
        const int k = kBuckets - 1 - 4 * lane - q;
        if (h[q] && k <= rhi) top_l = k;
      }
      const int top = __reduce_max_sync(kFull, top_l);
      const uint32_t dtop = min(dbucket_max(top < 0 ? 0 : top), dmax);  // bucket 127 is unbounded
      int lo_l = -1;  // the highest bucket that no longer fits (count or D range)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = kBuckets - 1 - 4 * lane - q;
        run += h[q];
        const uint32_t dmin_k = k == 0 ? 1u : dbucket_max(k - 1) + 1u;
        if (lo_l < 0 && k <= top && (run > kCap || dtop + 1u > (uint32_t)kHist + dmin_k)) lo_l = k;
      }
      const int lo = __reduce_max_sync(kFull, lo_l);
      uint32_t below = 0;  // candidates left for later rounds
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = kBuckets - 1 - 4 * lane - q;
        if (k <= lo) below += h[q];
      }
      below = __reduce_add_sync(kFull, below);
      if (lane == 31 && S.rounds == 0) {  // first round: the histogram covers every candidate
        const unsigned long long b0 = atomicAdd(&hdr->pool_used, (unsigned long long)inc);
        S.base = b0;
        if (b0 + inc > pool_cap - pool_cap / 2) {  // (the top half stages list overflow)
          if (wave + 1 < kDilateWaves) S.defer = 1;
          else S.fallback = 1;
        }
      }
      __syncwarp();
      if (lane == 0) {
        // a single bucket exceeds the list / range, or (defensive) too many rounds
        // a single bucket that exceeds the list / sort range (large objects: thousands of kept
        // balls of similar D reach the group) is written by exact-D scatter rounds below
        S.bigbucket = (lo == top && lo >= 0) ? 1 : 0;
        S.fallback = (S.fallback || ++S.rounds > kBuckets) ? 1 : 0;
        S.round_lo = lo + 1;
        S.round_top = top;
        S.next_hi = below ? lo : -1;
      }
    }
    __syncthreads();
    if (S.fallback || S.defer) break;
    if (S.bigbucket) {
      // exact-D scatter rounds over the bucket `top`, kHist D values at a time, highest first:
      // count the exact D of every candidate in the sub-range (no list), prefix-sum the counts
      // into cursors, gather again and store each candidate at its cursor.  Equal D may land in
      // any order (ties do not change the first cover), so no capacity limit applies.
      const int bk = S.round_top;
      const uint32_t dmin_b = bk == 0 ? 1u : dbucket_max(bk - 1) + 1u, dmax_b = min(dbucket_max(bk), dmax);
      for (int64_t dh = dmax_b; dh >= (int64_t)dmin_b; dh -= kHist) {
        const uint32_t dhu = (uint32_t)dh;
        if (dhu < dcut) break;
        const uint32_t dl = max(max(dmin_b, dcut), dhu >= (uint32_t)kHist ? dhu - (uint32_t)kHist + 1u : 1u);
        const int nbins = (int)(dhu - dl) + 1;
        for (int k = tid; k < kHist; k += kWarps * 32) S.dh[k] = 0;
        __syncthreads();
        gather<IS3D, kExactCount>(S, meta, cent, oct, g, b, tx0, ty0, tz0, nrx, nry, nrz, bk, bk, dhu, nullptr,
                                  nullptr, nullptr, 0, dl, dhu);
        const uint32_t cnt = block_exclusive_scan(S.dh, nbins, S.wsum);
        if (cnt) {
          gather<IS3D, kScatter>(S, meta, cent, oct, g, b, tx0, ty0, tz0, nrx, nry, nrz, bk, bk, dhu,
                                 pool + S.base + written, nullptr, nullptr, 0, dl, dhu);
          written += cnt;
        }
        if (tid == 0) atomicAdd(&hdr->n_rounds_extra, 1u);
        __syncthreads();
      }
      if (bk == 0) break;
      if (tid == 0) S.round_hi = bk - 1;
      __syncthreads();
      continue;
    }
    const int rlo = S.round_lo;
    if (S.count > kCap) {  // the list overflowed: gather again, keeping [rlo, rhi] only (they fit)
      if (tid == 0) atomicAdd(&hdr->n_regathers, 1u);
      __syncthreads();
      if (tid == 0) S.count = 0;
      __syncthreads();
      gather<IS3D, kListOnly>(S, meta, cent, oct, g, b, tx0, ty0, tz0, nrx, nry, nrz, max(rlo, bcut), rhi, 0, nullptr,
                              nullptr, nullptr, 0, dcut);
      __syncthreads();
    }
    // --- exact counting sort of the list indices by D (descending), D in [dlo, dhi]
    const int rtop = S.round_top;
    const uint32_t dhi = min(dbucket_max(rtop < 0 ? 0 : rtop), dmax), dlo = rlo == 0 ? 1u : dbucket_max(rlo - 1) + 1u;
    const int nb = (int)(dhi - dlo) + 1;
    const uint32_t n = min(S.count, (uint32_t)kCap);
    for (int k = tid; k < nb; k += kWarps * 32) S.hist[k] = 0;
    __syncthreads();
    for (uint32_t i = tid; i < n; i += kWarps * 32) {
      const uint32_t D = (uint32_t)(S.list[i] & 0xFFFFu);
      if (D >= dlo && D <= dhi) atomicAdd(&S.hist[dhi - D], 1u);
    }
    __syncthreads();
    {
      constexpr int kPer = kHist / (kWarps * 32);
      const int base = tid * kPer;
      uint32_t loc[kPer], sum = 0;
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        loc[j] = base + j < nb ? S.hist[base + j] : 0u;
        sum += loc[j];
      }
      uint32_t inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += v;
      }
      if (lane == 31) S.wsum[warp] = inc;
      __syncthreads();
      uint32_t run = inc - sum;
      for (int w = 0; w < warp; ++w) run += S.wsum[w];
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        if (base + j < nb) S.hist[base + j] = run;
        run += loc[j];
      }
      if (tid == kWarps * 32 - 1) S.total = run;
    }
    __syncthreads();
    for (uint32_t i = tid; i < n; i += kWarps * 32) {
      const uint32_t D = (uint32_t)(S.list[i] & 0xFFFFu);
      if (D >= dlo && D <= dhi) S.idx[atomicAdd(&S.hist[dhi - D], 1u)] = (uint16_t)i;
    }
    __syncthreads();
    const uint32_t total = S.total;
    const bool last_round = S.next_hi < 0;

    // --- append the round (exactly descending D) to the group's slice of the pool
    out = pool + S.base;
    for (uint32_t i = tid; i < total; i += kWarps * 32) out[written + i] = S.list[S.idx[i]];
    written += total;
    if (last_round) break;
    __syncthreads();
    if (tid == 0) {
      S.round_hi = S.next_hi;
      atomicAdd(&hdr->n_rounds_extra, 1u);
    }
    __syncthreads();
  }

  }
  if (S.defer) {  // the pool is full: the next wave gathers this group again
    if (tid == 0) {
      gcount[group] = kGroupDeferred;
      defer_out[atomicAdd(&hdr->n_defer[wave], 1u)] = (uint32_t)group;
    }
    return;
  }
  if (written > kGroupCountMask && tid == 0) S.fallback = 1;  // (no list is that long in practice)
  __syncthreads();
  if (S.fallback) {  // leave this group to k_dilate_atomic
    if (lane == 0 && active) fbl[atomicAdd(&hdr->n_fb, 1u)] = (uint32_t)mtile;
    if (tid == 0) {
      atomicAdd(&hdr->n_fallback, 1u);
      gcount[group] = kGroupFallback;
    }
    return;
  }
  if (tid == 0) {
    gcount[group] = ((uint32_t)wave << 29) | written;
    goff[group] = (uint32_t)S.base;
    atomicMax(&hdr->max_group_list, written);
    atomicAdd(&hdr->sum_group_list, (unsigned long long)written);
  }
}

__global__ void k_wave_reset(WsHeader* __restrict__ hdr, int wave) {
  if (threadIdx.x == 0 && hdr->n_defer[wave - 1] != 0u) {
    hdr->pool_used = 0ull;
    hdr->stage_used = 0ull;
    hdr->paint_next = 0u;
  }
}

// K5a kernel: wave 0 takes one group per CTA; a later wave loops over the groups the previous
// wave deferred (a list; few CTAs, and they leave at once when it is empty)
template <bool IS3D>
__global__ void __launch_bounds__(kWarps * 32, 7) k_dilate_gather(const uint32_t* __restrict__ fgm,
                                                                  const TileMeta* __restrict__ meta,
                                                                  const uint2* __restrict__ cent,
                                                                  const uint16_t* __restrict__ oct,
                                                                  uint32_t* __restrict__ fbl, Geom g, int gather_mode,
                                                                  unsigned long long* __restrict__ pool,
                                                                  unsigned long long pool_cap,
                                                                  uint32_t* __restrict__ gcount,
                                                                  uint32_t* __restrict__ goff,
                                                                  WsHeader* __restrict__ hdr, GroupDivs gd, int wave,
                                                                  const uint32_t* __restrict__ defer_in,
                                                                  uint32_t* __restrict__ defer_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  if (hdr->dmax > kU16Max) return;  // k_dilate_atomic handles it
  if (wave == 0) {
    gather_group<IS3D>(blockIdx.x, S, fgm, meta, cent, oct, fbl, g, gather_mode, pool, pool_cap, gcount, goff, hdr, gd,
                       wave, defer_out);
    return;
  }
  const uint32_t n = *(volatile uint32_t*)&hdr->n_defer[wave - 1];
  for (uint32_t k = blockIdx.x; k < n; k += gridDim.x) {
    gather_group<IS3D>(defer_in[k], S, fgm, meta, cent, oct, fbl, g, gather_mode, pool, pool_cap, gcount, goff, hdr,
                       gd, wave, defer_out);
    __syncthreads();  // the shared state is rebuilt for the next group
  }
}

// Fused K5b reductions: the warp's queued covering events (lanes = events): the label of each
// event's first cell (tile_labels: the tile origin in the label array), then the per-label
// warp aggregation and the global atomics (dilate_common.cuh accumulate_records).  Out of line:
// it runs once per 32 events and keeps the paint loop's registers free.
template <bool IS3D>
__device__ __noinline__ void flush_events(const uint32_t* qa, const uint32_t* qb, int n,
                                          const int32_t* __restrict__ tile_labels, int64_t Y, int64_t X, int64_t b,
                                          const Accum& acc, const unsigned long long* __restrict__ fxlut) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  int32_t L = 0;
  uint32_t cnt = 0, scnt = 0, D = 0;
  if (lane < n) {
    const uint32_t ea = qa[lane], eb = qb[lane];
    const int off = (int)(ea & 0xFFFFu), row = off >> 5;
    const int ly = IS3D ? (row & 7) : row, lz = IS3D ? (row >> 3) : 0;
    L = __ldg(tile_labels + ((int64_t)lz * Y + ly) * X + (off & 31));
    cnt = ea >> 16;
    D = eb & 0xFFFFu;
    scnt = eb >> 16;
  }
  __syncwarp();  // the queue may be refilled after this
  accumulate_records(L, cnt, scnt, D, lane, b, acc, fxlut);
}

template <bool IS3D, int NW, bool FUSED>
__device__ __forceinline__ void paint_tile(const uint32_t bid, const uint32_t* __restrict__ fgm,
                                           const uint32_t* __restrict__ shm, const TileMeta* __restrict__ meta,
                                           const Geom& g, const unsigned long long* __restrict__ pool,
                                           const uint32_t* __restrict__ gcount, const uint32_t* __restrict__ goff,
                                           int point_at, uint32_t* __restrict__ ltp, const int32_t* __restrict__ labels,
                                           const Accum& acc, const unsigned long long* __restrict__ fxlut,
                                           const uint32_t* __restrict__ Dp, int approx, WsHeader* __restrict__ hdr,
                                           const GroupDivs& gd, int wave) {
  using P = Shape<IS3D>;
  constexpr int TY = P::TY, TZ = P::TZ;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PaintSmem<NW, FUSED>& S = *reinterpret_cast<PaintSmem<NW, FUSED>*>(smem_raw);
  // bid numbers tiles: group bid / kWarps, tile bid % kWarps within it; wl = my warp's smem slot
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int warp = (int)(bid % kWarps);  // my tile within the group
  const int64_t group = bid / kWarps;

  // ---- group / tile coordinates --------------------------------------------------------
  // groups tile the layers [tz_lo, tz_hi) (all layers except on the slab path)
  uint32_t t = (uint32_t)group, rq;
  t = gd.x.divmod(t, rq);
  const int64_t gxi = rq;
  t = gd.y.divmod(t, rq);
  const int64_t gyi = rq;
  t = gd.z.divmod(t, rq);
  const int64_t gzi = rq;
  const int64_t b = t;
  const int64_t tx0 = gxi * P::GX, ty0 = gyi * P::GY, tz0 = g.tz_lo + gzi * P::GZ;
  const int64_t rox = tx0 * kTX, roy = ty0 * TY, roz = tz0 * TZ;  // group origin
  const int wx = warp % P::GX, wy = (warp / P::GX) % P::GY, wz = warp / (P::GX * P::GY);
  const int64_t mtx = tx0 + wx, mty = ty0 + wy, mtz = tz0 + wz;
  const bool have_tile = mtx < g.ntx && mty < g.nty && mtz < g.tz_hi;
  const int64_t mtile = have_tile ? ((b * g.ntz + mtz) * g.nty + mty) * g.ntx + mtx : 0;
  const int mox = wx * kTX, moy = wy * TY, moz = wz * TZ;  // my tile origin within the group
  const bool active = have_tile && meta[mtile].nfg != 0;
  uint32_t total = gcount[group];
  // background, left to k_dilate_atomic, deferred, or gathered by another wave
  if (!active || total >= kGroupDeferred || (total >> 29) != (uint32_t)wave) return;
  total &= kGroupCountMask;
  const unsigned long long* list = pool + goff[group];
  const int64_t item = b * g.Z * g.Y * g.X;

  // ---- per-warp init: values, foreground masks, coverage ----------------------------------
  uint16_t* val = S.val[wl];
  if (!FUSED) {
    uint4* v4 = reinterpret_cast<uint4*>(val);
#pragma unroll 4
    for (int i = lane; i < kRows * 32 / 8; i += 32) v4[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  // lane owns rows `lane` (0) and `lane + 32` (1): foreground and covered masks in registers
  const uint32_t f0 = active ? fgm[mtile * kRows + lane] : 0u, f1 = active ? fgm[mtile * kRows + lane + 32] : 0u;
  // fused: shell masks of the same rows, and the queue of covering events.  An event is one
  // ball covering `count` still-uncovered cells of one label (its own), `scount` of them shell
  // cells, with LT^2 = D for each (exact descending order: the first cover is the max).  A
  // full queue is flushed: lanes = events, the label of each event's first cell is read, and
  // the events are summed per label in the warp before the global atomics.
  const uint32_t s0 = FUSED ? shm[mtile * kRows + lane] : 0u, s1 = FUSED ? shm[mtile * kRows + lane + 32] : 0u;
  int nev = 0;  // queued events (warp-uniform)
  uint32_t* qa = S.qa[wl];
  uint32_t* qb = S.qb[wl];
  const int64_t tgx = rox + mox, tgy = roy + moy, tgz = roz + moz;  // my tile's origin in the item
  auto ev_flush = [&]() {
    flush_events<IS3D>(qa, qb, nev, labels + item + (tgz * g.Y + tgy) * g.X + tgx, g.Y, g.X, b, acc, fxlut);
    nev = 0;
  };
  auto ev_push = [&](uint32_t off, uint32_t cnt, uint32_t D, uint32_t scnt) {  // warp-uniform call, lane 0 stores
    if (lane == 0) {
      qa[nev] = off | (cnt << 16);
      qb[nev] = D | (scnt << 16);
    }
    if (++nev == 32) ev_flush();
  };
  uint32_t c0 = 0, c1 = 0;
  int ul0, uh0, ul1, uh1;  // x range of the uncovered foreground of rows lane / lane + 32
  uncovered_range(f0, ul0, uh0);
  uncovered_range(f1, ul1, uh1);
  const int ly0 = IS3D ? (lane & 7) : lane, lz0 = IS3D ? (lane >> 3) : 0;
  const int ly1 = IS3D ? ly0 : lane + 32;  // row lane + 32 lies 4 layers above row lane in 3D
  // rows of my tile that still hold uncovered foreground, per 8-column chunk of x
  // (in shared memory: four 64-bit masks read by two 16-byte loads per screened batch, instead
  // of eight registers the paint loop would push to local memory)
  unsigned long long* Uc = S.uc[wl];
#pragma unroll
  for (int c = 0; c < kUcChunks; ++c) {
    const unsigned long long m = (unsigned long long)__ballot_sync(kFull, (f0 >> (kUcW * c)) & kUcBits) |
                                 ((unsigned long long)__ballot_sync(kFull, (f1 >> (kUcW * c)) & kUcBits) << 32);
    if (lane == 0) Uc[c] = m;
  }
  __syncwarp();
  // uncovered foreground cells of my tile (warp-uniform); point mode once it is small
  int nu = (int)__reduce_add_sync(kFull, (uint32_t)(__popc(f0) + __popc(f1)));
  // FASTRS_APPROX_LT: the exact cover stops once at most 4 % of the
  // tile's foreground is uncovered; those cells take LT^2 = D (their own ball)
  const int stop = approx ? min(nu * 4 / 100, kPoint - 1) : 0;
  int4* sball = S.sball[wl];                 // survivors of a screened batch (cx, cy, cz, D)
  unsigned long long* scand = S.scand[wl];   // their candidate rows
  bool pmode = false;
  uint16_t* ulist = S.ulist[wl];
  uint2* pcell = S.pcell[wl];
  int ub[6] = {0, kTX - 1, 0, TY - 1, 0, TZ - 1};  // bounding box of the uncovered cells
  // the box from the coverage registers (row mode): x from the OR of the uncovered rows, y/z
  // from the rows that still hold uncovered cells
  auto ubox_rows = [&]() {
    const uint32_t l0 = f0 & ~c0, l1 = f1 & ~c1;
    const uint32_t orx = __reduce_or_sync(kFull, l0 | l1);
    ub[0] = orx ? __ffs(orx) - 1 : 0;
    ub[1] = orx ? 31 - __clz(orx) : -1;
    constexpr int kBig = 1 << 20;
    int ylo = kBig, yhi = -kBig, zlo = kBig, zhi = -kBig;
    if (l0) ylo = yhi = ly0, zlo = zhi = lz0;
    if (l1) {
      const int y1 = IS3D ? ly0 : ly1, z1 = IS3D ? lz0 + 4 : 0;
      ylo = min(ylo, y1), yhi = max(yhi, y1), zlo = min(zlo, z1), zhi = max(zhi, z1);
    }
    ub[2] = __reduce_min_sync(kFull, ylo);
    ub[3] = __reduce_max_sync(kFull, yhi);
    ub[4] = __reduce_min_sync(kFull, zlo);
    ub[5] = __reduce_max_sync(kFull, zhi);
  };
  auto ubox_refresh = [&]() {
    int x0 = 1 << 20, x1 = -1, y0 = 1 << 20, y1 = -1, z0 = 1 << 20, z1 = -1;
    for (int q = lane; q < nu; q += 32) {
      const int e = ulist[q], x = e & 31, row = e >> 5;
      const int ly = IS3D ? (row & 7) : row, lz = IS3D ? (row >> 3) : 0;
      x0 = min(x0, x); x1 = max(x1, x); y0 = min(y0, ly); y1 = max(y1, ly); z0 = min(z0, lz); z1 = max(z1, lz);
    }
    ub[0] = __reduce_min_sync(kFull, x0); ub[1] = __reduce_max_sync(kFull, x1);
    ub[2] = __reduce_min_sync(kFull, y0); ub[3] = __reduce_max_sync(kFull, y1);
    ub[4] = __reduce_min_sync(kFull, z0); ub[5] = __reduce_max_sync(kFull, z1);
  };
  ubox_rows();
  // list the still-uncovered cells (row*32 + x) of my rows in ulist (nu <= kPoint of them)
  auto make_ulist = [&]() {
    const uint32_t left[2] = {f0 & ~c0, f1 & ~c1};
    const uint32_t cnt = __popc(left[0]) + __popc(left[1]);
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += v;
    }
    uint32_t pos = inc - cnt;
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      uint32_t m = left[kk];
      const int row = lane + 32 * kk;
      const int ly = IS3D ? (row & 7) : row, lz = IS3D ? (row >> 3) : 0;
      while (m) {
        const int c = __ffs(m) - 1;
        m &= m - 1;
        // byte 3 (multiplied by the centre's zero byte 3) carries the cell's shell bit
        const uint32_t sb = ((kk ? s1 : s0) >> c) & 1u;
        pcell[pos] = make_uint2((uint32_t)(2 * c) | ((uint32_t)(2 * ly) << 8) | ((uint32_t)(2 * lz) << 16) | (sb << 24),
                                (uint32_t)(-(c * c + ly * ly + lz * lz)));
        ulist[pos++] = (uint16_t)(row * 32 + c);
      }
    }
    __syncwarp();
  };
  int nq = 0;  // point mode: queued balls in sball (warp-uniform)
  // Point tests, lanes = queued balls, loop over the uncovered cells p (broadcast reads):
  // |p - c|^2 < D  <=>  2p.c - |p|^2 > |c|^2 - D, one byte dot product (IDP4A) per cell and ball
  // when every queued centre lies within [-128, 127] of the tile (radius <= ~96); otherwise
  // the distance is formed directly.
  auto point_flush = [&]() {
    int cx = 0, cy = 0, cz = 0, D = 0;
    if (lane < nq) {
      const int4 bp = sball[lane];
      cx = bp.x;
      cy = bp.y;
      cz = bp.z;
      D = bp.w;
    }
    nq = 0;
    const bool in8 = (unsigned)(cx + 128) < 256u && (unsigned)(cy + 128) < 256u && (unsigned)(cz + 128) < 256u;
    const bool wide = !__all_sync(kFull, in8);
    const int T = D != 0 ? cx * cx + cy * cy + cz * cz - D : 0x7FFFFFFF;
    const int C8 = (cx & 0xFF) | ((cy & 0xFF) << 8) | ((cz & 0xFF) << 16);
    bool hit = false;
    uint32_t cov = 0;  // bit k: list entry lane + 32k got covered
    // 32-bit shared address of the cell list (one register across the loop instead of a
    // rematerialised 64-bit generic pointer)
    uint32_t pc_sh;
    asm volatile("mov.u32 %0, %1;" : "=r"(pc_sh) : "r"((uint32_t)__cvta_generic_to_shared(pcell)));
    // fused: the cells each ball (lane) covers first are counted on its lane and queued as one
    // event per ball at the end of the flush (first cell, count, D, shell count)
    uint32_t pcnt = 0, pscnt = 0, pfirst = 0;
    auto on_hit = [&](int q, uint32_t bm, uint32_t px) {
      const int w = __ffs(bm) - 1;
      if (lane == (q & 31)) cov |= 1u << (q >> 5);
      if (!FUSED) {
        const int wD = __shfl_sync(kFull, D, w);
        if (lane == 0) val[ulist[q]] = (uint16_t)wD;
      } else if (lane == w) {
        if (pcnt == 0) pfirst = ulist[q];
        ++pcnt;
        pscnt += (px >> 24) & 1u;
      }
      hit = true;
    };
    if (!wide) {
      for (int q = 0; q < nu; ++q) {
        uint2 pq;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(pq.x), "=r"(pq.y) : "r"(pc_sh + 8u * (uint32_t)q));
        const uint32_t bm = __ballot_sync(kFull, __dp4a((int)pq.x, C8, (int)pq.y) > T);
        if (bm) on_hit(q, bm, pq.x);
      }
    } else {
      for (int q = 0; q < nu; ++q) {
        const uint2 pq = pcell[q];
        const int dx = (int)(pq.x & 0xFFu) / 2 - cx, dy = (int)((pq.x >> 8) & 0xFFu) / 2 - cy,
                  dz = (int)((pq.x >> 16) & 0xFFu) / 2 - cz;
        const uint32_t bm = __ballot_sync(kFull, dx * dx + dy * dy + dz * dz < D);
        if (bm) on_hit(q, bm, pq.x);
      }
    }
    if (FUSED && hit) {
      const uint32_t who = __ballot_sync(kFull, pcnt != 0);
      const int n = __popc(who);
      if (nev + n > 32) ev_flush();
      if (pcnt) {
        const int at = nev + __popc(who & ((1u << lane) - 1u));
        qa[at] = pfirst | (pcnt << 16);
        qb[at] = (uint32_t)D | (pscnt << 16);
      }
      nev += n;
      if (nev == 32) ev_flush();
    }
    if (hit) {  // drop the covered cells from the lists (the order of the list does not matter)
      uint32_t ek[kPointW];
      uint2 pk[kPointW];
      bool keep[kPointW];
#pragma unroll
      for (int k = 0; k < kPointW; ++k) {
        const int idx = lane + 32 * k;
        keep[k] = idx < nu && !((cov >> k) & 1u);
        ek[k] = keep[k] ? ulist[idx] : 0u;
        pk[k] = keep[k] ? pcell[idx] : make_uint2(0u, 0u);
      }
      __syncwarp();
      uint32_t newn = 0;
#pragma unroll
      for (int k = 0; k < kPointW; ++k) {
        const uint32_t km = __ballot_sync(kFull, keep[k]);
        if (keep[k]) {
          const uint32_t at = newn + __popc(km & ((1u << lane) - 1u));
          ulist[at] = (uint16_t)ek[k];
          pcell[at] = pk[k];
        }
        newn += __popc(km);
      }
      nu = (int)newn;
      __syncwarp();
      ubox_refresh();
    }
    __syncwarp();
  };

  uint32_t n_rows = 0, n_painted = 0, n_covering = 0;  // (the last two warp-uniform)
  bool dirty = false;  // my rows' coverage changed since the masks were last refreshed
  {
    // --- cover: my tile, balls in descending D.  Lanes first screen 32 balls at a time (reach
    // + rows with uncovered foreground inside the ball's x-extent); the surviving balls are
    // then painted one by one with the lanes over the tile's rows (lane = row, row + 32).
    // Because the order is exactly descending, the first ball that covers a cell carries its
    // final value: each cell is written once and coverage is updated immediately.
    // the next batch's entries are loaded one iteration ahead (their latency overlaps the
    // current batch's screening and painting)
    unsigned long long e_next = lane < total ? list[lane] : 0ull;
    for (uint32_t i0 = 0; i0 < total && nu > stop; i0 += 32) {
      const uint32_t i = i0 + lane;
      const unsigned long long e_cur = e_next;
      if (i0 + 32 < total) e_next = i + 32 < total ? list[i + 32] : 0ull;
      if (!pmode && nu <= point_at) {
        // switch to point mode: list the still-uncovered cells
        make_ulist();
        pmode = true;
        ubox_refresh();
      }
      if (pmode) {
        // point tests.  The next 32 balls are screened against the bounding box of the
        // still-uncovered cells and the survivors queued (order kept = descending D); a full
        // queue is flushed: lanes = queued balls, loop over the uncovered cells, a cell takes
        // the D of the first (largest) ball containing it.
        int cx = 0, cy = 0, cz = 0, D = 0;
        if (i < total) {
          const unsigned long long e = e_cur;
          D = (int)(e & 0xFFFFu);
          cx = (int)((e >> 16) & 0xFFFFu) - kOff - mox;
          cy = (int)((e >> 32) & 0xFFFFu) - kOff - moy;
          cz = (int)((e >> 48) & 0xFFFFu) - kOff - moz;
          const int ddx = gap(ub[0], ub[1], cx), ddy = gap(ub[2], ub[3], cy), ddz = gap(ub[4], ub[5], cz);
          if (ddx * ddx + ddy * ddy + ddz * ddz > D - 1) D = 0;
        }
        const uint32_t sv = __ballot_sync(kFull, D != 0);
        if (nq + __popc(sv) > 32) point_flush();
        if (nu <= stop) break;
        if (D != 0) sball[nq + __popc(sv & ((1u << lane) - 1u))] = make_int4(cx, cy, cz, D);
        nq += __popc(sv);
        __syncwarp();
        continue;
      }
      unsigned long long cand = 0;
      int cx = 0, cy = 0, cz = 0, D = 0;
      if (i < total) {
        const unsigned long long e = e_cur;
        D = (int)(e & 0xFFFFu);
        cx = (int)((e >> 16) & 0xFFFFu) - kOff - mox;
        cy = (int)((e >> 32) & 0xFFFFu) - kOff - moy;
        cz = (int)((e >> 48) & 0xFFFFu) - kOff - moz;
        const int R2 = D - 1;
        const int ddx = gap(ub[0], ub[1], cx), ddy = gap(ub[2], ub[3], cy), ddz = gap(ub[4], ub[5], cz);
        const int gx2 = ddx * ddx, gy2 = ddy * ddy, gz2 = ddz * ddz;
        if (gx2 + gy2 + gz2 <= R2) {
          // the extent of ball ∩ B along each axis (B = the bounding box of the tile's uncovered
          // cells): the half-chord at B's nearest point in the other two axes (a ball reaching
          // B from outside meets it in a cap much narrower than its radius)
          const int hx = isqrt16(R2 - gy2 - gz2), hy = isqrt16(R2 - gx2 - gz2);
          const int hz = IS3D ? isqrt16(R2 - gx2 - gy2) : 0;
          const int xa = max(cx - hx, ub[0]), xb = min(cx + hx, ub[1]);
          unsigned long long ux = 0;  // rows with uncovered foreground inside the ball's x-extent
#pragma unroll
          for (int c2 = 0; c2 < kUcChunks / 2; ++c2) {
            const ulonglong2 ua = reinterpret_cast<const ulonglong2*>(Uc)[c2];
            if (xa <= kUcW * (2 * c2) + kUcW - 1 && xb >= kUcW * (2 * c2)) ux |= ua.x;
            if (xa <= kUcW * (2 * c2 + 1) + kUcW - 1 && xb >= kUcW * (2 * c2 + 1)) ux |= ua.y;
          }
          cand = row_box<IS3D>(max(cy - hy, ub[2]), min(cy + hy, ub[3]), max(cz - hz, ub[4]), min(cz + hz, ub[5])) & ux;
        }
      }
      // survivors, compacted in lane order (= descending D) into the warp's buffer, then painted
      // one by one: every lane reads the ball (broadcast) and handles its own two rows
      const uint32_t act = __ballot_sync(kFull, cand != 0);
      if (act) {
        if (cand) {
          const int slot = __popc(act & ((1u << lane) - 1u));
          sball[slot] = make_int4(cx, cy, cz, D);
          scand[slot] = cand;
        }
        __syncwarp();
        const int ns = __popc(act);
        n_painted += ns;
#ifdef FASTRS_PAINT_OLD
        for (int j = 0; j < ns; ++j) {
          const int4 bp = sball[j];
          const int jR2 = bp.w - 1;
          uint32_t ecnt = 0, escnt = 0;  // fused: cells of my rows this ball covers first
          int efirst = -1;
          const uint2 jc2 = reinterpret_cast<const uint2*>(scand)[j];  // candidate rows 0-31 | 32-63
          const uint16_t dv = (uint16_t)bp.w;
          // 3D: rows lane and lane + 32 share ly, and lie 4 layers apart
          const int dy0 = ly0 - bp.y, dz0 = lz0 - bp.z;
          const int base0 = jR2 - dy0 * dy0;
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            const uint32_t hm = hf ? jc2.y : jc2.x;
            if (hm == 0u) continue;  // the ball has no candidate row in this half (warp-uniform)
            if (!((hm >> lane) & 1u)) continue;
            int hrem;
            if (IS3D) {
              const int dz = hf ? dz0 + 4 : dz0;
              hrem = base0 - dz * dz;
            } else {
              const int dy = (hf ? ly1 : ly0) - bp.y;
              hrem = jR2 - dy * dy;
            }
            if (hrem < 0) continue;
            // cheap reject: the row's uncovered cells all lie in [ul, uh]; the ball's chord
            // reaches none of them when the nearest point of that range is outside it
            const int ddx = max(max((hf ? ul1 : ul0) - bp.x, bp.x - (hf ? uh1 : uh0)), 0);
            if (ddx * ddx > hrem) continue;
            const int w = isqrt16(hrem);
            const int l = max(bp.x - w, 0), rr = min(bp.x + w, kTX - 1);
            if (l > rr) continue;
            ++n_rows;
            uint32_t m = (hf ? (f1 & ~c1) : (f0 & ~c0)) & range_mask(l, rr);
            if (!m) continue;
            dirty = true;
            if (hf) {
              c1 |= m;
              uncovered_range(f1 & ~c1, ul1, uh1);
            } else {
              c0 |= m;
              uncovered_range(f0 & ~c0, ul0, uh0);
            }
            if (FUSED) {
              ecnt += __popc(m);
              escnt += __popc(m & (hf ? s1 : s0));
              if (efirst < 0) efirst = (32 * hf + lane) * 32 + __ffs(m) - 1;
            } else {
              uint16_t* vr = val + (32 * hf + lane) * 32;
              do {
                const int c = __ffs(m) - 1;
                m &= m - 1;
                vr[c] = dv;
              } while (m);
            }
          }
          if (FUSED) {
            const uint32_t who = __ballot_sync(kFull, ecnt != 0);
            if (who) {
              ++n_covering;
              const uint32_t tc = __reduce_add_sync(kFull, ecnt), ts = __reduce_add_sync(kFull, escnt);
              const int off = __shfl_sync(kFull, efirst, __ffs(who) - 1);
              ev_push((uint32_t)off, tc, (uint32_t)bp.w, ts);
            }
          }
        }
#else
        // per ball: both of my rows in straight-line code (a row that is not a candidate, or
        // that the chord misses, gets an empty mask); the rare covering ball takes the branch
        const uint32_t lbit = 1u << lane;
        for (int j = 0; j < ns; ++j) {
          const int4 bp = sball[j];
          const uint2 jc2 = reinterpret_cast<const uint2*>(scand)[j];  // candidate rows 0-31 | 32-63
          const int jR2 = bp.w - 1;
          int h0, h1;
          if (IS3D) {  // rows lane and lane + 32 share ly and lie 4 layers apart
            const int dy0 = ly0 - bp.y, dz0 = lz0 - bp.z, dz1 = dz0 + 4;
            const int base0 = jR2 - dy0 * dy0;
            h0 = base0 - dz0 * dz0;
            h1 = base0 - dz1 * dz1;
          } else {
            const int dy0 = ly0 - bp.y, dy1 = ly1 - bp.y;
            h0 = jR2 - dy0 * dy0;
            h1 = jR2 - dy1 * dy1;
          }
          // the nearest uncovered cell of each row must lie within the chord (cheap reject)
          const int dd0 = max(max(ul0 - bp.x, bp.x - uh0), 0), dd1 = max(max(ul1 - bp.x, bp.x - uh1), 0);
          const bool t0 = (jc2.x & lbit) && dd0 * dd0 <= h0, t1 = (jc2.y & lbit) && dd1 * dd1 <= h1;
          uint32_t m0 = 0, m1 = 0;
          if (t0) {
            const int w = isqrt16(h0);
            m0 = (f0 & ~c0) & range_mask(max(bp.x - w, 0), min(bp.x + w, kTX - 1));
          }
          if (t1) {
            const int w = isqrt16(h1);
            m1 = (f1 & ~c1) & range_mask(max(bp.x - w, 0), min(bp.x + w, kTX - 1));
          }
          const uint32_t who = __ballot_sync(kFull, (m0 | m1) != 0);
          if (who) {
            dirty = true;
            if (m0) {
              c0 |= m0;
              uncovered_range(f0 & ~c0, ul0, uh0);
            }
            if (m1) {
              c1 |= m1;
              uncovered_range(f1 & ~c1, ul1, uh1);
            }
            if (FUSED) {
              ++n_covering;
              const uint32_t ecnt = __popc(m0) + __popc(m1), escnt = __popc(m0 & s0) + __popc(m1 & s1);
              const int efirst = m0 ? lane * 32 + __ffs(m0) - 1 : (32 + lane) * 32 + __ffs(m1) - 1;
              const uint32_t tc = __reduce_add_sync(kFull, ecnt), ts = __reduce_add_sync(kFull, escnt);
              const int off = __shfl_sync(kFull, efirst, __ffs(who) - 1);
              ev_push((uint32_t)off, tc, (uint32_t)bp.w, ts);
            } else {
              const uint16_t dv = (uint16_t)bp.w;
#pragma unroll
              for (int hf = 0; hf < 2; ++hf) {
                uint32_t m = hf ? m1 : m0;
                uint16_t* vr = val + (32 * hf + lane) * 32;
                while (m) {
                  const int c = __ffs(m) - 1;
                  m &= m - 1;
                  vr[c] = dv;
                }
              }
            }
          }
        }
#endif
        __syncwarp();
      }
      // refresh the uncovered-row masks (only when this batch covered something)
      if (__any_sync(kFull, dirty)) {
        dirty = false;
        const uint32_t left[2] = {f0 & ~c0, f1 & ~c1};
#pragma unroll
        for (int c = 0; c < kUcChunks; ++c) {
          const unsigned long long m = (unsigned long long)__ballot_sync(kFull, (left[0] >> (kUcW * c)) & kUcBits) |
                                       ((unsigned long long)__ballot_sync(kFull, (left[1] >> (kUcW * c)) & kUcBits) << 32);
          if (lane == 0) Uc[c] = m;
        }
        nu = (int)__reduce_add_sync(kFull, (uint32_t)(__popc(left[0]) + __popc(left[1])));
        ubox_rows();
        __syncwarp();
      }
    }
    if (pmode && nq > 0 && nu > stop) point_flush();  // the queue's last balls
    if (approx && nu > 0) {
      // the approximate mode's remaining cells: LT^2 = D (lanes over the listed cells)
      if (!pmode) make_ulist();
      for (int q0 = 0; q0 < nu; q0 += 32) {
        const int q = q0 + lane;
        int32_t L = 0;
        uint32_t d = 0, sb = 0;
        if (q < nu) {
          const uint32_t e = ulist[q];
          const int row = (int)(e >> 5), x = (int)(e & 31u);
          const int ly = IS3D ? (row & 7) : row, lz = IS3D ? (row >> 3) : 0;
          const int64_t gi = item + ((tgz + lz) * g.Y + (tgy + ly)) * g.X + tgx + x;
          d = __ldg(Dp + gi);
          if (FUSED) {
            L = __ldg(labels + gi);
            sb = d == 1u ? 1u : 0u;  // shell <=> D == 1
          } else {
            val[e] = (uint16_t)d;
          }
        }
        if (FUSED) accumulate_records(L, L != 0 ? 1u : 0u, sb, d, lane, b, acc, fxlut);
      }
      nu = 0;
    }
  }


  n_rows = __reduce_add_sync(kFull, n_rows);
  if (lane == 0 && n_rows) atomicAdd(&hdr->n_intervals, (unsigned long long)n_rows);
  if (lane == 0 && n_painted) atomicAdd(&hdr->n_painted, (unsigned long long)n_painted);
  if (lane == 0 && n_covering) atomicAdd(&hdr->n_covering, (unsigned long long)n_covering);
  if (FUSED) {
    if (nev) ev_flush();
    // every foreground cell lies in some kept ball that reaches the tile
    if (nu != 0 && lane == 0) atomicOr(&hdr->status, kStInternal);
    return;
  }
  // ---- my tile's LT^2 -> the LT plane (coalesced rows); shell and reductions run in the
  // streaming epilogue kernel (lt.cu)
  // the LT plane holds u16 values whenever Dmax <= 65535 (always the case here)
  const int64_t gx = rox + mox + lane;
  const int64_t gy0 = roy + moy, gz0 = roz + moz;
  const bool full = gz0 + TZ <= g.Z && gy0 + TY <= g.Y && gx < g.X;  // interior tile: no bounds tests
  uint16_t* lt16 = reinterpret_cast<uint16_t*>(ltp) + item + (gz0 * g.Y + gy0) * g.X + gx;
  if (full) {
#pragma unroll 8
    for (int row = 0; row < kRows; ++row) {
      const int ly = row % TY, lz = row / TY;
      lt16[((int64_t)lz * g.Y + ly) * g.X] = val[row * 32 + lane];
    }
  } else {
    for (int row = 0; row < kRows; ++row) {
      const int ly = row % TY, lz = row / TY;
      if (gz0 + lz < g.Z && gy0 + ly < g.Y && gx < g.X) lt16[((int64_t)lz * g.Y + ly) * g.X] = val[row * 32 + lane];
    }
  }
}


// Persistent K5b: resident CTAs of NW independent warps take tiles from a global counter in
// launch order (the four tiles of a group one after another), so no warp slot idles between
// short tiles.
template <bool IS3D, int NW, int MINB, bool FUSED>
__global__ void __launch_bounds__(NW * 32, MINB) k_dilate_paint(const uint32_t* __restrict__ fgm,
                                                              const uint32_t* __restrict__ shm,
                                                              const TileMeta* __restrict__ meta, Geom g,
                                                              const unsigned long long* __restrict__ pool,
                                                              const uint32_t* __restrict__ gcount,
                                                              const uint32_t* __restrict__ goff, int point_at,
                                                              uint32_t* __restrict__ ltp,
                                                              const int32_t* __restrict__ labels, Accum acc,
                                                              const unsigned long long* __restrict__ fxlut,
                                                              const uint32_t* __restrict__ Dp, int approx,
                                                              WsHeader* __restrict__ hdr, uint32_t nbid, GroupDivs gd,
                                                              int wave) {
  if (hdr->dmax > kU16Max) return;  // k_dilate_atomic handles it
  if (wave > 0 && *(volatile uint32_t*)&hdr->n_defer[wave - 1] == 0u) return;  // nothing gathered this wave
  const int lane = threadIdx.x & 31;
  for (;;) {
    uint32_t bid = 0;
    if (lane == 0) bid = atomicAdd(&hdr->paint_next, 1u);
    bid = __shfl_sync(kFull, bid, 0);
    if (bid >= nbid) break;
    paint_tile<IS3D, NW, FUSED>(bid, fgm, shm, meta, g, pool, gcount, goff, point_at, ltp, labels, acc, fxlut, Dp, approx,
                                hdr, gd, wave);
    __syncwarp();
  }
}

}  // namespace

int64_t dilate_groups(const Geom& g) {
  const int GX = g.ndim == 3 ? 1 : 2, GY = 2, GZ = g.ndim == 3 ? 2 : 1;
  return g.B * ((g.ntx + GX - 1) / GX) * ((g.nty + GY - 1) / GY) * ((g.ntz + GZ - 1) / GZ);
}
// candidate pool: N/2 entries (C4: 4.3 GB; measured demand 0.16 entries per element); a group
// that does not fit is left to the fallback kernel
int64_t dilate_pool_entries(const Geom& g) {
  const int64_t n = g.N / 2 > (1 << 20) ? g.N / 2 : (1 << 20);
  return n < 0xFFFFFFFFll ? n : 0xFFFFFFFFll;  // offsets are u32
}

namespace {
int point_at_knob() { return kPoint; }  // uncovered cells at which a warp switches to point tests
int64_t launched_groups(const Geom& g) {
  const int GX = g.ndim == 3 ? 1 : 2, GY = 2, GZ = g.ndim == 3 ? 2 : 1;
  return g.B * ((g.ntx + GX - 1) / GX) * ((g.nty + GY - 1) / GY) * ((g.tz_hi - g.tz_lo + GZ - 1) / GZ);
}
}  // namespace

void launch_dilate_gather(const uint32_t* fgm, TileMeta* meta, const uint2* centres, const uint16_t* oct, uint32_t* fbl,
                          unsigned long long* pool, uint32_t* gcount, uint32_t* goff, const Geom& g, int gather_mode,
                          WsHeader* hdr, cudaStream_t st, int wave, uint32_t* deflists) {
  const int64_t ngroups = launched_groups(g);
  if (ngroups <= 0) return;
  unsigned long long pool_cap = (unsigned long long)dilate_pool_entries(g);
  if (const char* pd = getenv("FASTRS_POOL_DIV")) {  // test hook: a smaller pool (exercises the waves)
    const long long dv = atoll(pd);
    if (dv > 1) pool_cap = pool_cap / (unsigned long long)dv > 64 ? pool_cap / (unsigned long long)dv : 64;
  }
#ifdef FASTRS_GATHER_STATS
  {
    static const unsigned long long zero3[3] = {0, 0, 0};
    cudaMemcpyToSymbolAsync(g_stats_ptr, zero3, sizeof(zero3), 0, cudaMemcpyHostToDevice, st);
  }
#endif
  // each wave (and chunk) reuses the pool: its counters restart (a later wave: one tiny kernel,
  // which also restarts the paint's work counter, and only when the previous wave deferred groups)
  if (wave == 0) {
    cudaMemsetAsync(&hdr->stage_used, 0, sizeof(hdr->stage_used), st);
    cudaMemsetAsync(&hdr->pool_used, 0, sizeof(hdr->pool_used), st);
    cudaMemsetAsync(hdr->n_defer, 0, sizeof(hdr->n_defer), st);  // (the host pipeline runs waves per chunk)
  } else {
    k_wave_reset<<<1, 32, 0, st>>>(hdr, wave);
  }
  {
    // wave 0: one CTA per group; later waves: a few CTAs loop over the previous wave's list
    uint32_t grid = (uint32_t)ngroups;
    if (wave > 0) {
      int dev = 0, nsm = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      grid = (uint32_t)(nsm * 7) < grid ? (uint32_t)(nsm * 7) : grid;
    }
    const uint32_t* din = deflists + (size_t)((wave + 1) & 1) * (size_t)ngroups;  // written by wave - 1
    uint32_t* dout = deflists + (size_t)(wave & 1) * (size_t)ngroups;
    if (g.ndim == 3)
      k_dilate_gather<true><<<grid, kWarps * 32, sizeof(Smem), st>>>(fgm, meta, centres, oct, fbl, g, gather_mode, pool,
                                                                     pool_cap, gcount, goff, hdr, group_divs(g), wave,
                                                                     din, dout);
    else
      k_dilate_gather<false><<<grid, kWarps * 32, sizeof(Smem), st>>>(fgm, meta, centres, oct, fbl, g, gather_mode, pool,
                                                                      pool_cap, gcount, goff, hdr, group_divs(g), wave,
                                                                      din, dout);
  }
#ifdef FASTRS_GATHER_STATS
  cudaMemcpyFromSymbolAsync(hdr->g_stats, g_stats_ptr, 3 * sizeof(unsigned long long), 0, cudaMemcpyDeviceToDevice, st);
#endif
}

namespace {
template <bool IS3D, int NW, int MINB, bool FUSED>
void paint_go(int64_t ngroups, const uint32_t* fgm, const uint32_t* shm, const TileMeta* meta, const Geom& g,
              const unsigned long long* pool, const uint32_t* gcount, const uint32_t* goff, uint32_t* ltp,
              const int32_t* labels, const Accum& acc, const uint32_t* D, int approx, WsHeader* hdr,
              cudaStream_t st, int wave) {
  const uint32_t nbid = (uint32_t)(ngroups * kWarps);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t cap = (uint32_t)nsm * MINB * NW;  // resident warps
  const uint32_t grid = ((nbid < cap ? nbid : cap) + NW - 1) / NW;
  if (wave == 0) cudaMemsetAsync(&hdr->paint_next, 0, sizeof(uint32_t), st);  // (later waves: k_wave_reset)
  k_dilate_paint<IS3D, NW, MINB, FUSED><<<grid, NW * 32, sizeof(PaintSmem<NW, FUSED>), st>>>(
      fgm, shm, meta, g, pool, gcount, goff, point_at_knob(), ltp, labels, acc, device_fxlut(dev), D, approx, hdr, nbid,
      group_divs(g), wave);
}
}  // namespace

void launch_dilate_paint(const uint32_t* fgm, const uint32_t* shm, const TileMeta* meta,
                         const unsigned long long* pool, const uint32_t* gcount, const uint32_t* goff, const Geom& g,
                         uint32_t* ltp, const int32_t* labels, const Accum* acc, const uint32_t* D, bool approx,
                         WsHeader* hdr, cudaStream_t st, int wave) {
  const int ap = approx && D ? 1 : 0;
  const int64_t ngroups = launched_groups(g);
  if (ngroups <= 0) return;
  Accum a{};
  if (acc) a = *acc;
  if (g.ndim == 3) {
    if (acc) paint_go<true, kPaintNW, kPaintMinB, true>(ngroups, fgm, shm, meta, g, pool, gcount, goff, ltp, labels, a, D, ap, hdr, st, wave);
    else paint_go<true, kPaintNW, kPaintMinB, false>(ngroups, fgm, shm, meta, g, pool, gcount, goff, ltp, labels, a, D, ap, hdr, st, wave);
  } else {
    if (acc) paint_go<false, kPaintNW, kPaintMinB, true>(ngroups, fgm, shm, meta, g, pool, gcount, goff, ltp, labels, a, D, ap, hdr, st, wave);
    else paint_go<false, kPaintNW, kPaintMinB, false>(ngroups, fgm, shm, meta, g, pool, gcount, goff, ltp, labels, a, D, ap, hdr, st, wave);
  }
}

cudaError_t dilate_cover_setup() {
  cudaError_t e = cudaFuncSetAttribute(k_dilate_gather<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(Smem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_dilate_gather<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
  return e;
}

}  // namespace fastrs
