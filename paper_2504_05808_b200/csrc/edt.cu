// Exact label-aware squared EDT as three separable passes.
//
// D(p) = min over sites s of |p - s|^2, sites = elements with another label (plus the
// virtual border layer with FASTRS_BORDER_BACKGROUND): the substrate of local thickness
// (§4, "exact squared-distance computation via separable per-axis
// passes").  The passes reduce the global label-aware problem to per-RUN problems: along
// each axis an element only interacts with the same-label run it lies in, because every
// element beyond a run end is dominated by the run end's neighbour, which is itself a site
// at distance 0 in the partial field.
//
//   K1 edt_x : warp per row.  Two warp sweeps with ballot/ffs find run starts and ends;
//              g = (distance to the nearest run end's neighbour)^2.  Fused: label
//              validation (a1) and the y/z run-start flags packed into bits 31/30 (S2), so
//              later passes never re-read labels.
//   K2/K3    : column passes along y / z.  A CTA stages a [256 + 2*48][32] column tile in
//              shared memory (coalesced 128-byte rows) and each thread runs the exact
//              windowed scan  best = min(best, g(p +- dq) + dq^2)  until dq^2 >= best; the
//              default kernel packs both scan directions into u16 halves (one
//              VIADDMNMX.U16x2 per row pair, run ends folded into the staged values) and
//              hands CTAs with values >= 2^14-1 to the exact 32-bit kernel.  The final pass
//              emits D, Dmax, n_fg and flags elements with no site (ENOSITE).
#include <cstdlib>
#include <type_traits>
#include <mutex>

#include "common.cuh"

namespace fastrs {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

// K1, one warp per x-row.  FULL: X % 32 == 0 (no bounds tests).  Ly / Lz point at the row above
// in y / z, or at a row of -1 sentinels (no such neighbour: "first of its run" holds, as for a
// different label), so the loops carry no pointer tests.
template <int U, bool FULL>
__global__ void __launch_bounds__(256) k_edt_x(const int32_t* __restrict__ lab,
                                               const int32_t* __restrict__ below, const int32_t* __restrict__ sent,
                                               uint32_t* __restrict__ out, int64_t nrows, int X, int64_t Y, int64_t Z,
                                               int32_t max_label, int border, int is3d,
                                               WsHeader* __restrict__ hdr) {
  extern __shared__ uint16_t s_end[];
  const int warps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * warps + warp;
  if (row >= nrows) return;
  uint16_t* ends = s_end + (size_t)warp * X;
  const int64_t y = row % Y;
  const int64_t z = (row / Y) % Z;
  const int32_t* L = lab + row * X;
  const int32_t* Ly = y > 0 ? L - X : sent;
  // z-1 neighbour: the previous slice, or (slab path) the caller's slice just below the slab
  const int32_t* Lz = is3d ? (z > 0 ? L - X * Y : (below ? below + y * X : sent)) : sent;
  uint32_t* O = out + row * X;
  const int nchunk = (X + 31) >> 5;
  const uint32_t far = (uint32_t)kFull;  // "no site on this side" (unsigned distance)

  // sweep 1 (right to left): end of the run containing x (pointers step by 32 elements)
  int carry_end = X - 1;
  int32_t right_next = 0;
  const int32_t* pL = L + ((nchunk - 1) << 5) + lane;
#pragma unroll U
  for (int c = nchunk - 1; c >= 0; --c, pL -= 32) {
    const int x = (c << 5) + lane;
    const bool in = FULL || x < X;
    const int32_t v = in ? __ldg(pL) : 0;
    int32_t r = __shfl_down_sync(kFull, v, 1);
    if (lane == 31) r = right_next;
    const bool is_end = in && (x == X - 1 || v != r);
    const uint32_t m = __ballot_sync(kFull, is_end);
    const uint32_t ge = m & (kFull << lane);
    const int e = ge ? (c << 5) + __ffs(ge) - 1 : carry_end;
    if (in) ends[x] = (uint16_t)e;
    if (m) carry_end = (c << 5) + __ffs(m) - 1;
    right_next = __shfl_sync(kFull, v, 0);
  }

  // sweep 2 (left to right): start of the run, distances, flags
  int carry_start = 0;
  int32_t left_prev = 0;
  uint32_t bad = 0;
  const int32_t *qL = L + lane, *qY = Ly + lane, *qZ = Lz + lane;
  uint32_t* qO = O + lane;
#pragma unroll U
  for (int c = 0; c < nchunk; ++c, qL += 32, qY += 32, qZ += 32, qO += 32) {
    const int x = (c << 5) + lane;
    const bool in = FULL || x < X;
    const int32_t v = in ? __ldg(qL) : 0;
    const int32_t vy = in ? __ldg(qY) : 0, vz = in ? __ldg(qZ) : 0;
    int32_t l = __shfl_up_sync(kFull, v, 1);
    if (lane == 0) l = left_prev;
    const bool is_start = in && (x == 0 || v != l);
    const uint32_t m = __ballot_sync(kFull, is_start);
    const uint32_t le = m & (kFull >> (31 - lane));
    const int s = le ? (c << 5) + 31 - __clz(le) : carry_start;
    if (m) carry_start = (c << 5) + 31 - __clz(m);
    left_prev = __shfl_sync(kFull, v, 31);
    if (in) {
      uint32_t g = 0;
      if (v != 0) {
        bad |= (uint32_t)v > (uint32_t)max_label;  // also v < 0
        const int e = ends[x];
        const uint32_t dl = (s > 0 || border) ? (uint32_t)(x - s + 1) : far;
        const uint32_t dr = (e < X - 1 || border) ? (uint32_t)(e + 1 - x) : far;
        const uint32_t d = min(dl, dr);
        g = d == far ? kInf : d * d;
      }
      *qO = g | (vy != v ? kBitY : 0u) | (vz != v ? kBitZ : 0u);
    }
  }
  if (__any_sync(kFull, bad) && lane == 0) atomicOr(&hdr->status, kStBadLabel);
}

// K1, segment form (X % 128 == 0, 16-byte aligned rows; the default): one warp per x-row, and
// lane l owns the SEGMENT of 32 consecutive elements [32 s, 32 s + 32), s = 32 b + l, of each
// 1024-element block b.  The warp-wide sweeps of k_edt_x above spend a shuffle, a ballot and a
// bit scan on every 32 elements in each direction; here the per-element work is lane-local
// straight-line code on two 32-bit masks:
//   A. coalesced 16-byte label loads, transposed through shared memory (XOR-swizzled 16-byte
//      granules, conflict-free both ways); each lane builds the boundary mask B (bit j: a site
//      lies just left of element j, i.e. label(j) != label(j-1), or j = 0 with the border flag)
//      and the foreground mask F of its segment;
//   B. per segment, the nearest boundary before it (prefix max) and after it (suffix min; the
//      virtual boundary X with the border flag), as warp scans over the segments;
//   C. per element: s = last boundary <= x, e = first boundary > x, g = min(x - s + 1, e - x)^2
//      (kInf when neither exists), by one forward and one backward pass over the mask with
//      constant bit positions; the values go back through shared memory to coalesced 16-byte
//      stores, where the y/z run-start flags are formed from coalesced loads of the rows below.
// Same output word as k_edt_x, bit for bit.
constexpr int kSegFar = 1 << 20;  // "no boundary on this side" (|distance| stays far above 32768)
__device__ __forceinline__ int swz(int G) { return G ^ ((G >> 3) & 7); }  // 16-byte granule swizzle

#ifndef FASTRS_K1_MINB
#define FASTRS_K1_MINB 5
#endif
#ifndef FASTRS_K1_CPASYNC
#define FASTRS_K1_CPASYNC 1
#endif
constexpr bool kK1CpAsync = FASTRS_K1_CPASYNC != 0;
__global__ void __launch_bounds__(256, FASTRS_K1_MINB) k_edt_x_seg(const int32_t* __restrict__ lab,
                                                   const int32_t* __restrict__ below, const int32_t* __restrict__ sent,
                                                   uint32_t* __restrict__ out, int64_t nrows, int X, int64_t Y,
                                                   int64_t Z, int32_t max_label, int border, int is3d,
                                                   WsHeader* __restrict__ hdr, FastDiv fY, FastDiv fZ) {
  extern __shared__ __align__(16) uint32_t s_seg[];
  const int warps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * warps + warp;
  if (row >= nrows) return;
  const int NS = X >> 5;  // segments of the row (a multiple of 4)
  uint32_t* buf = s_seg + (size_t)warp * (1024 + 4 * NS);  // transpose buffer: 256 granules
  int4* buf4 = reinterpret_cast<int4*>(buf);
  uint32_t* sB = buf + 1024;
  uint32_t* sF = sB + NS;
  int* sP = reinterpret_cast<int*>(sF + NS);
  int* sN = sP + NS;
  int64_t y, z;
  if (nrows < (1ll << 32)) {  // 32-bit split (multiply-high) instead of 64-bit divisions
    uint32_t yr;
    const uint32_t q = fY.divmod((uint32_t)row, yr);
    y = yr;
    z = q - fZ.div(q) * fZ.d;
  } else {
    y = row % Y;
    z = (row / Y) % Z;
  }
  const int32_t* L = lab + row * X;
  const int32_t* Ly = y > 0 ? L - X : sent;
  const int32_t* Lz = is3d ? (z > 0 ? L - X * Y : (below ? below + y * X : sent)) : sent;
  uint32_t* O = out + row * X;
  const int nblk = (X + 1023) >> 10;
  uint32_t bad = 0;

  // ---- A: boundary and foreground masks per segment ----------------------------------------
  int32_t carry = 0;  // the last label of the previous block
  for (int blk = 0; blk < nblk; ++blk) {
    const int e0 = blk << 10;
    const int ng = min(1024, X - e0) >> 2;  // granules in this block (a multiple of 32)
    const int4* src = reinterpret_cast<const int4*>(L + e0);
    if (kK1CpAsync) {  // round 2c: every granule of the block in flight at once (no register hop)
      for (int G = lane; G < ng; G += 32) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(buf4 + swz(G));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src + G) : "memory");
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    } else {
      for (int G = lane; G < ng; G += 32) buf4[swz(G)] = __ldg(src + G);
    }
    __syncwarp();
    const int seg = (blk << 5) + lane;
    int32_t pv = lane > 0 ? (int32_t)buf[swz(lane * 8 - 1) * 4 + 3] : carry;
    if (seg < NS) {
      uint32_t Bm = 0, Fm = 0;
      if (lane == 0 && blk == 0) pv = buf4[swz(0)].x;  // element 0: a boundary only with the border flag
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int4 w = buf4[swz(lane * 8 + j)];
        Bm |= (w.x != pv ? 1u : 0u) << (4 * j);
        Bm |= (w.y != w.x ? 1u : 0u) << (4 * j + 1);
        Bm |= (w.z != w.y ? 1u : 0u) << (4 * j + 2);
        Bm |= (w.w != w.z ? 1u : 0u) << (4 * j + 3);
        Fm |= (w.x != 0 ? 1u : 0u) << (4 * j);
        Fm |= (w.y != 0 ? 1u : 0u) << (4 * j + 1);
        Fm |= (w.z != 0 ? 1u : 0u) << (4 * j + 2);
        Fm |= (w.w != 0 ? 1u : 0u) << (4 * j + 3);
        bad |= ((uint32_t)w.x > (uint32_t)max_label) | ((uint32_t)w.y > (uint32_t)max_label) |
               ((uint32_t)w.z > (uint32_t)max_label) | ((uint32_t)w.w > (uint32_t)max_label);  // also v < 0
        pv = w.w;
      }
      if (seg == 0 && border) Bm |= 1u;
      sB[seg] = Bm;
      sF[seg] = Fm;
    }
    carry = __shfl_sync(kFull, pv, 31);
    __syncwarp();
  }

  // ---- B: nearest boundary before / after each segment ---------------------------------------
  {
    int run = -kSegFar;  // prefix max of the boundaries of the segments before
    for (int s0 = 0; s0 < NS; s0 += 32) {
      const int s = s0 + lane;
      const uint32_t Bm = s < NS ? sB[s] : 0u;
      const int last = Bm ? 32 * s + 31 - __clz(Bm) : -kSegFar;
      int inc = last;  // prefix max over lanes <= lane
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc = max(inc, v);
      }
      int exc = __shfl_up_sync(kFull, inc, 1);
      if (lane == 0) exc = -kSegFar;
      if (s < NS) sP[s] = max(run, exc);
      run = max(run, __shfl_sync(kFull, inc, 31));
    }
    run = border ? X : kSegFar;  // suffix min of the boundaries of the segments after
    for (int s0 = ((NS - 1) >> 5) << 5; s0 >= 0; s0 -= 32) {
      const int s = s0 + lane;
      const uint32_t Bm = s < NS ? sB[s] : 0u;
      const int first = Bm ? 32 * s + __ffs(Bm) - 1 : kSegFar;
      int inc = first;  // suffix min over lanes >= lane
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_down_sync(kFull, inc, o);
        if (lane + o < 32) inc = min(inc, v);
      }
      int exc = __shfl_down_sync(kFull, inc, 1);
      if (lane == 31) exc = kSegFar;
      if (s < NS) sN[s] = min(run, exc);
      run = min(run, __shfl_sync(kFull, inc, 0));
    }
  }
  __syncwarp();

  // ---- C: distances per segment, then coalesced stores with the y/z run-start flags ----------
  for (int blk = 0; blk < nblk; ++blk) {
    const int e0 = blk << 10;
    const int ng = min(1024, X - e0) >> 2;
    const int seg = (blk << 5) + lane;
    if (seg < NS) {
      const uint32_t Bm = sB[seg], Fm = sF[seg];
      const int base = 32 * seg;
      uint32_t gv[32];
      int s = sP[seg] - base;  // relative position of the last boundary so far
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if ((Bm >> j) & 1u) s = j;
        gv[j] = (uint32_t)(j + 1 - s);  // x - s + 1
      }
      int e = sN[seg] - base;  // relative position of the next boundary
#pragma unroll
      for (int j = 31; j >= 0; --j) {
        if (j < 31 && ((Bm >> (j + 1)) & 1u)) e = j + 1;
        const uint32_t d = min(min(gv[j], (uint32_t)(e - j)), 32768u);
        gv[j] = ((Fm >> j) & 1u) ? min(d * d, kInf) : 0u;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        buf4[swz(lane * 8 + j)] = make_int4((int)gv[4 * j], (int)gv[4 * j + 1], (int)gv[4 * j + 2], (int)gv[4 * j + 3]);
    }
    __syncwarp();
    const int4* sl = reinterpret_cast<const int4*>(L + e0);
    const int4* sy = reinterpret_cast<const int4*>(Ly + e0);
    const int4* sz = reinterpret_cast<const int4*>(Lz + e0);
    uint4* dst = reinterpret_cast<uint4*>(O + e0);
    for (int G = lane; G < ng; G += 32) {
      const int4 gq = buf4[swz(G)];
      const int4 v = __ldg(sl + G), vy = __ldg(sy + G), vz = __ldg(sz + G);
      uint4 r;
      r.x = (uint32_t)gq.x | (vy.x != v.x ? kBitY : 0u) | (vz.x != v.x ? kBitZ : 0u);
      r.y = (uint32_t)gq.y | (vy.y != v.y ? kBitY : 0u) | (vz.y != v.y ? kBitZ : 0u);
      r.z = (uint32_t)gq.z | (vy.z != v.z ? kBitY : 0u) | (vz.z != v.z ? kBitZ : 0u);
      r.w = (uint32_t)gq.w | (vy.w != v.w ? kBitY : 0u) | (vz.w != v.w ? kBitZ : 0u);
      dst[G] = r;
    }
    __syncwarp();
  }
  if (__any_sync(kFull, bad) && lane == 0) atomicOr(&hdr->status, kStBadLabel);
}

constexpr int kColS = 256;  // positions per CTA
constexpr int kColH = 48;   // staged halo on each side
constexpr int kColRows = kColS + 2 * kColH;
constexpr int kColWarps = 8;
#ifndef FASTRS_SCAN_U
#define FASTRS_SCAN_U 4
#endif
constexpr int kScan16U = FASTRS_SCAN_U;  // row pairs per iteration of the 16-bit two-sided scan loop
#ifndef FASTRS_COL_PP
#define FASTRS_COL_PP 4
#endif
// positions per thread of the 16-bit column scan (1, 2 or 4).  C4 (round 2b): PP 2 4.41 / 4.24 ms
// (y / z), PP 4 4.12 / 4.08 (U = 2: 4.19 / 4.15; 4 CTAs/SM: 4.66 / 4.62)
constexpr int kColPP = FASTRS_COL_PP;
#ifndef FASTRS_COL_CPASYNC
#define FASTRS_COL_CPASYNC 1
#endif
constexpr bool kColCpAsync = FASTRS_COL_CPASYNC != 0;  // K2/K3 staging by cp.async (round 2c)
#ifndef FASTRS_COL_PREFETCH_L2
#define FASTRS_COL_PREFETCH_L2 0
#endif
constexpr int kColPrefetch = FASTRS_COL_PREFETCH_L2;  // L2 prefetch distance in CTAs per SM (0: off; 5 measured 2.83 / 3.07 vs 2.75 / 2.66 ms)

// Slow path of the column scan for an element whose window leaves the staged rows: the same
// exact scan in 32-bit arithmetic, every read from global memory (L2).  Round 2c: the reads of
// kSgBatch consecutive rows are issued together and then consumed in order (loads past the
// stopping row are speculative and in bounds), so a scan of n rows waits ~n / kSgBatch L2 round
// trips instead of n (ncu r02f: 43 % of K2/K3 stall samples were this loop's dependent loads).
#ifndef FASTRS_SG_BATCH
#define FASTRS_SG_BATCH 8
#endif
constexpr int kSgBatchList = FASTRS_SG_BATCH;
template <int kSgBatch>
__device__ __forceinline__ uint32_t scan_global_rows(const uint32_t* __restrict__ at, int64_t astride, int32_t n_up,
                                                  int32_t n_dn, uint32_t v, uint32_t chbit, bool up_end_site,
                                                  bool dn_end_site) {
  // at = the element's word; n_up / n_dn = staged rows above / below it; up_end_site: the row
  // just past the top of the staged axis is a site (the grid end with the border flag);
  // dn_end_site: likewise below row 0 (more grid before the slab, or the border flag)
  uint32_t best = v & kMask;
  {  // upwards: row p + d; a word with its run-start bit is a site at d
    int32_t d = 1;
    const uint32_t* q = at + astride;
    bool done = false;
    while (!done && (uint32_t)(d * d) < best) {
      uint32_t w[kSgBatch];
#pragma unroll
      for (int k = 0; k < kSgBatch; ++k) w[k] = (d + k <= n_up) ? __ldg(q + k * astride) : 0u;
#pragma unroll
      for (int k = 0; k < kSgBatch; ++k) {
        const uint32_t d2 = (uint32_t)((d + k) * (d + k));
        if (d2 >= best) { done = true; break; }
        if (d + k > n_up) {  // end of the staged axis (slab path: h^2 >= D guarantees the grid end)
          if (up_end_site) best = min(best, d2);
          done = true;
          break;
        }
        if (w[k] & chbit) { best = min(best, d2); done = true; break; }
        best = min(best, (w[k] & kMask) + d2);
      }
      d += kSgBatch;
      q += kSgBatch * astride;
    }
  }
  {  // downwards: row p - d; the row above it starting its run puts a site at d
    int32_t d = 1;
    uint32_t chk = v & chbit;
    const uint32_t* q = at - astride;
    bool done = false;
    while (!done && (uint32_t)(d * d) < best) {
      uint32_t w[kSgBatch];
#pragma unroll
      for (int k = 0; k < kSgBatch; ++k) w[k] = (d + k <= n_dn) ? __ldg(q - k * astride) : chbit;
#pragma unroll
      for (int k = 0; k < kSgBatch; ++k) {
        const uint32_t d2 = (uint32_t)((d + k) * (d + k));
        if (d2 >= best) { done = true; break; }
        if (chk) {
          if (d + k <= n_dn || dn_end_site) best = min(best, d2);
          done = true;
          break;
        }
        best = min(best, (w[k] & kMask) + d2);
        chk = w[k] & chbit;
      }
      d += kSgBatch;
      q -= kSgBatch * astride;
    }
  }
  return best;
}

__device__ __noinline__ uint32_t scan_global(const uint32_t* __restrict__ in, int64_t base, int64_t astride, int64_t p,
                                             int64_t L, uint32_t v, uint32_t chbit, int border, int64_t gofs,
                                             int64_t Lg) {
  return scan_global_rows<1>(in + base + p * astride, astride, (int32_t)(L - 1 - p), (int32_t)p, v, chbit,
                          border && gofs + L >= Lg, gofs > 0 || border);
}

struct ColArgs {
  const uint32_t* in;
  uint32_t* out;
  int64_t L, astride;
  int X, nxb, nseg;
  int64_t n_inner, inner_mult, outer_mult;
  uint32_t chbit;
  int border;
  int64_t p_lo, p_hi, gofs, Lg;
  FastDiv f_nxb, f_nseg, f_ninner;  // the CTA index split (block indices are 32-bit)
  int defer;  // 16-bit kernel: a scan that leaves the staged window lists its CTA for the envelope pass
  // 16-bit kernel (round 2c): an element whose scan leaves the staged window (and is not deferred to
  // the envelope pass) is appended here as (base << 24 | p) instead of scanned in line; the list
  // kernel scans it with batched L2 reads.  Null (or a full list): the in-line 32-bit scan.
  unsigned long long* slow;
  uint32_t slow_cap;
  int pf_ahead;  // 16-bit kernel: L2 prefetch of CTA blockIdx + pf_ahead's rows (0: off)
};

// ---- exact 32-bit column pass (one CTA = 256 positions x 32 columns) --------------------
// The CTA stages a [256 + 2*48] x 32 column tile of packed words and each thread runs the
// exact windowed scan  best = min(best, g(p +- dq) + dq^2)  until dq^2 >= best or a run end
// (a site at distance dq); reads outside the staged window go to global (L2).  Runs for the
// CTAs listed by the 16-bit kernel below (saturated values), or for every CTA when listed
// is NULL.
template <bool FINAL>
__device__ __forceinline__ void col32_body(const ColArgs& a, int64_t bid, uint32_t* tile, WsHeader* __restrict__ hdr) {
  const uint32_t* __restrict__ in = a.in;
  const int64_t L = a.L, astride = a.astride;
  const uint32_t chbit = a.chbit;
  const int border = a.border;
  uint32_t bq = (uint32_t)bid, xbr, segr, inr;
  bq = a.f_nxb.divmod(bq, xbr);
  const int xb = (int)xbr;
  bq = a.f_nseg.divmod(bq, segr);
  const int seg = (int)segr;
  const uint32_t outer = bq;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t oq = a.f_ninner.divmod(outer, inr);
  const int64_t base = (int64_t)oq * a.outer_mult + (int64_t)inr * a.inner_mult + (int64_t)xb * 32 + lane;
  const bool xin = xb * 32 + lane < a.X;
  const int64_t s0 = a.p_lo + (int64_t)seg * kColS;
  const int64_t lo = s0 - kColH > 0 ? s0 - kColH : 0;
  const int64_t hi = s0 + kColS + kColH < L ? s0 + kColS + kColH : L;
  for (int64_t r = lo + warp; r < hi; r += kColWarps)
    tile[(r - lo) * 32 + lane] = xin ? __ldg(in + base + r * astride) : 0u;
  __syncthreads();

  uint32_t dmax = 0, nfg = 0, nosite = 0;
  const int64_t pend = s0 + kColS < a.p_hi ? s0 + kColS : a.p_hi;
  for (int64_t p = s0 + warp; p < pend; p += kColWarps) {
    const uint32_t v = tile[(p - lo) * 32 + lane];
    const uint32_t g = v & kMask;
    uint32_t res = FINAL ? 0u : v;
    if (xin && g != 0) {
      uint32_t best = g;
      const int i = (int)(p - lo), nt = (int)(hi - lo);
      bool slow = false;
      {  // up side: rows p+1, p+2, ... until a run end (a site) or dq^2 >= best
        uint32_t dq2 = 1, inc = 3;
        const uint32_t* w_ptr = tile + (i + 1) * 32 + lane;
        const uint32_t* w_end = tile + nt * 32 + lane;
        while (dq2 < best) {
          if (w_ptr >= w_end) {
            if (hi < L) slow = true;  // more rows exist beyond the staged window
            else if (border && a.gofs + L >= a.Lg) best = min(best, dq2);  // the grid end
            break;
          }
          const uint32_t w = *w_ptr;
          if (w & chbit) {
            best = min(best, dq2);
            break;
          }
          best = min(best, (w & kMask) + dq2);
          dq2 += inc;
          inc += 2;
          w_ptr += 32;
        }
      }
      {  // down side: element p-dq lies outside the run iff p-dq+1 starts it
        uint32_t dq2 = 1, inc = 3, chk = v & chbit;
        int r = i - 1;
        while (dq2 < best) {
          if (chk) {
            if (a.gofs + lo + r >= 0 || border) best = min(best, dq2);
            break;
          }
          if (r < 0) {  // lo > 0 here (element 0 of the axis always starts a run)
            slow = true;
            break;
          }
          const uint32_t w = tile[r * 32 + lane];
          best = min(best, (w & kMask) + dq2);
          chk = w & chbit;
          dq2 += inc;
          inc += 2;
          --r;
        }
      }
      if (slow) best = scan_global(in, base, astride, p, L, v, chbit, border, a.gofs, a.Lg);
      dmax = max(dmax, best);
      if (FINAL) {
        res = best;
        nfg += 1;
        nosite |= best >= kInf;
      } else {
        res = best | (v & (kBitY | kBitZ));
      }
    }
    if (xin) a.out[base + (p - a.p_lo) * astride] = res;
  }
  if (!FINAL) {  // the max partial distance bounds the next pass's window (slab z halo)
    dmax = __reduce_max_sync(kFull, dmax);
    if (lane == 0 && dmax) atomicMax(&hdr->dxymax, dmax);
  } else {
    dmax = __reduce_max_sync(kFull, dmax);
    nfg = __reduce_add_sync(kFull, nfg);
    nosite = __any_sync(kFull, nosite);
    if (lane == 0) {
      if (dmax) atomicMax(&hdr->dmax, dmax);
      if (nfg) atomicAdd(&hdr->n_fg, (unsigned long long)nfg);
      if (nosite) atomicOr(&hdr->status, kStNoSite);
    }
  }
}

template <bool FINAL>
__global__ void __launch_bounds__(256) k_edt_col(ColArgs a, const uint32_t* __restrict__ listed,
                                                 WsHeader* __restrict__ hdr) {
  __shared__ __align__(16) uint32_t tile[kColRows * 32];
  if (!listed) {
    col32_body<FINAL>(a, blockIdx.x, tile, hdr);
    return;
  }
  const uint32_t n = *(volatile uint32_t*)&hdr->sat_n;
  for (uint32_t k = blockIdx.x; k < n; k += gridDim.x) {
    col32_body<FINAL>(a, listed[k], tile, hdr);
    __syncthreads();  // the tile is restaged for the next listed CTA
  }
}

// ---- exact lower-envelope column pass for the CTAs the 16-bit kernel lists ----------------
// The windowed scan costs O(sqrt(D)) per element, which is unbounded for large objects (a sphere
// of radius 240 takes 0.35 s per 512^3 pass).  The CTAs the 16-bit kernel cannot finish (a value
// >= 2^14-1 or a window beyond the staged rows) are recomputed here by the lower envelope of the
// parabolas (x - q)^2 + g(q) (Felzenszwalb-Huttenlocher), O(1) amortised per element:
//  * one warp per listed CTA, lane = column (32 columns of the CTA), sequential along the axis;
//  * only positions within R = isqrt(max g over the CTA's positions) + 1 of [s0, pend) can hold
//    an argmin (the minimum is <= g(p) <= R^2), so each lane walks [s0 - R, pend - 1 + R];
//  * the envelope is built per same-label run, with the run-end sites as parabolas of height 0
//    (the element before a run start / after a run end; the virtual border layer with the flag);
//  * intersections are compared exactly as fractions in 64-bit integers;
//  * the per-lane stack lives in global scratch (the K5 candidate pool, idle during the EDT):
//    entry k of a lane at scratch[slot][k][lane] (coalesced when the lanes are in step).
// Same results as the windowed scan, bit for bit (the minimum of integers is unique).
__device__ __forceinline__ bool fh_le(const uint2 a, const uint2 b, const uint2 c) {
  // isect(b, c) <= isect(a, b) for positions a < b < c; isect(i, j) = ((g_j + j^2) - (g_i + i^2)) / (2 (j - i))
  const long long ia = (int)a.x, ib = (int)b.x, ic = (int)c.x;
  const long long nab = ((long long)b.y + ib * ib) - ((long long)a.y + ia * ia), dab = 2 * (ib - ia);
  const long long nbc = ((long long)c.y + ic * ic) - ((long long)b.y + ib * ib), dbc = 2 * (ic - ib);
  return nbc * dab <= nab * dbc;
}

template <bool FINAL>
__global__ void __launch_bounds__(256) k_edt_col_fh(ColArgs a, const uint32_t* __restrict__ listed,
                                                    WsHeader* __restrict__ hdr, uint2* __restrict__ scratch,
                                                    int nslots) {
  const int lane = threadIdx.x & 31;
  const int slot = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  if (slot >= nslots) return;
  const uint32_t n = *(volatile uint32_t*)&hdr->sat_n;
  const int64_t L = a.L, astride = a.astride;
  const uint32_t chbit = a.chbit;
  uint2* env = scratch + (size_t)slot * 32 * (size_t)(L + 2) + lane;
  for (uint32_t t = slot; t < n; t += nslots) {
    uint32_t bq = listed[t], xbr, segr, inr;
    bq = a.f_nxb.divmod(bq, xbr);
    bq = a.f_nseg.divmod(bq, segr);
    const uint32_t oq = a.f_ninner.divmod(bq, inr);
    const int64_t base = (int64_t)oq * a.outer_mult + (int64_t)inr * a.inner_mult + (int64_t)xbr * 32 + lane;
    const bool xin = (int)xbr * 32 + lane < a.X;
    const int64_t s0 = a.p_lo + (int64_t)segr * kColS;
    const int64_t pend = s0 + kColS < a.p_hi ? s0 + kColS : a.p_hi;
    uint32_t dmax = 0, nfg = 0, nosite = 0;
    if (xin) {
      const uint32_t* col = a.in + base;
      auto word = [&](int64_t q) { return __ldg(col + q * astride); };
      uint32_t mg = 0;
      for (int64_t p = s0; p < pend; ++p) mg = max(mg, word(p) & kMask);
      int64_t R = L;
      if (mg < kInf) {
        R = (int64_t)sqrtf((float)mg);
        while (R * R > (int64_t)mg) --R;
        while ((R + 1) * (R + 1) <= (int64_t)mg) ++R;
        R += 1;
      }
      const int64_t lo = s0 - R > 0 ? s0 - R : 0, hi = pend - 1 + R < L - 1 ? pend - 1 + R : L - 1;
      int64_t q = lo;
      while (q < pend) {
        // the run [ra, rb] of the walked range that starts at q
        const int64_t ra = q;
        uint32_t w = word(q);
        const bool true_start = q == 0 || (w & chbit) != 0u;
        int ne = 0;
        auto push = [&](int pos, uint32_t gq) {
          const uint2 c = make_uint2((uint32_t)pos, gq);
          while (ne >= 2 && fh_le(env[(size_t)(ne - 2) * 32], env[(size_t)(ne - 1) * 32], c)) --ne;
          env[(size_t)ne * 32] = c;
          ++ne;
        };
        if (true_start && (a.gofs + ra - 1 >= 0 || a.border)) push((int)(ra - 1), 0u);
        for (;;) {
          const uint32_t gq = w & kMask;
          if (gq < kInf) push((int)q, gq);
          ++q;
          if (q > hi) break;
          w = word(q);
          if (w & chbit) break;  // q starts the next run
        }
        const int64_t rb = q - 1;
        const bool true_end = q <= hi || q >= L;  // (q > hi and q < L: the run continues past the walk)
        if (true_end && (rb + 1 < L || (a.border && a.gofs + L >= a.Lg))) push((int)(rb + 1), 0u);
        // evaluate the run's positions inside [s0, pend)
        const int64_t pa = ra > s0 ? ra : s0, pb = rb < pend - 1 ? rb : pend - 1;
        int k = 0;
        for (int64_t p = pa; p <= pb; ++p) {
          const uint32_t v = word(p);
          const uint32_t g = v & kMask;
          uint32_t res = FINAL ? 0u : v;
          if (g != 0) {
            uint32_t best = kInf;
            if (ne > 0) {
              uint2 ek = env[(size_t)k * 32];
              while (k + 1 < ne) {  // advance while the next parabola is at least as low at p
                const uint2 en = env[(size_t)(k + 1) * 32];
                const long long i0 = (int)ek.x, i1 = (int)en.x;
                const long long num = ((long long)en.y + i1 * i1) - ((long long)ek.y + i0 * i0), den = 2 * (i1 - i0);
                if (num > (long long)p * den) break;
                ek = en;
                ++k;
              }
              const long long d = p - (long long)(int)ek.x;
              const long long f = d * d + (long long)ek.y;
              best = f < (long long)kInf ? (uint32_t)f : kInf;
            }
            dmax = max(dmax, best);
            if (FINAL) {
              res = best;
              nfg += 1;
              nosite |= best >= kInf;
            } else {
              res = best | (v & (kBitY | kBitZ));
            }
          }
          a.out[base + (p - a.p_lo) * astride] = res;
        }
      }
    }
    dmax = __reduce_max_sync(kFull, dmax);
    if (!FINAL) {
      if (lane == 0 && dmax) atomicMax(&hdr->dxymax, dmax);
    } else {
      nfg = __reduce_add_sync(kFull, nfg);
      nosite = __any_sync(kFull, nosite);
      if (lane == 0) {
        if (dmax) atomicMax(&hdr->dmax, dmax);
        if (nfg) atomicAdd(&hdr->n_fg, (unsigned long long)nfg);
        if (nosite) atomicOr(&hdr->status, kStNoSite);
      }
    }
  }
}

// ---- 16-bit two-sided column pass (the default) -------------------------------------------
// Same exact windowed scan, restated so that one SIMD instruction advances both sides:
//  * a site met on the way is folded into the staged values: scanning up from p, element q is
//    outside p's run exactly when q starts a run, so up(q) = 0 there (a site at distance dq);
//    scanning down, q is outside when q+1 starts a run, so down(q) = 0 there.  Terms read past
//    a site are >= dq^2 > the site's own term, so they never change the minimum and the scan
//    needs no branch at run ends;
//  * values are clamped to kCap16 = 2^14 - 1 and each element's (up, down) pair is packed as
//    two u16 halves: one VIADDMNMX.U16x2 computes min(best, g(p+dq) + dq^2) and
//    min(best, g(p-dq) + dq^2) at once (dq^2 < kCap16 while scanning, so no half overflows);
//  * rows outside the axis are staged as virtual rows: 0 (a site) at the grid border with
//    FASTRS_BORDER_BACKGROUND, else kCap16 (no contribution).
// A result >= kCap16 (a clamped value or no site at all) cannot be trusted: the CTA lists
// itself and the exact 32-bit kernel above recomputes it (`sat_n` / `listed`).  Below kCap16
// the result is exact: the winning term involves an unclamped value (K2/K3).
constexpr uint32_t kCap16 = 16383u;
// a scan longer than this leaves its element to the envelope pass (its CTA is listed); shorter
// scans beyond the staged window read L2 per element (C4: a few elements of prolate grains;
// deferring them costs a whole-CTA envelope pass, edt_y 4.52 -> 5.34 ms)
constexpr int kDeferReach = 128;

// PP = 2 (the default): each thread scans two consecutive positions i, i+1 of its column at once.
// The halves of the SIMD pairs are the two positions: up pair (up(i+dq), up(i+1+dq)) and down
// pair (down(i-dq), down(i+1-dq)) are formed from two consecutive staged rows, of which one is
// new per dq and side, so a row load serves both positions: per dq and two elements 2 shared
// loads, 2 PRMT, 2 VIADDMNMX and the dq^2 step, against 2 loads, 1 PRMT, 1 VIADDMNMX and the step
// per element for PP = 1.  A background position enters with best = 0 and never extends the scan.
template <bool FINAL, int U, int PP>
// C4 sweep (round 2b): MINB 5 + prefetch: edt_y 4.41 / edt_z 4.24 ms; MINB 5 alone 4.53 / 4.52;
// MINB 4 (+ prefetch) 5.22 / 5.14 (4.81 / 4.72); no bound (62 registers) 4.56 / 4.50.  Five CTAs
// (45 KB of shared memory each) fill the SM's 228 KB.
#ifndef FASTRS_COL_MINB
#define FASTRS_COL_MINB 5
#endif
#ifndef FASTRS_COL_NO_PREFETCH
#define FASTRS_COL_PREFETCH
#endif
__global__ void __launch_bounds__(256, FASTRS_COL_MINB) k_edt_col16(ColArgs a, uint32_t* __restrict__ satlist,
                                                   WsHeader* __restrict__ hdr) {
  __shared__ __align__(16) uint32_t tile[kColRows * 32];
  const uint32_t* __restrict__ in = a.in;
  const int64_t L = a.L, astride = a.astride;
  const uint32_t chbit = a.chbit;
  int64_t bid = blockIdx.x;
  uint32_t bq = (uint32_t)bid, xbr, segr, inr;
  bq = a.f_nxb.divmod(bq, xbr);
  const int xb = (int)xbr;
  bq = a.f_nseg.divmod(bq, segr);
  const int seg = (int)segr;
  const uint32_t outer = bq;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t oq = a.f_ninner.divmod(outer, inr);
  const int64_t base = (int64_t)oq * a.outer_mult + (int64_t)inr * a.inner_mult + (int64_t)xb * 32 + lane;
  const bool xin = xb * 32 + lane < a.X;
  const int64_t s0 = a.p_lo + (int64_t)seg * kColS;
  const int64_t lo = s0 - kColH;  // staged rows [lo, lo + kColRows), virtual outside [0, L)
  auto word = [&](int64_t q) -> uint32_t { return (xin && q >= 0 && q < L) ? __ldg(in + base + q * astride) : 0u; };
  // virtual rows: above the axis only up-scans read them, below it only down-scans
  const uint32_t vup = (a.border && a.gofs + L >= a.Lg) ? 0u : kCap16;
  uint32_t vdn = kCap16;
  if (lo < 0) vdn = a.gofs == 0 ? (a.border ? 0u : kCap16) : ((word(0) & chbit) ? 0u : kCap16);
  constexpr int kPer = kColRows / kColWarps;
  if (kColPrefetch > 0 && a.pf_ahead > 0 && blockIdx.x + a.pf_ahead < gridDim.x) {
    // round 2c: warm L2 with the staged rows of the CTA launched ~one residency later (CTAs start
    // in index order): one 128-byte line per row, rows split over the threads
    uint32_t pq = blockIdx.x + (uint32_t)a.pf_ahead, pxr, psr, pir;
    pq = a.f_nxb.divmod(pq, pxr);
    pq = a.f_nseg.divmod(pq, psr);
    const uint32_t poq = a.f_ninner.divmod(pq, pir);
    const int64_t pbase = (int64_t)poq * a.outer_mult + (int64_t)pir * a.inner_mult + (int64_t)pxr * 32;
    const int64_t plo = a.p_lo + (int64_t)psr * kColS - kColH;
    for (int r = threadIdx.x; r < kColRows; r += kColWarps * 32) {
      const int64_t q = plo + r;
      if (q >= 0 && q < L) asm volatile("prefetch.global.L2 [%0];" ::"l"(in + pbase + q * astride));
    }
  }
  if (kColCpAsync && (a.X & 3) == 0 && (astride & 3) == 0 && xb * 32 + 32 <= a.X) {
    // staging (round 2c): the raw words of every in-axis row by cp.async, all 16-byte chunks in
    // flight at once (the per-warp load batches of the register path left 42 % of the stall
    // samples at the barrier after staging), then the (up, down) pairs in place, top down per warp
    // each warp copies its own 44 rows (lane: chunk lane & 7 of rows lane >> 3 + 4 i), so only
    // the warp waits for them; the raw word above the block comes straight from global
    static_assert(kPer % 4 == 0, "4 rows x 8 chunks per warp pass");
    const int rb = warp * kPer;  // this warp's rows [rb, rb + kPer) of the tile
    const int part = lane & 7, r4 = lane >> 3;
    const uint32_t* gp = in + (base - lane) + (lo + rb + r4) * astride + 4 * part;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(tile + (rb + r4) * 32 + 4 * part);
#pragma unroll
    for (int i = 0; i < kPer / 4; ++i) {
      const int64_t q = lo + rb + r4 + 4 * i;
      if (q >= 0 && q < L)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa + i * 4 * 32 * 4), "l"(gp + 4 * i * astride)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    uint32_t wn = word(lo + rb + kPer);
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncwarp();
    uint32_t* trow = tile + (rb + kPer - 1) * 32 + lane;
    if (lo + rb >= 0 && lo + rb + kPer <= L) {  // every row of the block inside the axis
#pragma unroll 11
      for (int k = kPer - 1; k >= 0; --k) {
        const uint32_t wq = *trow;
        const uint32_t gq = min(wq & kMask, kCap16);
        *trow = ((wq & chbit) ? 0u : gq) | (((wn & chbit) ? 0u : gq) << 16);
        trow -= 32;
        wn = wq;
      }
    } else {
      for (int k = kPer - 1; k >= 0; --k) {
        const int64_t q = lo + rb + k;
        uint32_t pr, wq = 0u;
        if (q < 0) pr = vdn | (vdn << 16);
        else if (q >= L) pr = vup | (vup << 16);
        else {
          wq = *trow;
          const uint32_t gq = min(wq & kMask, kCap16);
          pr = ((wq & chbit) ? 0u : gq) | (((wn & chbit) ? 0u : gq) << 16);
        }
        *trow = pr;
        trow -= 32;
        wn = wq;
      }
    }
  } else {  // staging: warp w transforms the contiguous rows [lo + 44w, lo + 44w + 44), top down
    const int64_t r0 = lo + (int64_t)warp * kPer;
    uint32_t* trow = tile + (r0 - lo + kPer - 1) * 32 + lane;
    if (xin && r0 >= 0 && r0 + kPer < L) {  // interior block (the common case): no bounds tests
      const uint32_t* src = in + base + (r0 + kPer) * astride;
      uint32_t wn = __ldg(src);
#pragma unroll 11
      for (int k = kPer - 1; k >= 0; --k) {
        src -= astride;
        const uint32_t wq = __ldg(src);
        const uint32_t gq = min(wq & kMask, kCap16);
        *trow = ((wq & chbit) ? 0u : gq) | (((wn & chbit) ? 0u : gq) << 16);
        trow -= 32;
        wn = wq;
      }
    } else {
      uint32_t wn = word(r0 + kPer);
      for (int k = kPer - 1; k >= 0; --k) {
        const int64_t q = r0 + k;
        const uint32_t wq = word(q);
        uint32_t pr;
        if (q < 0) pr = vdn | (vdn << 16);
        else if (q >= L) pr = vup | (vup << 16);
        else {
          const uint32_t gq = min(wq & kMask, kCap16);
          pr = ((wq & chbit) ? 0u : gq) | (((wn & chbit) ? 0u : gq) << 16);
        }
        *trow = pr;
        trow -= 32;
        wn = wq;
      }
    }
  }
  __syncthreads();

  uint32_t dmax = 0, nfg = 0, sat = 0;
  const int64_t pend = s0 + kColS < a.p_hi ? s0 + kColS : a.p_hi;
  // the raw word of p (its value and run flags) is loaded one iteration ahead; pointers step
  // by 8 rows (no 64-bit index arithmetic per element)
  const int np = (int)(pend - s0);
  const int64_t step = (int64_t)kColWarps * astride;
  const uint32_t* src = in + base + (s0 + warp) * astride;
  uint32_t* dst = a.out + base + (s0 + warp - a.p_lo) * astride;
  if constexpr (PP == 4) {
    // four consecutive positions i..i+3 per thread: SIMD pairs A = (i, i+1), B = (i+2, i+3) per
    // side; per dq one new staged row per side (sliding windows of four rows), 4 PRMT and 4
    // VIADDMNMX for four elements (PP = 2: 2 and 2 for two)
    const int64_t step4 = (int64_t)(4 * kColWarps) * astride;
    const uint32_t* src4 = in + base + (s0 + 4 * warp) * astride;
    uint32_t* dst4 = a.out + base + (s0 + 4 * warp - a.p_lo) * astride;
    // FB: a full CTA (256 positions, every lane inside the grid) drops the per-element bounds tests
    auto run4 = [&](auto fb) {
      constexpr bool FB = decltype(fb)::value;
      for (int j = 4 * warp; j < np; j += 4 * kColWarps) {
        uint32_t v[4], bst[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int m = 0; m < 4; ++m) v[m] = (FB || (xin && j + m < np)) ? __ldg(src4 + m * astride) : 0u;
        const uint32_t g0 = v[0] & kMask, g1 = v[1] & kMask, g2 = v[2] & kMask, g3 = v[3] & kMask;
        if ((g0 | g1 | g2 | g3) != 0) {
          const uint32_t gc0 = min(g0, kCap16), gc1 = min(g1, kCap16), gc2 = min(g2, kCap16), gc3 = min(g3, kCap16);
          const int i = kColH + j;
          const uint32_t gm = max(max(gc0, gc1), max(gc2, gc3));
          float r;
          asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"((float)gm));
          const int reach = (int)r + 1;
          if (reach + U - 1 <= min(i, kColRows - 4 - i)) {
            uint32_t buA = gc0 | (gc1 << 16), buB = gc2 | (gc3 << 16), bdA = buA, bdB = buB;
            uint32_t bmax2 = gm * 0x00010001u;
            uint32_t dq2p = 0x00010001u, incp = 0x00030003u;
            const uint32_t* t = tile + i * 32 + lane;  // row i
            uint32_t u0 = t[32], u1 = t[64], u2 = t[96];  // up window: rows i+dq .. i+2+dq (dq = 1)
            uint32_t d1 = t[0], d2 = t[32], d3 = t[64];   // down window: rows i+1-dq .. i+3-dq
            const uint32_t* up = t + 128;                  // row i+4 (= i+3+dq at dq = 1)
            const uint32_t* dn = t - 32;                   // row i-1 (= i-dq)
            while (dq2p < bmax2) {
#pragma unroll
              for (int uu = 0; uu < U; ++uu) {
                const uint32_t u3 = up[32 * uu];   // row i+3+dq
                const uint32_t d0 = dn[-32 * uu];  // row i-dq
                buA = __viaddmin_u16x2(__byte_perm(u0, u1, 0x5410), dq2p, buA);
                buB = __viaddmin_u16x2(__byte_perm(u2, u3, 0x5410), dq2p, buB);
                bdA = __viaddmin_u16x2(__byte_perm(d0, d1, 0x7632), dq2p, bdA);
                bdB = __viaddmin_u16x2(__byte_perm(d2, d3, 0x7632), dq2p, bdB);
                dq2p += incp;
                incp += 0x00020002u;
                u0 = u1, u1 = u2, u2 = u3;
                d3 = d2, d2 = d1, d1 = d0;
              }
              up += 32 * U;
              dn -= 32 * U;
              const uint32_t mA = __vminu2(buA, bdA), mB = __vminu2(buB, bdB), mm = __vmaxu2(mA, mB);
              bmax2 = __vmaxu2(mm, __byte_perm(mm, 0, 0x1032));
            }
            const uint32_t mA = __vminu2(buA, bdA), mB = __vminu2(buB, bdB);
            bst[0] = mA & 0xFFFFu, bst[1] = mA >> 16, bst[2] = mB & 0xFFFFu, bst[3] = mB >> 16;
          } else if (a.defer && reach > kDeferReach) {  // the exact envelope pass recomputes this CTA
            bst[0] = bst[1] = bst[2] = bst[3] = kCap16;
          } else if (a.slow) {  // exact, 32-bit, in the list kernel (placeholder 0 written here)
            const uint32_t nm = (uint32_t)((g0 != 0u) + (g1 != 0u) + (g2 != 0u) + (g3 != 0u));
            uint32_t at = atomicAdd(&hdr->slow_n, nm);
#pragma unroll
            for (int m = 0; m < 4; ++m)
              if (v[m] & kMask) {
                if (at < a.slow_cap) a.slow[at] = ((unsigned long long)base << 24) | (unsigned long long)(s0 + j + m);
                else bst[m] = scan_global(in, base, astride, s0 + j + m, L, v[m], chbit, a.border, a.gofs, a.Lg);
                ++at;
              }
          } else {  // exact, 32-bit
#pragma unroll
            for (int m = 0; m < 4; ++m)
              if (v[m] & kMask) bst[m] = scan_global(in, base, astride, s0 + j + m, L, v[m], chbit, a.border, a.gofs, a.Lg);
          }
        }
        // branch-free epilogue: a background element has best 0 and its word is just its run
        // flags, so best | flags is right for both; `sat` is derived from dmax after the loop
        if (FB || xin) {
#pragma unroll
          for (int m = 0; m < 4; ++m)
            if (FB || j + m < np) dst4[m * astride] = FINAL ? bst[m] : (bst[m] | (v[m] & (kBitY | kBitZ)));
        }
        dmax = max(dmax, max(max(bst[0], bst[1]), max(bst[2], bst[3])));
        if (FINAL) nfg += (uint32_t)((v[0] & kMask) != 0u) + (uint32_t)((v[1] & kMask) != 0u) +
                          (uint32_t)((v[2] & kMask) != 0u) + (uint32_t)((v[3] & kMask) != 0u);
        src4 += step4;
        dst4 += step4;
      }
    };
    if (np == kColS && (xb * 32 + 32 <= a.X)) run4(std::true_type{});
    else run4(std::false_type{});
    sat |= dmax >= kCap16;  // a clamped or deferred result (every result of this path is <= kCap16)
  } else if constexpr (PP == 2) {
    const int64_t step2 = (int64_t)(2 * kColWarps) * astride;
    const uint32_t* src2 = in + base + (s0 + 2 * warp) * astride;
    uint32_t* dst2 = a.out + base + (s0 + 2 * warp - a.p_lo) * astride;
    auto finish = [&](uint32_t v, uint32_t best) -> uint32_t {
      uint32_t res = FINAL ? 0u : v;
      if ((v & kMask) != 0) {
        sat |= best >= kCap16;
        dmax = max(dmax, best);
        if (FINAL) {
          res = best;
          nfg += 1;
        } else {
          res = best | (v & (kBitY | kBitZ));
        }
      }
      return res;
    };
#ifdef FASTRS_COL_PREFETCH
    uint32_t n0 = (xin && 2 * warp < np) ? __ldg(src2) : 0u;
    uint32_t n1 = (xin && 2 * warp + 1 < np) ? __ldg(src2 + astride) : 0u;
#endif
    for (int j = 2 * warp; j < np; j += 2 * kColWarps) {
      const bool has1 = j + 1 < np;
#ifdef FASTRS_COL_PREFETCH
      const uint32_t v0 = n0, v1 = n1;
      if (xin && j + 2 * kColWarps < np) n0 = __ldg(src2 + step2);
      if (xin && j + 2 * kColWarps + 1 < np) n1 = __ldg(src2 + step2 + astride);
#else
      const uint32_t v0 = xin ? __ldg(src2) : 0u;
      const uint32_t v1 = (xin && has1) ? __ldg(src2 + astride) : 0u;
#endif
      const uint32_t g0 = v0 & kMask, g1 = v1 & kMask;
      uint32_t best0 = 0, best1 = 0;
      if ((g0 | g1) != 0) {
        const uint32_t gc0 = min(g0, kCap16), gc1 = min(g1, kCap16);
        const int i = kColH + j;
        float r;
        asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"((float)max(gc0, gc1)));
        const int reach = (int)r + 1;
        if (reach + U - 1 <= min(i, kColRows - 2 - i)) {
          uint32_t bu = gc0 | (gc1 << 16), bd = bu;
          const uint32_t gm = max(gc0, gc1);
          uint32_t bmax2 = gm * 0x00010001u;
          uint32_t dq2p = 0x00010001u, incp = 0x00030003u;
          const uint32_t* t = tile + i * 32 + lane;  // row i
          uint32_t uprev = t[32], dprev = t[0];    // rows i+1 and i
          const uint32_t* up = t + 64;             // row i+2
          const uint32_t* dn = t - 32;             // row i-1
          while (dq2p < bmax2) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint32_t wu = up[32 * u];   // row i+1+dq
              const uint32_t wd = dn[-32 * u];  // row i-dq
              // (up(i+dq), up(i+1+dq)) and (down(i-dq), down(i+1-dq))
              bu = __viaddmin_u16x2(__byte_perm(uprev, wu, 0x5410), dq2p, bu);
              bd = __viaddmin_u16x2(__byte_perm(wd, dprev, 0x7632), dq2p, bd);
              dq2p += incp;
              incp += 0x00020002u;
              uprev = wu;
              dprev = wd;
            }
            up += 32 * U;
            dn -= 32 * U;
            const uint32_t m2 = __vminu2(bu, bd);
            bmax2 = __vmaxu2(m2, __byte_perm(m2, 0, 0x1032));
          }
          const uint32_t m2 = __vminu2(bu, bd);
          best0 = m2 & 0xFFFFu;
          best1 = m2 >> 16;
        } else {  // exact, 32-bit
          if (a.defer && reach > kDeferReach) {  // the exact envelope pass recomputes this CTA (O(1) per element)
            best0 = best1 = kCap16;
          } else {
            if (g0) best0 = scan_global(in, base, astride, s0 + j, L, v0, chbit, a.border, a.gofs, a.Lg);
            if (g1) best1 = scan_global(in, base, astride, s0 + j + 1, L, v1, chbit, a.border, a.gofs, a.Lg);
          }
        }
      }
      const uint32_t r0 = finish(v0, best0), r1 = finish(v1, best1);
      if (xin) {
        *dst2 = r0;
        if (has1) dst2[astride] = r1;
      }
      src2 += step2;
      dst2 += step2;
    }
  } else {
    const uint32_t* trow = tile + (kColH + warp) * 32 + lane;  // row p of the tile
    uint32_t v_next = (xin && warp < np) ? __ldg(src) : 0u;
    for (int j = warp; j < np; j += kColWarps) {
      const uint32_t v = v_next;
      src += step;
      if (xin && j + kColWarps < np) v_next = __ldg(src);
      const uint32_t g = v & kMask;
      uint32_t res = FINAL ? 0u : v;
      if (g != 0) {  // (lanes beyond X read 0)
        const uint32_t gc = min(g, kCap16);
        const int i = kColH + j;
        // dq^2 < best <= gc bounds the scan: isqrt(gc - 1) + U - 1 rows on each side suffice
        float r;
        asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"((float)gc));
        const int reach = (int)r + 1;
        uint32_t best;
        if (reach + U - 1 <= min(i, kColRows - 1 - i)) {
          // dq2p = (dq^2, dq^2) and bmin2 = (m, m), m = min of the two halves of best2: the u32
          // compare dq2p < bmin2 is dq^2 < m
          uint32_t best2 = gc * 0x00010001u, bmin2 = best2;
          uint32_t dq2p = 0x00010001u, incp = 0x00030003u;
          const uint32_t* up = trow + 32;
          const uint32_t* dn = trow - 32;
          while (dq2p < bmin2) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
              // low half: up(p + dq), high half: down(p - dq)
              const uint32_t pr = __byte_perm(up[32 * u], dn[-32 * u], 0x7610);
              best2 = __viaddmin_u16x2(pr, dq2p, best2);
              dq2p += incp;
              incp += 0x00020002u;
            }
            up += 32 * U;
            dn -= 32 * U;
            bmin2 = __vminu2(best2, __byte_perm(best2, 0, 0x1032));
          }
          best = bmin2 & 0xFFFFu;
        } else {
          best = (a.defer && reach > kDeferReach) ? kCap16
                                                  : scan_global(in, base, astride, s0 + j, L, v, chbit, a.border, a.gofs, a.Lg);
        }
        sat |= best >= kCap16;  // clamped, or no site at all (ENOSITE comes from the 32-bit kernel)
        dmax = max(dmax, best);
        if (FINAL) {
          res = best;
          nfg += 1;
        } else {
          res = best | (v & (kBitY | kBitZ));
        }
      }
      if (xin) *dst = res;
      dst += step;
      trow += 32 * kColWarps;
    }
  }
  // a CTA that saw a saturated value is recomputed by the 32-bit kernel (its statistics too)
  if (a.defer == 2) sat = 1;
  if (__syncthreads_or(sat)) {
    if (threadIdx.x == 0) satlist[atomicAdd(&hdr->sat_n, 1u)] = blockIdx.x;
    return;
  }
  dmax = __reduce_max_sync(kFull, dmax);
  if (!FINAL) {
    if (lane == 0 && dmax) atomicMax(&hdr->dxymax, dmax);
  } else {
    nfg = __reduce_add_sync(kFull, nfg);
    if (lane == 0) {
      if (dmax) atomicMax(&hdr->dmax, dmax);
      if (nfg) atomicAdd(&hdr->n_fg, (unsigned long long)nfg);
    }
  }
}

// the elements K2/K3 listed (their scans leave the staged window): one thread each, the exact
// 32-bit scan with kSgBatchList L2 reads in flight; max / n-site statistics as the CTA would
template <bool FINAL>
__global__ void __launch_bounds__(256) k_edt_col_slow(ColArgs a, const WsHeader* __restrict__ hdr_in,
                                                      WsHeader* __restrict__ hdr) {
  const uint32_t n = min(hdr_in->slow_n, a.slow_cap);
  uint32_t dmax = 0;
  bool nosite = false;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const unsigned long long e = a.slow[t];
    const int64_t base = (int64_t)(e >> 24), p = (int64_t)(e & 0xFFFFFFull);
    const uint32_t* at = a.in + base + p * a.astride;
    const uint32_t v = __ldg(at);
    const uint32_t best = scan_global_rows<kSgBatchList>(at, a.astride, (int32_t)(a.L - 1 - p), (int32_t)p, v, a.chbit,
                                                         a.border && a.gofs + a.L >= a.Lg, a.gofs > 0 || a.border);
    a.out[base + (p - a.p_lo) * a.astride] = FINAL ? best : (best | (v & (kBitY | kBitZ)));
    dmax = max(dmax, best);
    nosite |= best >= kInf;
  }
  dmax = __reduce_max_sync(kFull, dmax);
  nosite = __any_sync(kFull, nosite);
  if ((threadIdx.x & 31) == 0) {
    if (dmax) atomicMax(FINAL ? &hdr->dmax : &hdr->dxymax, dmax);
    if (FINAL && nosite) atomicOr(&hdr->status, kStNoSite);
  }
}

}  // namespace

// a per-device row of -1 labels (16384 entries): the y / z neighbour row of the first row / slice
std::mutex g_sent_mu;
int32_t* g_sent[64];

void launch_edt_x(const int32_t* labels, const int32_t* labels_below, uint32_t* out, const Geom& g,
                  int32_t max_label, bool border, WsHeader* hdr, cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(g_sent_mu);
    if (!g_sent[dev] && cudaMalloc(&g_sent[dev], 16384 * sizeof(int32_t)) == cudaSuccess)
      cudaMemset(g_sent[dev], 0xFF, 16384 * sizeof(int32_t));
  }
  const int64_t nrows = g.B * g.Z * g.Y;
  int warps = (int)(49152 / (2 * g.X));
  warps = warps < 1 ? 1 : (warps > 8 ? 8 : warps);
  const size_t smem = (size_t)warps * g.X * sizeof(uint16_t);
  const int64_t blocks = (nrows + warps - 1) / warps;
  const bool aligned = ((uintptr_t)labels % 16 == 0) && ((uintptr_t)out % 16 == 0) &&
                       (!labels_below || (uintptr_t)labels_below % 16 == 0);
  if (g.X % 128 == 0 && aligned && !getenv("FASTRS_K1_WARP")) {  // segment form (the default)
    const size_t per_warp = (size_t)(1024 + 4 * (g.X / 32)) * sizeof(uint32_t);
    int sw = (int)(49152 / per_warp);
    sw = sw < 1 ? 1 : (sw > 8 ? 8 : sw);
    const int64_t sblocks = (nrows + sw - 1) / sw;
    k_edt_x_seg<<<(unsigned)sblocks, sw * 32, sw * per_warp, st>>>(labels, labels_below, g_sent[dev], out, nrows,
                                                                   (int)g.X, g.Y, g.Z, max_label, border ? 1 : 0,
                                                                   g.ndim == 3 ? 1 : 0, hdr,
                                                                   FastDiv((uint32_t)g.Y), FastDiv((uint32_t)g.Z));
    return;
  }
  // sweep unroll 2: measured on C4 4.13 ms vs 4.46 (4), 4.35 (8), 4.26 (16) (round 1)
  if (g.X % 32 == 0)
    k_edt_x<2, true><<<(unsigned)blocks, warps * 32, smem, st>>>(labels, labels_below, g_sent[dev], out, nrows, (int)g.X,
                                                                 g.Y, g.Z, max_label, border ? 1 : 0,
                                                                 g.ndim == 3 ? 1 : 0, hdr);
  else
    k_edt_x<2, false><<<(unsigned)blocks, warps * 32, smem, st>>>(labels, labels_below, g_sent[dev], out, nrows,
                                                                  (int)g.X, g.Y, g.Z, max_label, border ? 1 : 0,
                                                                  g.ndim == 3 ? 1 : 0, hdr);
}

int64_t col_blocks(const Geom& g) {
  const int64_t nxb = (g.X + 31) / 32;
  const int64_t by = nxb * ((g.Y + kColS - 1) / kColS) * g.B * g.Z;
  const int64_t bz = g.ndim == 3 ? nxb * ((g.Z + kColS - 1) / kColS) * g.B * g.Y : 0;
  return by > bz ? by : bz;
}

// axis 1 = y, axis 2 = z.  16-bit kernel, then the exact 32-bit kernel over the CTAs it listed
// (satlist NULL: the 32-bit kernel everywhere).
void launch_edt_col(const uint32_t* in, uint32_t* out, const Geom& g, int axis, bool final_pass, bool border,
                    WsHeader* hdr, uint32_t* satlist, cudaStream_t st, int64_t p_lo, int64_t p_hi, int64_t gofs,
                    int64_t Lg, void* scratch, size_t scratch_bytes) {
  ColArgs a{};
  a.in = in;
  a.out = out;
  a.border = border ? 1 : 0;
  if (axis == 1) {
    a.L = g.Y;
    a.astride = g.X;
    a.n_inner = 1;
    a.inner_mult = 0;
    a.outer_mult = g.Y * g.X;
    a.chbit = kBitY;
  } else {
    a.L = g.Z;
    a.astride = g.Y * g.X;
    a.n_inner = g.Y;
    a.inner_mult = g.X;
    a.outer_mult = g.Z * g.Y * g.X;
    a.chbit = kBitZ;
  }
  const int64_t n_outer = axis == 1 ? g.B * g.Z : g.B * g.Y;
  if (p_hi < 0) p_hi = a.L;
  if (Lg < 0) Lg = a.L;
  a.p_lo = p_lo;
  a.p_hi = p_hi;
  a.gofs = gofs;
  a.Lg = Lg;
  a.X = (int)g.X;
  a.nxb = (int)((g.X + 31) / 32);
  a.nseg = (int)((p_hi - p_lo + kColS - 1) / kColS);
  if (a.nseg <= 0) return;
  a.f_nxb = FastDiv((uint32_t)a.nxb);
  a.f_nseg = FastDiv((uint32_t)a.nseg);
  a.f_ninner = FastDiv((uint32_t)a.n_inner);
  const int64_t blocks = (int64_t)a.nxb * a.nseg * n_outer;
  if (!satlist) {
    if (final_pass) k_edt_col<true><<<(unsigned)blocks, kColWarps * 32, 0, st>>>(a, nullptr, hdr);
    else k_edt_col<false><<<(unsigned)blocks, kColWarps * 32, 0, st>>>(a, nullptr, hdr);
    return;
  }
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaMemsetAsync(&hdr->sat_n, 0, sizeof(uint32_t), st);
  const unsigned fix_grid = (unsigned)(nsm * 2);
  // the envelope fix-up: one warp per listed CTA, a (L + 2)-entry stack per lane in the scratch
  const size_t per_slot = (size_t)32 * (size_t)(a.L + 2) * sizeof(uint2);
  int64_t nslots = scratch ? (int64_t)(scratch_bytes / per_slot) : 0;
  if (nslots > (int64_t)nsm * 16) nslots = (int64_t)nsm * 16;
  if (nslots > 0 && !getenv("FASTRS_COL_WINDOWED")) {
    a.defer = getenv("FASTRS_COL_FH_ALL") ? 2 : 1;  // 2 (test hook): every CTA takes the envelope pass
    // the slow-scan list lives at the start of the scratch; the list kernel consumes it before
    // the envelope pass reuses the scratch for its stacks.  FASTRS_COL_INLINE (test hook): none
    if (!getenv("FASTRS_COL_INLINE") && a.L < (1 << 24) && g.B * g.Z * g.Y * g.X < (1ll << 40)) {
      const size_t cap = scratch_bytes / sizeof(unsigned long long);
      a.slow = (unsigned long long*)scratch;
      a.slow_cap = (uint32_t)(cap < (size_t)(1u << 24) ? cap : (size_t)(1u << 24));
      if (const char* sc = getenv("FASTRS_COL_SLOW_CAP")) a.slow_cap = (uint32_t)atoi(sc);  // test hook
      cudaMemsetAsync(&hdr->slow_n, 0, sizeof(uint32_t), st);
    }
    const unsigned fh_grid = (unsigned)((nslots + 7) / 8);
    const unsigned slow_grid = (unsigned)(nsm * 4);
    a.pf_ahead = nsm * kColPrefetch;
    if (final_pass) {
      k_edt_col16<true, kScan16U, kColPP><<<(unsigned)blocks, kColWarps * 32, 0, st>>>(a, satlist, hdr);
      if (a.slow) k_edt_col_slow<true><<<slow_grid, 256, 0, st>>>(a, hdr, hdr);
      k_edt_col_fh<true><<<fh_grid, 256, 0, st>>>(a, satlist, hdr, (uint2*)scratch, (int)nslots);
    } else {
      k_edt_col16<false, kScan16U, kColPP><<<(unsigned)blocks, kColWarps * 32, 0, st>>>(a, satlist, hdr);
      if (a.slow) k_edt_col_slow<false><<<slow_grid, 256, 0, st>>>(a, hdr, hdr);
      k_edt_col_fh<false><<<fh_grid, 256, 0, st>>>(a, satlist, hdr, (uint2*)scratch, (int)nslots);
    }
    return;
  }
  if (final_pass) {
    k_edt_col16<true, kScan16U, kColPP><<<(unsigned)blocks, kColWarps * 32, 0, st>>>(a, satlist, hdr);
    k_edt_col<true><<<fix_grid, kColWarps * 32, 0, st>>>(a, satlist, hdr);
  } else {
    k_edt_col16<false, kScan16U, kColPP><<<(unsigned)blocks, kColWarps * 32, 0, st>>>(a, satlist, hdr);
    k_edt_col<false><<<fix_grid, kColWarps * 32, 0, st>>>(a, satlist, hdr);
  }
}

}  // namespace fastrs
