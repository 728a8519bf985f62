// K5 (default path): exact ball dilation LT^2(p) = max{ D(q) : |p-q|^2 < D(q) }
// by "sorted cover", fused with the shell test and the per-label reductions.
//
// Work organisation.  A CTA of 4 warps owns a group of 4 output tiles (3D: 1x2x2 tiles of
// 32x8x8, 2D: 2x2 tiles of 32x64; a tile = 64 rows of 32 elements); each warp owns one
// tile privately (values, coverage masks), so the hot loop has no atomics and no
// inter-warp conflicts, while the candidate gather is shared by the 4 tiles.
//   1. gather   : the CTA collects every kept maximal ball (K4 output) whose ball reaches
//                 the group's box into a shared list (8-byte packed centre + D) and a
//                 histogram of a monotone bucket of D (8 buckets per octave).  K4's lists
//                 are sorted by bucket, so a home tile is abandoned as soon as its remaining
//                 balls are too small to reach the group.
//   2. sort     : a counting sort of list indices by bucket, descending.
//   3. cover    : each warp walks the non-empty buckets from the largest D down.  A ball is
//                 tested against the bounding boxes of the still-uncovered foreground
//                 elements of its tile (8 regions) and skipped when it cannot reach any of
//                 them; else its rows are visited (lanes over the ball's rows): rows whose
//                 uncovered mask misses the ball's x-extent are skipped, the others get the
//                 interval |x-qx| <= isqrt(D-1-dy^2-dz^2), and only cells not covered by an
//                 EARLIER bucket are max-updated.  Cells covered by an earlier bucket hold a
//                 value >= every D of later buckets, so skipping them is exact; within a
//                 bucket updates are plain max, so the result does not depend on the order
//                 inside a bucket.
//   4. epilogue : LT^2 per element, shell (D == 1), per-label reductions (shared with the
//                 fallback kernel in lt.cu).
// Exactness never depends on a test being tight: every skip is justified by cells already
// holding a value >= D.  Gathers larger than the list are processed in D-descending rounds;
// the pathological case (one bucket alone larger than the list) hands the group to the
// atomic fallback kernel k_dilate_atomic (lt.cu), which also handles Dmax > 65535.
#include "common.cuh"
#include "dilate_common.cuh"

namespace fastrs {
namespace {

constexpr int kWarps = 4;  // warps per CTA = tiles per group
constexpr int kCap = 2048;
constexpr int kBuckets = 128;
constexpr int kRegions = 8;
constexpr int kOff = 16384;  // coordinate bias of packed candidates

// ceil(2^16 / n): (r * c_magic[n]) >> 16 == r / n exactly for r < 64
__constant__ uint32_t c_magic[65] = {
    0,    65536, 32768, 21846, 16384, 13108, 10923, 9363, 8192, 7282, 6554, 5958, 5462, 5042, 4682, 4370, 4096,
    3856, 3641,  3450,  3277,  3121,  2979,  2850,  2731, 2622, 2521, 2428, 2341, 2260, 2185, 2115, 2048, 1986,
    1928, 1873,  1821,  1772,  1725,  1681,  1639,  1599, 1561, 1525, 1490, 1457, 1425, 1395, 1366, 1338, 1311,
    1286, 1261,  1237,  1214,  1192,  1171,  1150,  1130, 1111, 1093, 1075, 1058, 1041, 1024};

struct Smem {
  unsigned long long list[kCap];     // gathered candidates (centre relative to the group), gather order
  uint16_t val[kWarps][kRows * 32];  // LT^2 per element of each warp's tile (D <= 65535 here)
  uint16_t idx[kCap];                // indices into list, sorted by D bucket (descending)
  uint32_t fg[kWarps][kRows];        // foreground mask per row
  uint32_t cov[kWarps][kRows];       // covered by an earlier bucket
  uint32_t cur[kWarps][kRows];       // covered in the current bucket
  int box[kWarps][kRegions][6];      // uncovered-foreground bounding boxes (x0,x1,y0,y1,z0,z1)
  uint32_t hist[kBuckets];
  uint32_t start[kBuckets + 1];
  uint32_t nonempty[4];              // non-empty buckets of the round (bitmask)
  uint32_t count;
  int round_lo, round_hi, next_hi, fallback;
};

template <bool IS3D>
struct Shape {
  static constexpr int TY = IS3D ? 8 : 64, TZ = IS3D ? 8 : 1;
  static constexpr int GX = IS3D ? 1 : 2, GY = 2, GZ = IS3D ? 2 : 1;  // tiles per group
  static constexpr int RX = GX * kTX, RY = GY * TY, RZ = GZ * TZ;     // group box
};

__device__ __forceinline__ unsigned long long pack(int x, int y, int z, uint32_t D) {
  return (unsigned long long)D | ((unsigned long long)(uint16_t)(x + kOff) << 16) |
         ((unsigned long long)(uint16_t)(y + kOff) << 32) | ((unsigned long long)(uint16_t)(z + kOff) << 48);
}

__device__ __forceinline__ int gap(int lo, int hi, int c) { return c < lo ? lo - c : (c > hi ? c - hi : 0); }

// floor(sqrt(h)) for 0 <= h < 2^16 via the hardware approximation (error << 1/512)
__device__ __forceinline__ int isqrt16(int h) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"((float)h));
  return (int)(r + 1e-3f);
}

__device__ __forceinline__ uint32_t range_mask(int l, int r) {  // bits l..r (0 <= l <= r <= 31)
  return (r == 31 ? 0xFFFFFFFFu : ((1u << (r + 1)) - 1u)) & (0xFFFFFFFFu << l);
}

// Gather the candidates reaching the group box with bucket in [blo, bhi] into S.list.
// HIST: also histogram them (the first pass of a round).
template <bool IS3D, bool HIST>
__device__ __forceinline__ void gather(Smem& S, const TileMeta* __restrict__ meta, const uint2* __restrict__ cent,
                                       const Geom& g, int64_t b, int64_t tx0, int64_t ty0, int64_t tz0, int nrx,
                                       int nry, int nrz, int blo, int bhi) {
  using P = Shape<IS3D>;
  const int tid = threadIdx.x, lane = tid & 31;
  const int nx = P::GX + 2 * nrx, ny = P::GY + 2 * nry, nz = P::GZ + 2 * nrz;
  const int nneigh = nx * ny * nz;
  for (int nb0 = 0; nb0 < nneigh; nb0 += kWarps * 32) {
    const int n = nb0 + tid;
    bool reach = false;
    int64_t ht = 0;
    uint32_t hcount = 0;
    int hox = 0, hoy = 0, hoz = 0, hg2 = 0;
    if (n < nneigh) {
      const int ix = n % nx, iy = (n / nx) % ny, iz = n / (nx * ny);
      const int64_t hx = tx0 + ix - nrx, hy = ty0 + iy - nry, hz = tz0 + iz - nrz;
      if (hx >= 0 && hx < g.ntx && hy >= 0 && hy < g.nty && hz >= 0 && hz < g.ntz) {
        ht = ((b * g.ntz + hz) * g.nty + hy) * g.ntx + hx;
        const TileMeta hm = meta[ht];
        hox = (ix - nrx) * kTX;
        hoy = (iy - nry) * P::TY;
        hoz = (iz - nrz) * P::TZ;
        // gap between the home tile box and the group box
        const int gx = hox < 0 ? -(hox + kTX - 1) : (hox > P::RX - 1 ? hox - (P::RX - 1) : 0);
        const int gy = hoy < 0 ? -(hoy + P::TY - 1) : (hoy > P::RY - 1 ? hoy - (P::RY - 1) : 0);
        const int gz = hoz < 0 ? -(hoz + P::TZ - 1) : (hoz > P::RZ - 1 ? hoz - (P::RZ - 1) : 0);
        hg2 = gx * gx + gy * gy + gz * gz;
        reach = hm.count && hg2 <= (int)hm.maxD - 1 && dbucket(hm.maxD) >= blo;
        hcount = hm.count;
      }
    }
    uint32_t rm = __ballot_sync(kFull, reach);
    while (rm) {
      const int j = __ffs(rm) - 1;
      rm &= rm - 1;
      const int64_t hts = __shfl_sync(kFull, ht, j);
      const uint32_t cnt = __shfl_sync(kFull, hcount, j);
      const int bx = __shfl_sync(kFull, hox, j), by = __shfl_sync(kFull, hoy, j), bz = __shfl_sync(kFull, hoz, j);
      const int g2 = __shfl_sync(kFull, hg2, j);
      const uint2* src = cent + (size_t)hts * kTileVol;
      // the home tile's list is sorted by D bucket, descending: stop once the remaining balls
      // are too small to reach the group, or below the round's bucket range
      for (uint32_t e0 = 0; e0 < cnt; e0 += 32) {
        bool take = false;
        int bk = -1;
        unsigned long long pe = 0;
        if (e0 + lane < cnt) {
          const uint2 e = __ldg(src + e0 + lane);
          const int v = (int)e.x;
          const int cx = bx + (v & 31), cy = by + ((v >> 5) % P::TY), cz = bz + v / (32 * P::TY);
          const int ddx = gap(0, P::RX - 1, cx), ddy = gap(0, P::RY - 1, cy), ddz = gap(0, P::RZ - 1, cz);
          bk = dbucket(e.y);
          if (ddx * ddx + ddy * ddy + ddz * ddz <= (int)e.y - 1) {
            take = bk >= blo && bk <= bhi;
            pe = pack(cx, cy, cz, e.y);
          }
        }
        const int last = (int)min(cnt - e0, 32u) - 1;
        const int bk_last = __shfl_sync(kFull, bk, last);
        const bool more = (int)dbucket_max(bk_last) - 1 >= g2 && bk_last >= blo;
        const uint32_t tm = __ballot_sync(kFull, take);
        if (tm) {
          if (HIST) {
            const uint32_t grp = __match_any_sync(kFull, take ? bk : -1);
            if (take && lane == __ffs(grp) - 1) atomicAdd(&S.hist[bk], (uint32_t)__popc(grp));
          }
          uint32_t base = 0;
          if (lane == 0) base = atomicAdd(&S.count, (uint32_t)__popc(tm));
          base = __shfl_sync(kFull, base, 0);
          const uint32_t pos = base + __popc(tm & ((1u << lane) - 1u));
          if (take && pos < kCap) S.list[pos] = pe;
        }
        if (!more) break;
      }
    }
  }
}

template <bool IS3D>
__global__ void __launch_bounds__(kWarps * 32) k_dilate_cover(const int32_t* __restrict__ lab,
                                                             const uint32_t* __restrict__ Dg,
                                                             TileMeta* __restrict__ meta,
                                                             const uint2* __restrict__ cent, Geom g, Accum acc,
                                                             int do_reduce, uint32_t* __restrict__ lt2_out,
                                                             float* __restrict__ lt_out, WsHeader* __restrict__ hdr) {
  using P = Shape<IS3D>;
  constexpr int TY = P::TY, TZ = P::TZ;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t dmax = hdr->dmax;
  if (dmax > kU16Max) return;  // k_dilate_atomic handles it

  // ---- group / tile coordinates --------------------------------------------------------
  const int64_t ngx = (g.ntx + P::GX - 1) / P::GX, ngy = (g.nty + P::GY - 1) / P::GY, ngz = (g.ntz + P::GZ - 1) / P::GZ;
  int64_t t = blockIdx.x;
  const int64_t gxi = t % ngx;
  t /= ngx;
  const int64_t gyi = t % ngy;
  t /= ngy;
  const int64_t gzi = t % ngz;
  const int64_t b = t / ngz;
  const int64_t tx0 = gxi * P::GX, ty0 = gyi * P::GY, tz0 = gzi * P::GZ;
  const int64_t rox = tx0 * kTX, roy = ty0 * TY, roz = tz0 * TZ;  // group origin
  const int wx = warp % P::GX, wy = (warp / P::GX) % P::GY, wz = warp / (P::GX * P::GY);
  const int64_t mtx = tx0 + wx, mty = ty0 + wy, mtz = tz0 + wz;
  const bool have_tile = mtx < g.ntx && mty < g.nty && mtz < g.ntz;
  const int64_t mtile = have_tile ? ((b * g.ntz + mtz) * g.nty + mty) * g.ntx + mtx : 0;
  const int mox = wx * kTX, moy = wy * TY, moz = wz * TZ;  // my tile origin within the group
  const bool active = have_tile && meta[mtile].nfg != 0;
  if (__syncthreads_or(active) == 0) return;  // the whole group is background
  const int64_t item = b * g.Z * g.Y * g.X;

  // ---- per-warp init: values, foreground masks, coverage ----------------------------------
  uint16_t* val = S.val[warp];
  uint32_t* fgw = S.fg[warp];
  uint32_t* covw = S.cov[warp];
  uint32_t* curw = S.cur[warp];
  for (int i = lane; i < kRows * 32 / 2; i += 32) reinterpret_cast<uint32_t*>(val)[i] = 0;
#pragma unroll 4
  for (int row = 0; row < kRows; ++row) {
    const int ly = row % TY, lz = row / TY;
    const int64_t gz = roz + moz + lz, gy = roy + moy + ly, gx = rox + mox + lane;
    bool f = false;
    if (active && gz < g.Z && gy < g.Y && gx < g.X) f = __ldg(Dg + item + (gz * g.Y + gy) * g.X + gx) != 0;
    const uint32_t m = __ballot_sync(kFull, f);
    if (lane == 0) {
      fgw[row] = m;
      covw[row] = 0;
      curw[row] = 0;
    }
  }
  __syncwarp();

  // uncovered-foreground bounding boxes of the 8 regions of my tile (tile coordinates):
  // 3D: x halves x y halves x z halves; 2D: x halves x y quarters
  auto refresh_boxes = [&]() {
    int* bxs = &S.box[warp][0][0];
    uint32_t u[2];
    int ly[2], lz[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {  // each lane inspects rows lane and lane+32
      const int row = lane + 32 * k;
      ly[k] = row % TY;
      lz[k] = row / TY;
      u[k] = fgw[row] & ~covw[row];
    }
#pragma unroll
    for (int r = 0; r < kRegions; ++r) {
      uint32_t xm = 0;
      int ylo = 1 << 20, yhi = -1, zlo = 1 << 20, zhi = -1;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        bool inreg;
        if (IS3D)
          inreg = ((ly[k] >> 2) == ((r >> 1) & 1)) && ((lz[k] >> 2) == (r >> 2));
        else
          inreg = ((ly[k] >> 4) == (r >> 1));
        const uint32_t ur = inreg ? (u[k] & ((r & 1) ? 0xFFFF0000u : 0x0000FFFFu)) : 0u;
        if (ur) {
          xm |= ur;
          ylo = min(ylo, ly[k]);
          yhi = max(yhi, ly[k]);
          zlo = min(zlo, lz[k]);
          zhi = max(zhi, lz[k]);
        }
      }
      xm = __reduce_or_sync(kFull, xm);
      ylo = __reduce_min_sync(kFull, ylo);
      yhi = __reduce_max_sync(kFull, yhi);
      zlo = __reduce_min_sync(kFull, zlo);
      zhi = __reduce_max_sync(kFull, zhi);
      if (lane == 0) {
        int* bx = bxs + r * 6;
        if (xm) {
          bx[0] = __ffs(xm) - 1;
          bx[1] = 31 - __clz(xm);
          bx[2] = ylo;
          bx[3] = yhi;
          bx[4] = zlo;
          bx[5] = zhi;
        } else {
          bx[0] = 1;
          bx[1] = 0;  // empty
        }
      }
    }
    __syncwarp();
  };
  if (active) refresh_boxes();

  const int rmax = dmax > 0 ? isqrt16((int)(dmax - 1)) : 0;
  const int nrx = (rmax + kTX - 1) / kTX, nry = (rmax + TY - 1) / TY, nrz = IS3D ? (rmax + TZ - 1) / TZ : 0;
  uint32_t n_rows = 0;

  // ---- rounds over D-bucket ranges (normally exactly one) --------------------------------
  if (tid == 0) {
    S.round_hi = kBuckets - 1;
    S.fallback = 0;
  }
  __syncthreads();
  for (;;) {
    const int rhi = S.round_hi;
    for (int i = tid; i < kBuckets; i += kWarps * 32) S.hist[i] = 0;
    if (tid == 0) S.count = 0;
    __syncthreads();
    gather<IS3D, true>(S, meta, cent, g, b, tx0, ty0, tz0, nrx, nry, nrz, 0, rhi);
    __syncthreads();
    // --- this round's bucket range [rlo, rhi]: as many buckets as fit the list (warp 0:
    // descending inclusive scan of the histogram, 4 buckets per lane)
    if (warp == 0) {
      uint32_t h[4], sum = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // lane l holds buckets 127-4l .. 124-4l (descending order)
        const int k = kBuckets - 1 - 4 * lane - q;
        h[q] = k <= rhi ? S.hist[k] : 0u;
        sum += h[q];
      }
      uint32_t inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += v;
      }
      uint32_t run = inc - sum;  // exclusive prefix before my first bucket
      int lo_l = -1;             // the highest bucket whose inclusive prefix exceeds kCap
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = kBuckets - 1 - 4 * lane - q;
        S.start[k + 1] = run;
        run += h[q];
        if (lo_l < 0 && k <= rhi && run > kCap) lo_l = k;
      }
      const int lo = __reduce_max_sync(kFull, lo_l);
      // non-empty buckets of the round [lo+1, rhi]
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        uint32_t bits = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int k = kBuckets - 1 - 4 * lane - q;
          if (h[q] && k > lo && k <= rhi && (k >> 5) == w) bits |= 1u << (k & 31);
        }
        bits = __reduce_or_sync(kFull, bits);
        if (lane == 0) S.nonempty[w] = bits;
      }
      if (lane == 0) {
        S.fallback = (lo == rhi && lo >= 0) ? 1 : 0;  // a single bucket exceeds the list
        S.round_lo = lo + 1;
        S.next_hi = lo;
      }
    }
    __syncthreads();
    if (S.fallback) break;
    const int rlo = S.round_lo;
    if (S.count > kCap) {  // the list overflowed: gather again, keeping [rlo, rhi] only (they fit)
      __syncthreads();
      if (tid == 0) S.count = 0;
      __syncthreads();
      gather<IS3D, false>(S, meta, cent, g, b, tx0, ty0, tz0, nrx, nry, nrz, rlo, rhi);
      __syncthreads();
    }
    // --- counting sort of the list indices by bucket (descending)
    const uint32_t total = min(S.count, (uint32_t)kCap);
    for (uint32_t i0 = warp * 32; i0 < total; i0 += kWarps * 32) {
      const uint32_t i = i0 + lane;
      int bk = -1;
      if (i < total) {
        bk = dbucket((uint32_t)(S.list[i] & 0xFFFFu));
        if (bk < rlo || bk > rhi) bk = -1;
      }
      const uint32_t grp = __match_any_sync(kFull, bk);
      uint32_t base = 0;
      if (bk >= 0 && lane == __ffs(grp) - 1) base = atomicAdd(&S.start[bk + 1], (uint32_t)__popc(grp));
      base = __shfl_sync(kFull, base, __ffs(grp) - 1);
      if (bk >= 0) S.idx[base + __popc(grp & ((1u << lane) - 1u))] = (uint16_t)i;
    }
    __syncthreads();
    const bool last_round = S.next_hi < 0;

    // --- cover: my tile, non-empty buckets from high to low ----------------------------------
    if (active) {
      for (int w4 = 3; w4 >= 0; --w4) {
        uint32_t bits = S.nonempty[w4];
        while (bits) {
          const int bk = w4 * 32 + 31 - __clz(bits);
          bits &= ~(1u << (bk & 31));
          // after the sort, start[bk+1] is the end of bucket bk and start[bk+2] its beginning
          const uint32_t s0 = bk == kBuckets - 1 ? 0u : S.start[bk + 2];
          const uint32_t s1 = S.start[bk + 1];
          for (uint32_t i0 = s0; i0 < s1; i0 += 32) {
            const uint32_t i = i0 + lane;
            bool need = false;
            int cx = 0, cy = 0, cz = 0, D = 0;
            if (i < s1) {
              const unsigned long long e = S.list[S.idx[i]];
              D = (int)(e & 0xFFFFu);
              cx = (int)((e >> 16) & 0xFFFFu) - kOff - mox;
              cy = (int)((e >> 32) & 0xFFFFu) - kOff - moy;
              cz = (int)((e >> 48) & 0xFFFFu) - kOff - moz;
              const int R2 = D - 1;
              // reaches my tile, and some region with uncovered foreground
              const int ddx = gap(0, kTX - 1, cx), ddy = gap(0, TY - 1, cy), ddz = gap(0, TZ - 1, cz);
              if (ddx * ddx + ddy * ddy + ddz * ddz <= R2) {
                const int* bxs = &S.box[warp][0][0];
#pragma unroll
                for (int r = 0; r < kRegions; ++r) {
                  const int* bx = bxs + r * 6;
                  if (bx[0] > bx[1]) continue;
                  const int gx = gap(bx[0], bx[1], cx), gy = gap(bx[2], bx[3], cy), gz = gap(bx[4], bx[5], cz);
                  need |= gx * gx + gy * gy + gz * gz <= R2;
                }
              }
            }
            uint32_t act = __ballot_sync(kFull, need);
            while (act) {
              const int k = __ffs(act) - 1;
              act &= act - 1;
              const int jx = __shfl_sync(kFull, cx, k), jy = __shfl_sync(kFull, cy, k), jz = __shfl_sync(kFull, cz, k);
              const int jD = __shfl_sync(kFull, D, k);
              const int R2 = jD - 1, rho = isqrt16(R2);
              const int y0 = max(0, jy - rho), y1 = min(TY - 1, jy + rho);
              const int z0 = max(0, jz - rho), z1 = min(TZ - 1, jz + rho);
              const int nyr = y1 - y0 + 1, nrows = nyr * (z1 - z0 + 1);
              const uint32_t magic = c_magic[nyr];
              const uint32_t xbox = range_mask(max(jx - rho, 0), min(jx + rho, kTX - 1));
              const uint16_t dv = (uint16_t)jD;
              for (int r = lane; r < nrows; r += 32) {
                const int zo = (int)(((uint32_t)r * magic) >> 16);
                const int yy = y0 + (r - zo * nyr), zz = z0 + zo;
                const int row = zz * TY + yy;
                // cheap row skip: nothing uncovered in this row under the ball's x-extent
                uint32_t m = fgw[row] & ~covw[row] & xbox;
                if (!m) continue;
                const int dy = yy - jy, dz = zz - jz;
                const int hrem = R2 - dy * dy - dz * dz;
                if (hrem < 0) continue;
                const int w = isqrt16(hrem);
                const int l = max(jx - w, 0), rr = min(jx + w, kTX - 1);
                if (l > rr) continue;
                ++n_rows;
                m &= range_mask(l, rr);
                if (!m) continue;
                curw[row] |= m;
                uint16_t* vr = val + row * 32;
                while (m) {
                  const int c = __ffs(m) - 1;
                  m &= m - 1;
                  if (vr[c] < dv) vr[c] = dv;
                }
              }
            }
          }
          __syncwarp();
          // bucket done: its coverage becomes "earlier-bucket" coverage
          uint32_t chg = 0;
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const int row = lane + 32 * k;
            const uint32_t c = curw[row];
            chg |= c & ~covw[row];
            covw[row] |= c;
            curw[row] = 0;
          }
          const bool any_new = __any_sync(kFull, chg != 0);
          __syncwarp();
          if (any_new) refresh_boxes();
        }
      }
    }
    if (last_round) break;  // no trailing barrier: warps go straight to their epilogue
    __syncthreads();
    if (tid == 0) S.round_hi = S.next_hi;
    __syncthreads();
  }

  if (S.fallback) {  // leave this group to k_dilate_atomic
    if (lane == 0 && have_tile) meta[mtile].pad = 1u;
    if (tid == 0) atomicAdd(&hdr->n_fallback, 1u);
    return;
  }
  if (!active) return;

  // ---- epilogue: my tile ------------------------------------------------------------------
  const int scale_log2 = sum_scale_log2(g.Z * g.Y * g.X, dmax);
  const double scale = ldexp(1.0, scale_log2);
  uint32_t bad = 0;
  for (int row = 0; row < kRows; ++row) {
    const int ly = row % TY, lz = row / TY;
    const int64_t gz = roz + moz + lz, gy = roy + moy + ly, gx = rox + mox + lane;
    if (gz >= g.Z || gy >= g.Y) continue;  // warp-uniform
    const uint32_t c = val[row * 32 + lane];
    bad |= row_epilogue(c, lane, gx < g.X, item + (gz * g.Y + gy) * g.X + gx, b, lab, Dg, acc, do_reduce, scale,
                        lt2_out, lt_out);
  }
  n_rows = __reduce_add_sync(kFull, n_rows);
  if (lane == 0 && n_rows) atomicAdd(&hdr->n_intervals, (unsigned long long)n_rows);
  if (bad) atomicOr(&hdr->status, kStInternal);
}

}  // namespace

size_t dilate_cover_smem() { return sizeof(Smem); }

void launch_dilate_cover(const int32_t* labels, const uint32_t* D, TileMeta* meta, const uint2* centres,
                         const Geom& g, const Accum& a, int do_reduce, uint32_t* lt2_out, float* lt_out, WsHeader* hdr,
                         cudaStream_t st) {
  const int GX = g.ndim == 3 ? 1 : 2, GY = 2, GZ = g.ndim == 3 ? 2 : 1;
  const int64_t ngroups = g.B * ((g.ntx + GX - 1) / GX) * ((g.nty + GY - 1) / GY) * ((g.ntz + GZ - 1) / GZ);
  const size_t smem = sizeof(Smem);
  if (g.ndim == 3)
    k_dilate_cover<true><<<(unsigned)ngroups, kWarps * 32, smem, st>>>(labels, D, meta, centres, g, a, do_reduce,
                                                                        lt2_out, lt_out, hdr);
  else
    k_dilate_cover<false><<<(unsigned)ngroups, kWarps * 32, smem, st>>>(labels, D, meta, centres, g, a, do_reduce,
                                                                         lt2_out, lt_out, hdr);
}

cudaError_t dilate_cover_setup() {
  cudaError_t e = cudaFuncSetAttribute(k_dilate_cover<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(Smem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_dilate_cover<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
  return e;
}

}  // namespace fastrs
