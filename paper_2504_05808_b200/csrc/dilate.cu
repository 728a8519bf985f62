// K5 (default path): exact ball dilation LT^2(p) = max{ D(q) : |p-q|^2 < D(q) }
// by "sorted cover", fused with the shell test and the per-label reductions.
//
// Work organisation.  A CTA owns a group of 4 output tiles (3D: 1x2x2 tiles of 32x8x8, 2D:
// 2x2 tiles of 32x64); each warp owns one tile privately (values, coverage masks), so the
// hot loop has no atomics and no inter-warp conflicts.
//   1. gather   : the CTA collects every kept maximal ball (K4 output) whose ball reaches
//                 the group's box into a shared list (8-byte packed centre + D).
//   2. sort     : a counting sort by a monotone bucket of D (8 buckets per octave).
//   3. cover    : each warp walks the buckets from the largest D down.  A ball is tested
//                 against the bounding boxes of the still-uncovered foreground elements of
//                 its tile (8 regions) and skipped when it cannot reach any of them; else
//                 its rows are emitted (lanes over the ball's rows, interval |x-qx| <=
//                 isqrt(D-1-dy^2-dz^2)), and only cells not covered by an EARLIER bucket are
//                 max-updated.  Cells covered by an earlier bucket hold a value >= every D
//                 of later buckets, so skipping them is exact; within a bucket updates are
//                 plain max, so the result never depends on the order inside a bucket.
//   4. epilogue : LT^2 per element, shell (D == 1), per-label reductions (shared with the
//                 fallback kernel in lt.cu).
// Exactness does not depend on any test being tight: every skip is justified by cells
// already holding a value >= D.  Overflowing gathers are processed in D-descending rounds;
// the pathological case (one bucket holding more than the list capacity) marks the tile
// for the atomic fallback kernel k_dilate_atomic (lt.cu), which also handles Dmax > 65535.
#include "common.cuh"
#include "dilate_common.cuh"

namespace fastrs {
namespace {

constexpr int kGroup = 4;
constexpr int kCap = 2048;
constexpr int kBuckets = 128;
constexpr int kRegions = 8;
constexpr int kOff = 16384;  // coordinate bias of packed candidates

__constant__ uint32_t c_magic[65] = {
    0,    65536, 32768, 21846, 16384, 13108, 10923, 9363, 8192, 7282, 6554, 5958, 5462, 5042, 4682, 4370, 4096,
    3856, 3641,  3450,  3277,  3121,  2979,  2850,  2731, 2622, 2521, 2428, 2341, 2260, 2185, 2115, 2048, 1986,
    1928, 1873,  1821,  1772,  1725,  1681,  1639,  1599, 1561, 1525, 1490, 1457, 1425, 1395, 1366, 1338, 1311,
    1286, 1261,  1237,  1214,  1192,  1171,  1150,  1130, 1111, 1093, 1075, 1058, 1041, 1024};

struct Smem {
  uint16_t val[kGroup][kRows * 32];
  uint32_t fg[kGroup][kRows];
  uint32_t cov[kGroup][kRows];
  uint32_t cur[kGroup][kRows];
  int box[kGroup][kRegions][6];
  unsigned long long listA[kCap];
  unsigned long long listB[kCap];
  uint32_t hist[kBuckets];
  uint32_t start[kBuckets + 1];
  uint32_t count;
  int round_lo, round_hi;  // bucket range [lo, hi] of the current round
  int next_hi;
  int fallback;
};

__device__ __forceinline__ int dbucket(uint32_t D) {
  const int msb = 31 - __clz(D);
  const int frac = msb >= 3 ? (int)((D >> (msb - 3)) & 7u) : (int)((D << (3 - msb)) & 7u);
  return msb * 8 + frac;  // monotone non-decreasing in D, 0..127 for D < 65536
}

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

template <bool IS3D>
__global__ void __launch_bounds__(kGroup * 32) k_dilate_cover(const int32_t* __restrict__ lab,
                                                             const uint32_t* __restrict__ Dg,
                                                             TileMeta* __restrict__ meta,
                                                             const uint2* __restrict__ cent, Geom g, Accum acc,
                                                             int do_reduce, uint32_t* __restrict__ lt2_out,
                                                             float* __restrict__ lt_out, WsHeader* __restrict__ hdr) {
  constexpr int TY = IS3D ? 8 : 64, TZ = IS3D ? 8 : 1;
  constexpr int GX = IS3D ? 1 : 2, GY = 2, GZ = IS3D ? 2 : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t dmax = hdr->dmax;
  if (dmax > kU16Max) return;  // k_dilate_atomic handles it

  // ---- group / tile coordinates --------------------------------------------------------
  const int64_t ngx = (g.ntx + GX - 1) / GX, ngy = (g.nty + GY - 1) / GY, ngz = (g.ntz + GZ - 1) / GZ;
  int64_t t = blockIdx.x;
  const int64_t gxi = t % ngx;
  t /= ngx;
  const int64_t gyi = t % ngy;
  t /= ngy;
  const int64_t gzi = t % ngz;
  const int64_t b = t / ngz;
  const int64_t tx0 = gxi * GX, ty0 = gyi * GY, tz0 = gzi * GZ;
  const int64_t rox = tx0 * kTX, roy = ty0 * TY, roz = tz0 * TZ;  // region origin
  const int RX = GX * kTX, RY = GY * TY, RZ = GZ * TZ;
  // my tile
  const int wx = warp % GX, wy = (warp / GX) % GY, wz = warp / (GX * GY);
  const int64_t mtx = tx0 + wx, mty = ty0 + wy, mtz = tz0 + wz;
  const bool have_tile = mtx < g.ntx && mty < g.nty && mtz < g.ntz;
  const int64_t mtile = have_tile ? ((b * g.ntz + mtz) * g.nty + mty) * g.ntx + mtx : 0;
  const int mox = wx * kTX, moy = wy * TY, moz = wz * TZ;  // my tile origin within the region
  bool active = have_tile && meta[mtile].nfg != 0;
  // whole CTA idle?
  if (__syncthreads_or(active) == 0) return;

  const int64_t item = b * g.Z * g.Y * g.X;
  // ---- per-warp init: values, foreground masks, coverage ----------------------------------
  uint16_t* val = S.val[warp];
  for (int i = lane; i < kRows * 32 / 2; i += 32) reinterpret_cast<uint32_t*>(val)[i] = 0;
  for (int row = 0; row < kRows; ++row) {
    const int ly = row % TY, lz = row / TY;
    const int64_t gz = roz + moz + lz, gy = roy + moy + ly, gx = rox + mox + lane;
    bool f = false;
    if (active && gz < g.Z && gy < g.Y && gx < g.X) f = __ldg(Dg + item + (gz * g.Y + gy) * g.X + gx) != 0;
    const uint32_t m = __ballot_sync(kFull, f);
    if (lane == 0) {
      S.fg[warp][row] = m;
      S.cov[warp][row] = 0;
      S.cur[warp][row] = 0;
    }
  }
  __syncwarp();

  // uncovered-foreground bounding boxes of the 8 regions of my tile
  auto refresh_boxes = [&]() {
    // regions: x halves (bit 0), y halves (bit 1), z halves (bit 2) (2D: y quarters)
    for (int r = 0; r < kRegions; ++r) {
      const int xh = r & 1;
      int rylo, ryhi, rzlo, rzhi;
      if (IS3D) {
        rylo = (r >> 1 & 1) * 4; ryhi = rylo + 3; rzlo = (r >> 2 & 1) * 4; rzhi = rzlo + 3;
      } else {
        rylo = (r >> 1) * 16; ryhi = rylo + 15; rzlo = 0; rzhi = 0;
      }
      uint32_t xm = 0;
      int ylo = 1 << 20, yhi = -1, zlo = 1 << 20, zhi = -1;
      for (int row = lane; row < kRows; row += 32) {
        const int ly = row % TY, lz = row / TY;
        if (ly < rylo || ly > ryhi || lz < rzlo || lz > rzhi) continue;
        const uint32_t u = S.fg[warp][row] & ~S.cov[warp][row] & (xh ? 0xFFFF0000u : 0x0000FFFFu);
        if (u) {
          xm |= u;
          ylo = min(ylo, ly); yhi = max(yhi, ly);
          zlo = min(zlo, lz); zhi = max(zhi, lz);
        }
      }
      xm = __reduce_or_sync(kFull, xm);
      ylo = __reduce_min_sync(kFull, ylo); yhi = __reduce_max_sync(kFull, yhi);
      zlo = __reduce_min_sync(kFull, zlo); zhi = __reduce_max_sync(kFull, zhi);
      if (lane == 0) {
        int* bx = S.box[warp][r];
        if (xm) {
          bx[0] = __ffs(xm) - 1; bx[1] = 31 - __clz(xm);
          bx[2] = ylo; bx[3] = yhi; bx[4] = zlo; bx[5] = zhi;
        } else {
          bx[0] = 1; bx[1] = 0;  // empty
        }
      }
    }
    __syncwarp();
  };
  if (active) refresh_boxes();

  const int rmax = dmax > 0 ? isqrt16((int)(dmax - 1)) : 0;
  const int nrx = (rmax + kTX - 1) / kTX, nry = (rmax + TY - 1) / TY, nrz = IS3D ? (rmax + TZ - 1) / TZ : 0;
  const int nx = GX + 2 * nrx, ny = GY + 2 * nry, nz = GZ + 2 * nrz;
  const int nneigh = nx * ny * nz;
  uint32_t n_rows = 0;

  // ---- rounds over D-bucket ranges (normally exactly one) --------------------------------
  if (tid == 0) {
    S.round_hi = kBuckets - 1;
    S.fallback = 0;
  }
  __syncthreads();
  for (;;) {
    const int rhi = S.round_hi;
    // --- gather: candidates with bucket <= rhi reaching the region, histogram all of them
    for (int i = tid; i < kBuckets; i += kGroup * 32) S.hist[i] = 0;
    if (tid == 0) S.count = 0;
    __syncthreads();
    for (int nb0 = 0; nb0 < nneigh; nb0 += kGroup * 32) {
      const int n = nb0 + tid;
      bool reach = false;
      int64_t ht = 0;
      uint32_t hcount = 0;
      int hox = 0, hoy = 0, hoz = 0;
      if (n < nneigh) {
        const int ix = n % nx, iy = (n / nx) % ny, iz = n / (nx * ny);
        const int64_t hx = tx0 + ix - nrx, hy = ty0 + iy - nry, hz = tz0 + iz - nrz;
        if (hx >= 0 && hx < g.ntx && hy >= 0 && hy < g.nty && hz >= 0 && hz < g.ntz) {
          ht = ((b * g.ntz + hz) * g.nty + hy) * g.ntx + hx;
          const TileMeta hm = meta[ht];
          hox = (int)(hx - tx0) * kTX;
          hoy = (int)(hy - ty0) * TY;
          hoz = (int)(hz - tz0) * TZ;
          // gap between the home tile box and the region box
          const int gx = hox < 0 ? -(hox + kTX - 1) : (hox > RX - 1 ? hox - (RX - 1) : 0);
          const int gy = hoy < 0 ? -(hoy + TY - 1) : (hoy > RY - 1 ? hoy - (RY - 1) : 0);
          const int gz = hoz < 0 ? -(hoz + TZ - 1) : (hoz > RZ - 1 ? hoz - (RZ - 1) : 0);
          reach = hm.count && gx * gx + gy * gy + gz * gz <= (int)hm.maxD - 1;
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
        const uint2* src = cent + (size_t)hts * kTileVol;
        for (uint32_t e0 = 0; e0 < cnt; e0 += 32) {
          bool take = false;
          int cx = 0, cy = 0, cz = 0, bk = 0;
          uint32_t Dq = 0;
          if (e0 + lane < cnt) {
            const uint2 e = __ldg(src + e0 + lane);
            const int v = (int)e.x;
            cx = bx + (v & 31);
            cy = by + ((v >> 5) % TY);
            cz = bz + v / (32 * TY);
            Dq = e.y;
            const int ddx = gap(0, RX - 1, cx), ddy = gap(0, RY - 1, cy), ddz = gap(0, RZ - 1, cz);
            if (ddx * ddx + ddy * ddy + ddz * ddz <= (int)Dq - 1) {
              bk = dbucket(Dq);
              take = bk <= rhi;
            }
          }
          const uint32_t tm = __ballot_sync(kFull, take);
          if (!tm) continue;
          // histogram (match groups -> one atomic per distinct bucket)
          const uint32_t grp = __match_any_sync(kFull, take ? bk : -1);
          if (take && lane == __ffs(grp) - 1) atomicAdd(&S.hist[bk], __popc(grp));
          uint32_t base = 0;
          if (lane == 0) base = atomicAdd(&S.count, __popc(tm));
          base = __shfl_sync(kFull, base, 0);
          const uint32_t pos = base + __popc(tm & ((1u << lane) - 1u));
          if (take && pos < kCap) S.listA[pos] = pack(cx, cy, cz, Dq);
        }
      }
    }
    __syncthreads();
    // --- decide this round's bucket range [rlo, rhi] so it fits the list
    if (tid == 0) {
      uint32_t sum = 0;
      int lo = rhi;
      while (lo >= 0 && sum + S.hist[lo] <= kCap) {
        sum += S.hist[lo];
        --lo;
      }
      // buckets (lo, rhi] fit; bucket lo (if >= 0) does not
      if (lo == rhi && lo >= 0) {
        S.fallback = 1;  // a single bucket exceeds the capacity
        S.round_lo = 0;
      } else {
        S.round_lo = lo + 1;
      }
      S.next_hi = lo;  // next round starts at bucket lo (or stop if < 0)
      // bucket starts (descending order of buckets) for [round_lo, rhi]
      uint32_t acc_s = 0;
      for (int k = kBuckets - 1; k >= 0; --k) {
        S.start[k + 1] = acc_s;  // start of bucket k is stored at start[k+1] (descending layout)
        if (k <= rhi && k >= S.round_lo) acc_s += S.hist[k];
      }
      S.start[0] = acc_s;
    }
    __syncthreads();
    if (S.fallback) break;
    const int rlo = S.round_lo;
    const uint32_t total_all = S.count;
    // --- scatter listA -> listB by bucket (descending), keeping only buckets in [rlo, rhi]
    if (total_all <= kCap) {
      for (uint32_t i0 = warp * 32; i0 < total_all; i0 += kGroup * 32) {
        const uint32_t i = i0 + lane;
        unsigned long long e = 0;
        int bk = -1;
        if (i < total_all) {
          e = S.listA[i];
          bk = dbucket((uint32_t)(e & 0xFFFFu));
          if (bk < rlo || bk > rhi) bk = -1;
        }
        const uint32_t grp = __match_any_sync(kFull, bk);
        uint32_t base = 0;
        if (bk >= 0 && lane == __ffs(grp) - 1) base = atomicAdd(&S.start[bk + 1], __popc(grp));
        base = __shfl_sync(kFull, base, __ffs(grp) - 1);
        if (bk >= 0) S.listB[base + __popc(grp & ((1u << lane) - 1u))] = e;
      }
    } else {
      // the list overflowed: re-gather is needed for buckets [rlo, rhi] only
      __syncthreads();
      if (tid == 0) S.count = 0;
      __syncthreads();
      for (int nb0 = 0; nb0 < nneigh; nb0 += kGroup * 32) {
        const int n = nb0 + tid;
        bool reach = false;
        int64_t ht = 0;
        uint32_t hcount = 0;
        int hox = 0, hoy = 0, hoz = 0;
        if (n < nneigh) {
          const int ix = n % nx, iy = (n / nx) % ny, iz = n / (nx * ny);
          const int64_t hx = tx0 + ix - nrx, hy = ty0 + iy - nry, hz = tz0 + iz - nrz;
          if (hx >= 0 && hx < g.ntx && hy >= 0 && hy < g.nty && hz >= 0 && hz < g.ntz) {
            ht = ((b * g.ntz + hz) * g.nty + hy) * g.ntx + hx;
            const TileMeta hm = meta[ht];
            hox = (int)(hx - tx0) * kTX;
            hoy = (int)(hy - ty0) * TY;
            hoz = (int)(hz - tz0) * TZ;
            const int gx = hox < 0 ? -(hox + kTX - 1) : (hox > RX - 1 ? hox - (RX - 1) : 0);
            const int gy = hoy < 0 ? -(hoy + TY - 1) : (hoy > RY - 1 ? hoy - (RY - 1) : 0);
            const int gz = hoz < 0 ? -(hoz + TZ - 1) : (hoz > RZ - 1 ? hoz - (RZ - 1) : 0);
            reach = hm.count && gx * gx + gy * gy + gz * gz <= (int)hm.maxD - 1;
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
          const uint2* src = cent + (size_t)hts * kTileVol;
          for (uint32_t e0 = 0; e0 < cnt; e0 += 32) {
            int bk = -1;
            unsigned long long pe = 0;
            if (e0 + lane < cnt) {
              const uint2 e = __ldg(src + e0 + lane);
              const int v = (int)e.x;
              const int cx = bx + (v & 31), cy = by + ((v >> 5) % TY), cz = bz + v / (32 * TY);
              const int ddx = gap(0, RX - 1, cx), ddy = gap(0, RY - 1, cy), ddz = gap(0, RZ - 1, cz);
              if (ddx * ddx + ddy * ddy + ddz * ddz <= (int)e.y - 1) {
                bk = dbucket(e.y);
                if (bk < rlo || bk > rhi) bk = -1;
                pe = pack(cx, cy, cz, e.y);
              }
            }
            const uint32_t grp = __match_any_sync(kFull, bk);
            uint32_t base = 0;
            if (bk >= 0 && lane == __ffs(grp) - 1) base = atomicAdd(&S.start[bk + 1], __popc(grp));
            base = __shfl_sync(kFull, base, __ffs(grp) - 1);
            if (bk >= 0) S.listB[base + __popc(grp & ((1u << lane) - 1u))] = pe;
          }
        }
      }
    }
    __syncthreads();

    // --- cover: my tile, buckets from high to low -----------------------------------------
    if (active) {
      for (int bk = rhi; bk >= rlo; --bk) {
        // after the scatter, start[bk+1] was advanced to the end of bucket bk
        const uint32_t s0 = bk == kBuckets - 1 ? 0u : S.start[bk + 2];
        const uint32_t s1 = S.start[bk + 1];
        if (s1 <= s0) continue;
        bool any_new = false;
        for (uint32_t i0 = s0; i0 < s1; i0 += 32) {
          const uint32_t i = i0 + lane;
          bool need = false;
          int cx = 0, cy = 0, cz = 0, D = 0;
          if (i < s1) {
            const unsigned long long e = S.listB[i];
            D = (int)(e & 0xFFFFu);
            cx = (int)((e >> 16) & 0xFFFFu) - kOff - mox;
            cy = (int)((e >> 32) & 0xFFFFu) - kOff - moy;
            cz = (int)((e >> 48) & 0xFFFFu) - kOff - moz;
            const int R2 = D - 1;
            // reaches my tile, and some region with uncovered foreground
            const int ddx = gap(0, kTX - 1, cx), ddy = gap(0, TY - 1, cy), ddz = gap(0, TZ - 1, cz);
            if (ddx * ddx + ddy * ddy + ddz * ddz <= R2) {
#pragma unroll
              for (int r = 0; r < kRegions; ++r) {
                const int* bx = S.box[warp][r];
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
            const int z0 = IS3D ? max(0, jz - rho) : 0, z1 = IS3D ? min(TZ - 1, jz + rho) : 0;
            const int nyr = y1 - y0 + 1, nrows = nyr * (z1 - z0 + 1);
            const uint32_t magic = c_magic[nyr];  // ceil(2^16/nyr): exact r/nyr for r < 64
            for (int r = lane; r < nrows; r += 32) {
              const int zo = (int)(((uint32_t)r * magic) >> 16);
              const int yy = y0 + (r - zo * nyr), zz = z0 + zo;
              const int dy = yy - jy, dz = zz - jz;
              const int hrem = R2 - dy * dy - dz * dz;
              if (hrem < 0) continue;
              const int w = isqrt16(hrem);
              const int l = max(jx - w, 0), rr = min(jx + w, kTX - 1);
              if (l > rr) continue;
              ++n_rows;
              const int row = zz * TY + yy;
              const uint32_t span = (rr == 31 ? 0xFFFFFFFFu : ((1u << (rr + 1)) - 1u)) & (0xFFFFFFFFu << l);
              uint32_t m = span & S.fg[warp][row] & ~S.cov[warp][row];
              if (!m) continue;
              S.cur[warp][row] |= m;
              uint16_t* vr = val + row * 32;
              const uint16_t dv = (uint16_t)jD;
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
        for (int row = lane; row < kRows; row += 32) {
          const uint32_t c = S.cur[warp][row];
          chg |= c & ~S.cov[warp][row];
          S.cov[warp][row] |= c;
          S.cur[warp][row] = 0;
        }
        any_new = __any_sync(kFull, chg != 0);
        __syncwarp();
        if (any_new) refresh_boxes();
      }
    }
    __syncthreads();
    if (S.next_hi < 0) break;
    if (tid == 0) S.round_hi = S.next_hi;
    __syncthreads();
  }

  if (S.fallback) {
    // leave this group to k_dilate_atomic (flag the tiles)
    if (lane == 0 && have_tile) meta[mtile].pad = 1u;
    if (tid == 0) atomicAdd(&hdr->n_fallback, 1u);
    return;
  }
  if (!active) return;

  // ---- epilogue ---------------------------------------------------------------------------
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
    k_dilate_cover<true><<<(unsigned)ngroups, kGroup * 32, smem, st>>>(labels, D, meta, centres, g, a, do_reduce,
                                                                        lt2_out, lt_out, hdr);
  else
    k_dilate_cover<false><<<(unsigned)ngroups, kGroup * 32, smem, st>>>(labels, D, meta, centres, g, a, do_reduce,
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
