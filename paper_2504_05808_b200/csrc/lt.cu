// Local thickness:  LT^2(p) = max{ D(q) : |p-q|^2 < D(q) }
// ("radius of the largest circle/sphere that fits in the object at any point",
// PAPER.md:85 §4; strict membership, reading c5).  A ball of q only covers elements of
// q's own label (anything at squared distance < D(q) from q is not a site), so no label
// test is needed.
//
//   K7 mtable   : per-device lattice containment table M(D,s) = max_{|u|^2 <= D-1} |u-s|^2
//                 for the 12 (3D) / 5 (2D) offset classes, built once.
//   K4 prune    : drop centre q when some offset s (26 / 8 neighbours first, then all
//                 |s|^2 <= 12 / 8) has D(q+s) > M(D(q), s), i.e. the lattice ball of q lies
//                 inside the ball of q+s.  Strict containment is a strict partial order, so
//                 every dropped ball lies in a kept maximal ball with a larger D: LT^2 is
//                 unchanged (exact).  Survivors are compacted per 32x8x8 (2D 32x64) home
//                 tile, in element order, with per-tile count / max D / #foreground.
//   K5 dilate   : one CTA per output tile.  It gathers the kept centres of every home tile
//                 whose max ball can reach it, and every centre emits, per intersected x-row
//                 of the tile, the interval |x - qx| <= isqrt(D-1-dy^2-dz^2).  An interval
//                 [l,r] costs two shared-memory atomicMax into the row's reverse sparse table
//                 (level k = floor(log2(r-l+1)), cells l and r-2^k+1); a register/shuffle
//                 push-down over the 6 levels ("warp-level max") yields LT^2 of the row.
//                 Fused epilogue: shell (D == 1, equivalent to a 4/6-neighbour with another
//                 label or the border), lt = sqrt((double)LT^2), and
//                 per-label segmented reductions (warp __match-style grouping by ballot,
//                 __reduce_*_sync, then one global atomic per group).
#include <mutex>
#include <vector>

#include "common.cuh"

namespace fastrs {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

__constant__ int c_off3[178];
__constant__ int c_cls3[kClasses3 + 1];
__constant__ int c_off2[24];
__constant__ int c_cls2[kClasses2 + 1];

// canonical class representatives (sorted descending), ordered by |s|^2
__constant__ int c_rep3[kClasses3][3] = {{1, 0, 0}, {1, 1, 0}, {1, 1, 1}, {2, 0, 0}, {2, 1, 0}, {2, 1, 1},
                                         {2, 2, 0}, {2, 2, 1}, {3, 0, 0}, {3, 1, 0}, {3, 1, 1}, {2, 2, 2}};
__constant__ int c_rep2[kClasses2][2] = {{1, 0}, {1, 1}, {2, 0}, {2, 1}, {2, 2}};
static const int h_rep3[kClasses3][3] = {{1, 0, 0}, {1, 1, 0}, {1, 1, 1}, {2, 0, 0}, {2, 1, 0}, {2, 1, 1},
                                         {2, 2, 0}, {2, 2, 1}, {3, 0, 0}, {3, 1, 0}, {3, 1, 1}, {2, 2, 2}};
static const int h_rep2[kClasses2][2] = {{1, 0}, {1, 1}, {2, 0}, {2, 1}, {2, 2}};

__device__ __forceinline__ int isqrt_i(int h) {
  int w = (int)sqrtf((float)h);
  while (w * w > h) --w;
  while ((w + 1) * (w + 1) <= h) ++w;
  return w;
}

// ---------------------------------------------------------------------------------------
// K7: lattice containment tables
// ---------------------------------------------------------------------------------------
__global__ void k_mtable3(uint32_t* M) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)kClasses3 * (kDcap3 + 1)) return;
  const int c = (int)(t / (kDcap3 + 1)), D = (int)(t % (kDcap3 + 1));
  if (D == 0) {
    M[t] = 0;
    return;
  }
  const int s0 = c_rep3[c][0], s1 = c_rep3[c][1], s2 = c_rep3[c][2];
  const int R2 = D - 1, r = isqrt_i(R2);
  uint32_t best = 0;
  for (int u0 = -r; u0 <= r; ++u0) {
    const int rem0 = R2 - u0 * u0, r1 = isqrt_i(rem0);
    for (int u1 = -r1; u1 <= r1; ++u1) {
      const int w = isqrt_i(rem0 - u1 * u1);  // u2 = -w maximises (u2 - s2)^2 for s2 >= 0
      const uint32_t v = (u0 - s0) * (u0 - s0) + (u1 - s1) * (u1 - s1) + (w + s2) * (w + s2);
      best = v > best ? v : best;
    }
  }
  M[t] = best;
}

__global__ void k_mtable2(uint32_t* M) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)kClasses2 * (kDcap2 + 1)) return;
  const int c = (int)(t / (kDcap2 + 1)), D = (int)(t % (kDcap2 + 1));
  if (D == 0) {
    M[t] = 0;
    return;
  }
  const int s0 = c_rep2[c][0], s1 = c_rep2[c][1];
  const int R2 = D - 1, r = isqrt_i(R2);
  uint32_t best = 0;
  for (int u0 = -r; u0 <= r; ++u0) {
    const int w = isqrt_i(R2 - u0 * u0);
    const uint32_t v = (u0 - s0) * (u0 - s0) + (w + s1) * (w + s1);
    best = v > best ? v : best;
  }
  M[t] = best;
}

struct DeviceTables {
  uint32_t* m3 = nullptr;
  uint32_t* m2 = nullptr;
};
std::mutex g_mu;
DeviceTables g_tables[64];

// ---------------------------------------------------------------------------------------
// K4: exact maximal-ball pruning + per-tile compaction
// ---------------------------------------------------------------------------------------
template <bool IS3D>
struct PruneTile {
  static constexpr int H = IS3D ? kHalo3 : kHalo2;
  static constexpr int TY = IS3D ? 8 : 64, TZ = IS3D ? 8 : 1;
  static constexpr int PX = kTX + 2 * H, PY = TY + 2 * H, PZ = IS3D ? TZ + 2 * H : 1;
  static constexpr int HZ = IS3D ? H : 0;
};

template <bool IS3D>
__global__ void __launch_bounds__(256) k_prune(const uint32_t* __restrict__ D, Geom g, TileMeta* __restrict__ meta,
                                               uint2* __restrict__ cent, const uint32_t* __restrict__ M,
                                               WsHeader* __restrict__ hdr) {
  using P = PruneTile<IS3D>;
  __shared__ uint32_t s[P::PZ * P::PY * P::PX];
  __shared__ uint32_t keepmask[kRows];
  __shared__ uint32_t pre[kRows];
  __shared__ uint32_t red_cnt[8], red_max[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t tile = blockIdx.x;
  int64_t t = tile;
  const int64_t tx = t % g.ntx;
  t /= g.ntx;
  const int64_t ty = t % g.nty;
  t /= g.nty;
  const int64_t tz = t % g.ntz;
  const int64_t b = t / g.ntz;
  const int64_t z0 = tz * P::TZ - P::HZ, y0 = ty * P::TY - P::H, x0 = tx * kTX - P::H;
  const uint32_t* Db = D + b * g.Z * g.Y * g.X;
  for (int i = tid; i < P::PZ * P::PY * P::PX; i += 256) {
    const int lx = i % P::PX, ly = (i / P::PX) % P::PY, lz = i / (P::PX * P::PY);
    const int64_t gz = z0 + lz, gy = y0 + ly, gx = x0 + lx;
    uint32_t v = 0;
    if (gz >= 0 && gz < g.Z && gy >= 0 && gy < g.Y && gx >= 0 && gx < g.X) v = __ldg(Db + (gz * g.Y + gy) * g.X + gx);
    s[i] = v;
  }
  if (tid < kRows) keepmask[tid] = 0;
  __syncthreads();

  const int ncls = IS3D ? kClasses3 : kClasses2;
  const int dcap = IS3D ? kDcap3 : kDcap2;
  uint32_t nfg = 0, maxd = 0;
  uint32_t keepbits = 0;
#pragma unroll 1
  for (int k = 0; k < kTileVol / 256; ++k) {
    const int v = k * 256 + tid;
    const int lx = v & 31, ly = (v >> 5) % P::TY, lz = v / (32 * P::TY);
    const int64_t gz = tz * P::TZ + lz, gy = ty * P::TY + ly, gx = tx * kTX + lx;
    const int sidx = ((lz + P::HZ) * P::PY + (ly + P::H)) * P::PX + (lx + P::H);
    const uint32_t d = s[sidx];
    bool keep = false;
    if (d != 0 && gz < g.Z && gy < g.Y && gx < g.X) {
      nfg += 1;
      keep = true;
      if (d <= (uint32_t)dcap) {
        for (int c = 0; c < ncls && keep; ++c) {
          const uint32_t m = __ldg(M + c * (dcap + 1) + d);
          const int jb = IS3D ? c_cls3[c] : c_cls2[c], je = IS3D ? c_cls3[c + 1] : c_cls2[c + 1];
          for (int j = jb; j < je; ++j) {
            const int off = IS3D ? c_off3[j] : c_off2[j];
            if (s[sidx + off] > m) {
              keep = false;
              break;
            }
          }
        }
      }
    }
    if (keep) {
      keepbits |= 1u << k;
      maxd = max(maxd, d);
    }
    const uint32_t bal = __ballot_sync(kFull, keep);
    if (lane == 0) keepmask[v >> 5] = bal;  // v>>5 = k*8 + warp: one word per (k, warp)
  }
  __syncthreads();
  // exclusive prefix over the 64 words (element order)
  if (warp == 0) {
    const uint32_t c0 = __popc(keepmask[2 * lane]), c1 = __popc(keepmask[2 * lane + 1]);
    uint32_t inc = c0 + c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t n = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += n;
    }
    const uint32_t ex = inc - c0 - c1;
    pre[2 * lane] = ex;
    pre[2 * lane + 1] = ex + c0;
  }
  __syncthreads();
  uint2* out = cent + tile * kTileVol;
#pragma unroll 1
  for (int k = 0; k < kTileVol / 256; ++k) {
    if (!((keepbits >> k) & 1u)) continue;
    const int v = k * 256 + tid;
    const int lx = v & 31, ly = (v >> 5) % P::TY, lz = v / (32 * P::TY);
    const int sidx = ((lz + P::HZ) * P::PY + (ly + P::H)) * P::PX + (lx + P::H);
    const uint32_t pos = pre[v >> 5] + __popc(keepmask[v >> 5] & ((1u << lane) - 1u));
    out[pos] = make_uint2((uint32_t)v, s[sidx]);
  }
  // tile metadata
  nfg = __reduce_add_sync(kFull, nfg);
  maxd = __reduce_max_sync(kFull, maxd);
  if (lane == 0) {
    red_cnt[warp] = nfg;
    red_max[warp] = maxd;
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t f = 0, m = 0;
    for (int w = 0; w < 8; ++w) {
      f += red_cnt[w];
      m = max(m, red_max[w]);
    }
    const uint32_t cnt = pre[kRows - 1] + __popc(keepmask[kRows - 1]);
    meta[tile] = TileMeta{cnt, m, f, 0};
    if (cnt) atomicAdd(&hdr->n_kept, (unsigned long long)cnt);
  }
}

// ---------------------------------------------------------------------------------------
// K5: dilation (reverse sparse tables) + shell + per-label reductions
// ---------------------------------------------------------------------------------------
constexpr int kRcap = 1024;

template <bool IS3D>
__global__ void __launch_bounds__(256) k_dilate(const int32_t* __restrict__ lab, const uint32_t* __restrict__ Dg,
                                                const TileMeta* __restrict__ meta, const uint2* __restrict__ cent,
                                                Geom g, Accum acc, int do_reduce, uint32_t* __restrict__ lt2_out,
                                                float* __restrict__ lt_out, WsHeader* __restrict__ hdr) {
  constexpr int TY = IS3D ? 8 : 64, TZ = IS3D ? 8 : 1;
  extern __shared__ uint32_t T[];  // kRows * kRowStride
  __shared__ uint32_t s_rt[kRcap];
  __shared__ uint32_t s_rpre[kRcap + 1];
  __shared__ int s_nr;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t tile = blockIdx.x;
  const TileMeta mt = meta[tile];
  if (mt.nfg == 0) return;
  int64_t t = tile;
  const int64_t tx = t % g.ntx;
  t /= g.ntx;
  const int64_t ty = t % g.nty;
  t /= g.nty;
  const int64_t tz = t % g.ntz;
  const int64_t b = t / g.ntz;
  const int64_t ox = tx * kTX, oy = ty * TY, oz = tz * TZ;

  for (int i = tid; i < kRows * kRowStride; i += 256) T[i] = 0;
  if (tid == 0) s_nr = 0;
  const uint32_t dmax = hdr->dmax;
  const int rmax = dmax > 0 ? isqrt_i((int)(dmax - 1)) : 0;
  const int rx = (rmax + kTX - 1) / kTX, ry = (rmax + TY - 1) / TY, rz = IS3D ? (rmax + TZ - 1) / TZ : 0;
  const int nx = 2 * rx + 1, ny = 2 * ry + 1, nz = 2 * rz + 1;
  const int nneigh = nx * ny * nz;
  __syncthreads();

  unsigned long long n_int = 0;
  for (int base = 0; base < nneigh; base += 256) {
    const int n = base + tid;
    if (n < nneigh) {
      const int ix = n % nx, iy = (n / nx) % ny, iz = n / (nx * ny);
      const int64_t hx = tx + ix - rx, hy = ty + iy - ry, hz = tz + iz - rz;
      if (hx >= 0 && hx < g.ntx && hy >= 0 && hy < g.nty && hz >= 0 && hz < g.ntz) {
        const int64_t ht = ((b * g.ntz + hz) * g.nty + hy) * g.ntx + hx;
        const TileMeta hm = meta[ht];
        if (hm.count) {
          // squared gap between the home tile box and this tile box
          const int64_t gx = hx < tx ? ox - (hx * kTX + kTX - 1) : (hx > tx ? hx * kTX - (ox + kTX - 1) : 0);
          const int64_t gy = hy < ty ? oy - (hy * TY + TY - 1) : (hy > ty ? hy * TY - (oy + TY - 1) : 0);
          const int64_t gz = hz < tz ? oz - (hz * TZ + TZ - 1) : (hz > tz ? hz * TZ - (oz + TZ - 1) : 0);
          if (gx * gx + gy * gy + gz * gz <= (int64_t)hm.maxD - 1) {
            const int k = atomicAdd(&s_nr, 1);
            s_rt[k] = (uint32_t)ht;
          }
        }
      }
    }
    __syncthreads();
    const int nr = s_nr;
    __syncthreads();  // every thread has read s_nr before anyone appends again
    if (nr > kRcap - 256 || base + 256 >= nneigh) {
      // exclusive prefix of the reaching tiles' counts
      if (warp == 0) {
        uint32_t run = 0;
        for (int i0 = 0; i0 < nr; i0 += 32) {
          const int i = i0 + lane;
          const uint32_t c = i < nr ? meta[s_rt[i]].count : 0;
          uint32_t inc = c;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(kFull, inc, o);
            if (lane >= o) inc += v;
          }
          if (i < nr) s_rpre[i] = run + inc - c;
          run += __shfl_sync(kFull, inc, 31);
        }
        if (lane == 0) s_rpre[nr] = run;
      }
      __syncthreads();
      const uint32_t total = s_rpre[nr];
      for (uint32_t cb = (uint32_t)warp * 32; cb < total; cb += 256) {
        const uint32_t idx = cb + lane;
        int cx = 0, cy = 0, cz = 0;
        uint32_t Dq = 0;
        if (idx < total) {
          int lo = 0, hi = nr;
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_rpre[mid] <= idx) lo = mid; else hi = mid;
          }
          const uint32_t ht = s_rt[lo];
          const uint2 e = cent[(size_t)ht * kTileVol + (idx - s_rpre[lo])];
          int64_t h = ht;
          const int64_t hx = h % g.ntx;
          h /= g.ntx;
          const int64_t hy = h % g.nty;
          h /= g.nty;
          const int64_t hz = h % g.ntz;
          const int v = (int)e.x;
          cx = (int)(hx * kTX + (v & 31) - ox);
          cy = (int)(hy * TY + ((v >> 5) % TY) - oy);
          cz = (int)(hz * TZ + (v / (32 * TY)) - oz);
          Dq = e.y;
          const int ddx = max(max(-cx, cx - (kTX - 1)), 0);
          const int ddy = max(max(-cy, cy - (TY - 1)), 0);
          const int ddz = max(max(-cz, cz - (TZ - 1)), 0);
          if ((int64_t)ddx * ddx + (int64_t)ddy * ddy + (int64_t)ddz * ddz > (int64_t)Dq - 1) Dq = 0;
        }
        uint32_t act = __ballot_sync(kFull, Dq != 0);
        while (act) {
          const int j = __ffs(act) - 1;
          act &= act - 1;
          const int jx = __shfl_sync(kFull, cx, j), jy = __shfl_sync(kFull, cy, j), jz = __shfl_sync(kFull, cz, j);
          const uint32_t jD = __shfl_sync(kFull, Dq, j);
          const int R2 = (int)jD - 1, rho = isqrt_i(R2);
          const int y0 = max(0, jy - rho), y1 = min(TY - 1, jy + rho);
          const int z0 = IS3D ? max(0, jz - rho) : 0, z1 = IS3D ? min(TZ - 1, jz + rho) : 0;
          const int nyr = y1 - y0 + 1, nrows = nyr * (z1 - z0 + 1);
          for (int r = lane; r < nrows; r += 32) {
            const int yy = y0 + r % nyr, zz = z0 + r / nyr;
            const int dy = yy - jy, dz = zz - jz;
            const int hrem = R2 - dy * dy - dz * dz;
            if (hrem < 0) continue;
            const int w = isqrt_i(hrem);
            const int l = max(jx - w, 0), rr = min(jx + w, kTX - 1);
            if (l > rr) continue;
            const int k = 31 - __clz(rr - l + 1);
            uint32_t* rowp = T + (zz * TY + yy) * kRowStride + k * 32;
            atomicMax(rowp + l, jD);
            const int l2 = rr - (1 << k) + 1;
            if (l2 != l) atomicMax(rowp + l2, jD);
            n_int += 1;
          }
        }
      }
      __syncthreads();
      if (tid == 0) s_nr = 0;
      __syncthreads();
    }
  }

  // push-down + epilogue, one warp per row
  const int scale_log2 = sum_scale_log2(g.Z * g.Y * g.X, dmax);
  const double scale = ldexp(1.0, scale_log2);
  const int64_t item = b * g.Z * g.Y * g.X;
  uint32_t bad = 0;
  for (int row = warp; row < kRows; row += 8) {
    const int ly = row % TY, lz = row / TY;
    const int64_t gz = oz + lz, gy = oy + ly, gx = ox + lane;
    const bool valid = gz < g.Z && gy < g.Y && gx < g.X;
    const uint32_t* Tr = T + row * kRowStride;
    uint32_t c = Tr[(kLevels - 1) * 32 + lane];
#pragma unroll
    for (int k = kLevels - 2; k >= 0; --k) {
      uint32_t upv = __shfl_up_sync(kFull, c, 1 << k);
      if (lane < (1 << k)) upv = 0;
      c = max(Tr[k * 32 + lane], max(c, upv));
    }
    int32_t L = 0;
    bool shell = false;
    unsigned long long fx = 0;
    if (valid) {
      const int64_t gi = item + (gz * g.Y + gy) * g.X + gx;
      L = __ldg(lab + gi);
      if (L != 0) {
        const uint32_t d = __ldg(Dg + gi);
        if (c < d) bad = 1;
        shell = d == 1;
        const double lt = sqrt((double)c);
        fx = (unsigned long long)__double2ull_rn(lt * scale);
        if (lt2_out) lt2_out[gi] = c;
        if (lt_out) lt_out[gi] = (float)lt;
      }
    }
    if (do_reduce) {
      if (L < 0 || L > acc.max_label) L = 0;
      uint32_t act = __ballot_sync(kFull, L != 0);
      while (act) {
        const int leader = __ffs(act) - 1;
        const int32_t key = __shfl_sync(kFull, L, leader);
        const uint32_t grp = __ballot_sync(kFull, L == key);
        const bool in = (grp >> lane) & 1u;
        const unsigned long long t1 = in ? fx : 0ull, t2 = (in && shell) ? fx : 0ull;
        const uint32_t h1 = __reduce_add_sync(kFull, (uint32_t)(t1 >> 24));
        const uint32_t l1 = __reduce_add_sync(kFull, (uint32_t)(t1 & 0xFFFFFFull));
        const uint32_t h2 = __reduce_add_sync(kFull, (uint32_t)(t2 >> 24));
        const uint32_t l2 = __reduce_add_sync(kFull, (uint32_t)(t2 & 0xFFFFFFull));
        const uint32_t mx = __reduce_max_sync(kFull, in ? c : 0u);
        const uint32_t nsh = __popc(__ballot_sync(kFull, in && shell));
        if (lane == leader) {
          const int64_t id = b * acc.max_label + (key - 1);
          atomicAdd(acc.vol + id, (unsigned long long)__popc(grp));
          if (nsh) atomicAdd(acc.nshell + id, (unsigned long long)nsh);
          atomicAdd(acc.sum + id, ((unsigned long long)h1 << 24) + l1);
          if (nsh) atomicAdd(acc.sumshell + id, ((unsigned long long)h2 << 24) + l2);
          atomicMax(acc.maxlt2 + id, mx);
        }
        act &= ~grp;
      }
    }
  }
  n_int = __reduce_add_sync(kFull, (uint32_t)n_int);
  if (lane == 0 && n_int) atomicAdd(&hdr->n_intervals, n_int);
  if (bad) atomicOr(&hdr->status, kStInternal);
}

}  // namespace

cudaError_t ensure_mtables(int dev) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  DeviceTables& dt = g_tables[dev];
  if (dt.m3) return cudaSuccess;
  // offset tables (shared-memory deltas of the pruning tiles), sorted by class
  {
    std::vector<int> off, cls(kClasses3 + 1, 0);
    using P = PruneTile<true>;
    for (int c = 0; c < kClasses3; ++c) {
      cls[c] = (int)off.size();
      for (int dz = -3; dz <= 3; ++dz)
        for (int dy = -3; dy <= 3; ++dy)
          for (int dx = -3; dx <= 3; ++dx) {
            int a[3] = {abs(dz), abs(dy), abs(dx)};
            if (a[0] < a[1]) std::swap(a[0], a[1]);
            if (a[1] < a[2]) std::swap(a[1], a[2]);
            if (a[0] < a[1]) std::swap(a[0], a[1]);
            if (a[0] == h_rep3[c][0] && a[1] == h_rep3[c][1] && a[2] == h_rep3[c][2])
              off.push_back((dz * P::PY + dy) * P::PX + dx);
          }
    }
    cls[kClasses3] = (int)off.size();
    if (off.size() != 178) return cudaErrorUnknown;
    cudaError_t e = cudaMemcpyToSymbol(c_off3, off.data(), sizeof(int) * off.size());
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_cls3, cls.data(), sizeof(int) * cls.size());
    if (e != cudaSuccess) return e;
  }
  {
    std::vector<int> off, cls(kClasses2 + 1, 0);
    using P = PruneTile<false>;
    for (int c = 0; c < kClasses2; ++c) {
      cls[c] = (int)off.size();
      for (int dy = -2; dy <= 2; ++dy)
        for (int dx = -2; dx <= 2; ++dx) {
          int a0 = abs(dy), a1 = abs(dx);
          if (a0 < a1) std::swap(a0, a1);
          if (a0 == h_rep2[c][0] && a1 == h_rep2[c][1]) off.push_back(dy * P::PX + dx);
        }
    }
    cls[kClasses2] = (int)off.size();
    if (off.size() != 24) return cudaErrorUnknown;
    cudaError_t e = cudaMemcpyToSymbol(c_off2, off.data(), sizeof(int) * off.size());
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_cls2, cls.data(), sizeof(int) * cls.size());
    if (e != cudaSuccess) return e;
  }
  uint32_t *m3 = nullptr, *m2 = nullptr;
  cudaError_t e = cudaMalloc(&m3, sizeof(uint32_t) * kClasses3 * (kDcap3 + 1));
  if (e == cudaSuccess) e = cudaMalloc(&m2, sizeof(uint32_t) * kClasses2 * (kDcap2 + 1));
  if (e != cudaSuccess) {
    cudaFree(m3);
    return e;
  }
  const int64_t n3 = (int64_t)kClasses3 * (kDcap3 + 1), n2 = (int64_t)kClasses2 * (kDcap2 + 1);
  k_mtable3<<<(unsigned)((n3 + 127) / 128), 128>>>(m3);
  k_mtable2<<<(unsigned)((n2 + 127) / 128), 128>>>(m2);
  e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFree(m3);
    cudaFree(m2);
    return e;
  }
  cudaFuncSetAttribute(k_dilate<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRows * kRowStride * 4);
  cudaFuncSetAttribute(k_dilate<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRows * kRowStride * 4);
  dt.m3 = m3;
  dt.m2 = m2;
  return cudaSuccess;
}

void release_mtables() {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& dt : g_tables) {
    if (dt.m3) cudaFree(dt.m3);
    if (dt.m2) cudaFree(dt.m2);
    dt.m3 = dt.m2 = nullptr;
  }
}

const uint32_t* mtable_ptr(int dev, bool is3d) { return is3d ? g_tables[dev].m3 : g_tables[dev].m2; }

void launch_prune(const uint32_t* D, const Geom& g, TileMeta* meta, uint2* centres, WsHeader* hdr,
                  cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (g.ndim == 3)
    k_prune<true><<<(unsigned)g.ntiles, 256, 0, st>>>(D, g, meta, centres, mtable_ptr(dev, true), hdr);
  else
    k_prune<false><<<(unsigned)g.ntiles, 256, 0, st>>>(D, g, meta, centres, mtable_ptr(dev, false), hdr);
}

void launch_dilate(const int32_t* labels, const uint32_t* D, const TileMeta* meta, const uint2* centres,
                   const Geom& g, const Accum* acc, uint32_t* lt2_out, float* lt_out, WsHeader* hdr,
                   cudaStream_t st) {
  Accum a{};
  if (acc) a = *acc;
  const size_t smem = (size_t)kRows * kRowStride * 4;
  if (g.ndim == 3)
    k_dilate<true><<<(unsigned)g.ntiles, 256, smem, st>>>(labels, D, meta, centres, g, a, acc ? 1 : 0, lt2_out,
                                                           lt_out, hdr);
  else
    k_dilate<false><<<(unsigned)g.ntiles, 256, smem, st>>>(labels, D, meta, centres, g, a, acc ? 1 : 0, lt2_out,
                                                            lt_out, hdr);
}

}  // namespace fastrs
