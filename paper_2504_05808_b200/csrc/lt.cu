// K5 fallback: ball dilation with a shared reverse sparse table and shared-memory atomics.
//   LT^2(p) = max{ D(q) : |p-q|^2 < D(q) }  ("radius of the largest circle/sphere
//   that fits in the object at any point", §4; strict membership, reading c5).
// One CTA per output tile gathers the kept centres of every home tile whose max ball can
// reach it; every centre emits, per intersected x-row of the tile, the interval
// |x - qx| <= isqrt(D-1-dy^2-dz^2), which costs two atomicMax into the row's reverse sparse
// table (level k = floor(log2(r-l+1)), cells l and r-2^k+1); a shuffle push-down over the 6
// levels yields LT^2 of the row.  Used only when Dmax > 65535 (the default kernel in
// dilate.cu stores u16 values) or for tiles the default kernel hands over (a single D bucket
// with more candidates than its list capacity).  Same fused epilogue (dilate_common.cuh).
#include "common.cuh"
#include "dilate_common.cuh"

namespace fastrs {
namespace {

__device__ __forceinline__ int isqrt_i(int h) {
  int w = (int)sqrtf((float)h);
  while (w * w > h) --w;
  while ((w + 1) * (w + 1) <= h) ++w;
  return w;
}

// ---------------------------------------------------------------------------------------
// K5: dilation (reverse sparse tables) + shell + per-label reductions
// ---------------------------------------------------------------------------------------
constexpr int kRcap = 1024;

template <bool IS3D>
__device__ __forceinline__ void dilate_tile_atomic(int64_t tile, const TileMeta* __restrict__ meta,
                                                   const uint2* __restrict__ cent, const Geom& g,
                                                   uint32_t* __restrict__ ltp, WsHeader* __restrict__ hdr, uint32_t* T,
                                                   uint32_t* s_rt, uint32_t* s_rpre, int& s_nr) {
  constexpr int TY = IS3D ? 8 : 64, TZ = IS3D ? 8 : 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t t = tile;
  const int64_t tx = t % g.ntx;
  t /= g.ntx;
  const int64_t ty = t % g.nty;
  t /= g.nty;
  const int64_t tz = t % g.ntz;
  const int64_t b = t / g.ntz;
  if (tz < g.tz_lo || tz >= g.tz_hi) return;  // slab path: halo tiles only feed the gather (uniform)
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

  // push-down, one warp per row -> the LT plane
  const int64_t item = b * g.Z * g.Y * g.X;
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
    if (valid) {  // the LT plane is u16 when Dmax <= 65535 (K5b writes it too), else u32
      const int64_t gi = item + (gz * g.Y + gy) * g.X + gx;
      if (hdr->dmax > kU16Max) ltp[gi] = c; else reinterpret_cast<uint16_t*>(ltp)[gi] = (uint16_t)c;
    }
  }
  n_int = __reduce_add_sync(kFull, (uint32_t)n_int);
  if (lane == 0 && n_int) atomicAdd(&hdr->n_intervals, n_int);
}

// Grid-stride over the work: every tile when Dmax > 65535 (the exact-order kernel stores u16
// values and leaves everything here), else the tiles it listed in fbl (hdr->n_fb of them).
template <bool IS3D>
__global__ void __launch_bounds__(256) k_dilate_atomic(const TileMeta* __restrict__ meta, const uint2* __restrict__ cent,
                                                Geom g, const uint32_t* __restrict__ fbl, uint32_t* __restrict__ ltp,
                                                WsHeader* __restrict__ hdr) {
  extern __shared__ uint32_t T[];  // kRows * kRowStride
  __shared__ uint32_t s_rt[kRcap];
  __shared__ uint32_t s_rpre[kRcap + 1];
  __shared__ int s_nr;
  const bool all = hdr->dmax > kU16Max;
  const int64_t nitems = all ? g.ntiles : (int64_t)hdr->n_fb;
  for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int64_t tile = all ? it : (int64_t)fbl[it];
    if (meta[tile].nfg != 0) dilate_tile_atomic<IS3D>(tile, meta, cent, g, ltp, hdr, T, s_rt, s_rpre, s_nr);
    __syncthreads();  // shared memory is reused by the next tile
  }
}


// ---------------------------------------------------------------------------------------
// K5 epilogue (streaming): per element LT^2 from the LT plane, shell (D == 1), LT outputs and
// optionally the per-label reductions (a7); one warp per x-row, 8 chunks of 32 elements in
// flight.  The S&R path does not use it: its reductions are fused into the paint.
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_epilogue(const int32_t* __restrict__ lab, const uint32_t* __restrict__ Dg,
                                                  const uint32_t* __restrict__ ltp, Geom g, int64_t z_lo, int64_t nz,
                                                  Accum acc, int do_reduce, uint32_t* __restrict__ lt2_out,
                                                  float* __restrict__ lt_out, const unsigned long long* __restrict__ fxlut,
                                                  WsHeader* __restrict__ hdr) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= g.B * nz * g.Y) return;
  const int64_t y = row % g.Y, zb = row / g.Y, z = z_lo + zb % nz, b = zb / nz;
  const int64_t base = ((b * g.Z + z) * g.Y + y) * g.X;
  const bool wide = hdr->dmax > kU16Max;  // LT plane element type: u32 if wide, else u16
  const uint16_t* ltp16 = reinterpret_cast<const uint16_t*>(ltp);
  const int X = (int)g.X;
  uint32_t bad = 0;
  constexpr int kEpiChunks = 8;  // 32-element chunks in flight per warp
  for (int x0 = 0; x0 < X; x0 += 32 * kEpiChunks) {
    int32_t L[kEpiChunks];
    uint32_t d[kEpiChunks], c[kEpiChunks];
#pragma unroll
    for (int k = 0; k < kEpiChunks; ++k) {
      const int x = x0 + 32 * k + lane;
      const bool in = x < X;
      L[k] = in ? __ldg(lab + base + x) : 0;
      d[k] = in ? __ldg(Dg + base + x) : 0u;
      c[k] = (in && L[k] != 0) ? (wide ? __ldg(ltp + base + x) : (uint32_t)__ldg(ltp16 + base + x)) : 0u;
    }
#pragma unroll
    for (int k = 0; k < kEpiChunks; ++k) {
      if (x0 + 32 * k >= X) break;  // warp-uniform
      bad |= row_epilogue_v(c[k], L[k], d[k], lane, base + x0 + 32 * k + lane, b, acc, do_reduce, lt2_out, lt_out,
                            fxlut);
    }
  }
  if (__any_sync(kFull, bad) && lane == 0) atomicOr(&hdr->status, kStInternal);
}

// Per-label reductions of the tiles painted by the atomic fallback kernel (grid-stride over
// the same work list as k_dilate_atomic): one CTA per tile, one warp per row, lane = x.
template <bool IS3D>
__global__ void __launch_bounds__(256) k_epilogue_fallback(const int32_t* __restrict__ lab, const uint32_t* __restrict__ Dg,
                                                           const uint32_t* __restrict__ ltp,
                                                           const TileMeta* __restrict__ meta,
                                                           const uint32_t* __restrict__ fbl, Geom g, Accum acc,
                                                           const unsigned long long* __restrict__ fxlut,
                                                           WsHeader* __restrict__ hdr) {
  constexpr int TY = IS3D ? 8 : 64, TZ = IS3D ? 8 : 1;
  const bool wide = hdr->dmax > kU16Max;
  const int64_t nitems = wide ? g.ntiles : (int64_t)hdr->n_fb;
  const uint16_t* ltp16 = reinterpret_cast<const uint16_t*>(ltp);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t bad = 0;
  for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int64_t tile = wide ? it : (int64_t)fbl[it];
    int64_t t = tile;
    const int64_t tx = t % g.ntx;
    t /= g.ntx;
    const int64_t ty = t % g.nty;
    t /= g.nty;
    const int64_t tz = t % g.ntz;
    const int64_t b = t / g.ntz;
    if (tz < g.tz_lo || tz >= g.tz_hi || meta[tile].nfg == 0) continue;  // (block-uniform)
    for (int row = warp; row < kRows; row += 8) {
      const int64_t gz = tz * TZ + row / TY, gy = ty * TY + row % TY, gx = tx * kTX + lane;
      const bool in = gz < g.Z && gy < g.Y && gx < g.X;
      const int64_t gi = ((b * g.Z + gz) * g.Y + gy) * g.X + gx;
      const int32_t L = in ? __ldg(lab + gi) : 0;
      const uint32_t d = in ? __ldg(Dg + gi) : 0u;
      const uint32_t c = (in && L != 0) ? (wide ? __ldg(ltp + gi) : (uint32_t)__ldg(ltp16 + gi)) : 0u;
      bad |= row_epilogue_v(c, L, d, lane, gi, b, acc, 1, nullptr, nullptr, fxlut);
    }
  }
  if (__any_sync(kFull, bad) && lane == 0) atomicOr(&hdr->status, kStInternal);
}

}  // namespace

cudaError_t dilate_atomic_setup() {
  cudaError_t e = cudaFuncSetAttribute(k_dilate_atomic<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kRows * kRowStride * 4);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_dilate_atomic<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRows * kRowStride * 4);
  return e;
}

void launch_dilate_fallback(TileMeta* meta, const uint2* centres, const uint32_t* fbl, const Geom& g, uint32_t* ltp,
                            WsHeader* hdr, cudaStream_t st) {
  const size_t smem = (size_t)kRows * kRowStride * 4;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)(g.ntiles < (int64_t)nsm * 4 ? g.ntiles : (int64_t)nsm * 4);
  if (g.ndim == 3)
    k_dilate_atomic<true><<<grid, 256, smem, st>>>(meta, centres, g, fbl, ltp, hdr);
  else
    k_dilate_atomic<false><<<grid, 256, smem, st>>>(meta, centres, g, fbl, ltp, hdr);
}

void launch_epilogue(const int32_t* labels, const uint32_t* D, const Geom& g, const Accum* acc, uint32_t* lt2_out,
                     float* lt_out, const uint32_t* ltp, WsHeader* hdr, cudaStream_t st) {
  Accum a{};
  if (acc) a = *acc;
  int dev = 0;
  cudaGetDevice(&dev);
  const int TZ = g.ndim == 3 ? kTZ3 : 1;
  const int64_t z_lo = g.tz_lo * TZ, z_hi = g.tz_hi * TZ < g.Z ? g.tz_hi * TZ : g.Z;
  const int64_t rows = g.B * (z_hi - z_lo) * g.Y;
  if (rows > 0)
    k_epilogue<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(labels, D, ltp, g, z_lo, z_hi - z_lo, a, acc ? 1 : 0, lt2_out,
                                                          lt_out, device_fxlut(dev), hdr);
}

void launch_epilogue_fallback(const int32_t* labels, const uint32_t* D, const TileMeta* meta, const uint32_t* fbl,
                              const Geom& g, const Accum& acc, const uint32_t* ltp, WsHeader* hdr, cudaStream_t st) {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)(g.ntiles < (int64_t)nsm * 8 ? g.ntiles : (int64_t)nsm * 8);
  if (g.ndim == 3)
    k_epilogue_fallback<true><<<grid, 256, 0, st>>>(labels, D, ltp, meta, fbl, g, acc, device_fxlut(dev), hdr);
  else
    k_epilogue_fallback<false><<<grid, 256, 0, st>>>(labels, D, ltp, meta, fbl, g, acc, device_fxlut(dev), hdr);
}

}  // namespace fastrs
