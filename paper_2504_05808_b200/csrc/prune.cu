// K7 lattice containment table and K4 exact maximal-ball pruning.
//
// Ball of q: B(q) = { p : |p-q|^2 <= D(q) - 1 } (strict membership, reading c5).  For a
// neighbour offset s, B(q) is contained in B(q+s) exactly when
//     D(q+s) > M(D(q), s),   M(D, s) = max_{u in Z^n, |u|^2 <= D-1} |u - s|^2,
// because every lattice point of B(q) is then within B(q+s).  Containment between balls of
// different centres is strict (two lattice balls with different centres are never equal
// sets), and strict containment is a strict partial order, so every dropped ball lies in
// a kept maximal ball with a larger D and LT^2 (max over covering balls) is unchanged.
// M depends on s only through its class (the ball is symmetric under sign changes and axis
// permutations): 3D 26-neighbourhood classes (1,0,0), (1,1,0), (1,1,1); 2D (1,0), (1,1).
// The table is built once per device for D <= kDcap; centres with a larger D are kept.
//
// K4 is row-vectorised: one warp per tile row, lane = x, every lane tests the same offset
// (warp-uniform, shared-memory reads conflict-free); survivors are compacted per home tile
// in element order with the tile's count / max D / #foreground (TileMeta).
#include <cuda.h>

#include <mutex>

#include "common.cuh"

namespace fastrs {
namespace {

constexpr unsigned kFullMask = 0xFFFFFFFFu;

// offset classes (canonical |s| sorted descending), by |s|^2: stage 1 = the first 3 (3D) / 2 (2D)
__constant__ int c_rep3[kClasses3][3] = {{1, 0, 0}, {1, 1, 0}, {1, 1, 1}, {2, 0, 0}, {2, 1, 0}, {2, 1, 1},
                                         {2, 2, 0}, {2, 2, 1}, {3, 0, 0}, {3, 1, 0}, {3, 1, 1}, {2, 2, 2}};
__constant__ int c_rep2[kClasses2][2] = {{1, 0}, {1, 1}, {2, 0}, {2, 1}, {2, 2}};
// class index (position in c_rep3 / c_rep2) of an offset, -1 if |s|^2 > 12 / 8 or s = 0
__host__ __device__ constexpr int class3(int dz, int dy, int dx) {
  const int a = dz < 0 ? -dz : dz, b = dy < 0 ? -dy : dy, c = dx < 0 ? -dx : dx;
  const int hi = a > b ? (a > c ? a : c) : (b > c ? b : c);
  const int lo = a < b ? (a < c ? a : c) : (b < c ? b : c);
  const int mid = a + b + c - hi - lo;
  const int key = hi * 100 + mid * 10 + lo;
  return key == 100 ? 0 : key == 110 ? 1 : key == 111 ? 2 : key == 200 ? 3 : key == 210 ? 4 : key == 211 ? 5 :
         key == 220 ? 6 : key == 221 ? 7 : key == 300 ? 8 : key == 310 ? 9 : key == 311 ? 10 : key == 222 ? 11 : -1;
}
__host__ __device__ constexpr int class2(int dy, int dx) {
  const int a = dy < 0 ? -dy : dy, b = dx < 0 ? -dx : dx;
  const int hi = a > b ? a : b, lo = a > b ? b : a;
  const int key = hi * 10 + lo;
  return key == 10 ? 0 : key == 11 ? 1 : key == 20 ? 2 : key == 21 ? 3 : key == 22 ? 4 : -1;
}

__device__ __forceinline__ int isqrt_t(int h) {
  int w = (int)sqrtf((float)h);
  while (w * w > h) --w;
  while ((w + 1) * (w + 1) <= h) ++w;
  return w;
}

// M(D, s) for the 3D classes (s0 >= s1 >= s2 >= 0): for each (u0,u1) in the disk the best u2
// is -w (w = isqrt of the remaining radius^2), which maximises (u2 - s2)^2.
__global__ void k_mtable3(uint32_t* M) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)kClasses3 * (kDcap3 + 1)) return;
  const int c = (int)(t / (kDcap3 + 1)), D = (int)(t % (kDcap3 + 1));
  if (D == 0) {
    M[t] = 0;
    return;
  }
  const int s0 = c_rep3[c][0], s1 = c_rep3[c][1], s2 = c_rep3[c][2];
  const int R2 = D - 1, r = isqrt_t(R2);
  uint32_t best = 0;
  for (int u0 = -r; u0 <= r; ++u0) {
    const int rem0 = R2 - u0 * u0, r1 = isqrt_t(rem0);
    for (int u1 = -r1; u1 <= r1; ++u1) {
      const int w = isqrt_t(rem0 - u1 * u1);
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
  const int R2 = D - 1, r = isqrt_t(R2);
  uint32_t best = 0;
  for (int u0 = -r; u0 <= r; ++u0) {
    const int w = isqrt_t(R2 - u0 * u0);
    const uint32_t v = (u0 - s0) * (u0 - s0) + (w + s1) * (w + s1);
    best = v > best ? v : best;
  }
  M[t] = best;
}

// fixed-point sqrt table of the LT sums: fx(c) = round(sqrt(c) * 2^32), c < kFxLut
__global__ void k_fxtable(unsigned long long* fx) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < kFxLut) fx[c] = (unsigned long long)__double2ull_rn(sqrt((double)c) * kFxScale);
}

struct DeviceTables {
  uint32_t* m3 = nullptr;
  uint4* m3s1 = nullptr;
  uint32_t* m2 = nullptr;
  unsigned long long* fx = nullptr;
};
std::mutex g_mu;
DeviceTables g_tables[64];

// 4-byte asynchronous global->shared copy; writes zero when !valid
__device__ __forceinline__ void cp_async4_zfill(uint32_t* smem, const uint32_t* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 4 : 0) : "memory");
}

// 16-byte asynchronous global->shared copy (both 16-byte aligned); zeros when !valid
__device__ __forceinline__ void cp_async16_zfill(uint32_t* smem, const uint32_t* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 16 : 0) : "memory");
}

template <bool IS3D>
struct PruneTile {
  static constexpr int H = IS3D ? 3 : 2;  // halo: |s_i| <= 3 (3D, |s|^2 <= 12) / 2 (2D, |s|^2 <= 8)
  static constexpr int TY = IS3D ? 8 : 64, TZ = IS3D ? 8 : 1;
  static constexpr int HX = 4;  // x halo of the staged rows: 4 (>= H) keeps rows 16-byte aligned
  static constexpr int PX = kTX + 2 * HX, PY = TY + 2 * H, PZ = IS3D ? TZ + 2 * H : 1;
  static constexpr int HZ = IS3D ? H : 0;
  static constexpr int NC = IS3D ? kClasses3 : kClasses2;   // classes
  static constexpr int C1 = IS3D ? 3 : 2;                   // stage-1 classes
};


// Stage-2 stripes: warp w takes the survivor slots w*32 + 256*j + l (l < 32) of the CTA-wide
// survivor list and compacts the ones it keeps in place into the same stripe (the k-th kept
// entry lands at or before the slot it was read from, and no other warp touches the stripe), so
// the bucket scatter needs no second pass over rows and no cross-warp prefix.
// stage-2 class order (3D): (2,1,0), (2,1,1), (2,2,1), (3,1,1), (3,1,0), then the classes that
// dropped no stage-1 survivor on C4: (2,0,0), (2,2,0), (3,0,0), (2,2,2)
#ifndef FASTRS_PRUNE_FAST_CLASSES
#define FASTRS_PRUNE_FAST_CLASSES 5
#endif
constexpr int kPruneFastClasses3 = FASTRS_PRUNE_FAST_CLASSES;  // stage-2 classes tested by default (3D)
__host__ __device__ constexpr int stage2_order3(int q) {
  return q == 0 ? 4 : q == 1 ? 5 : q == 2 ? 7 : q == 3 ? 10 : q == 4 ? 9 : q == 5 ? 3 : q == 6 ? 6 : q == 7 ? 8 : 11;
}

__device__ __forceinline__ int stripe_slot(int warp, int k) { return warp * 32 + ((k >> 5) << 8) + (k & 31); }

template <bool IS3D, bool TMA>
__global__ void __launch_bounds__(256, 6) k_prune(const uint32_t* __restrict__ D, Geom g, TileMeta* __restrict__ meta,
                                               uint2* __restrict__ cent, uint32_t* __restrict__ fgm,
                                               uint32_t* __restrict__ shm, uint16_t* __restrict__ oct,
                                               const uint32_t* __restrict__ M, const uint4* __restrict__ M1,
                                               int64_t tile0, WsHeader* __restrict__ hdr,
                                               const __grid_constant__ CUtensorMap tmap, FastDiv dx, FastDiv dy,
                                               FastDiv dz, int nc2, int pf_ahead) {
  using P = PruneTile<IS3D>;
  __shared__ __align__(128) uint32_t s[P::PZ * P::PY * P::PX];
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ uint32_t red_cnt[8], red_max[8];
  __shared__ uint16_t surv[kTileVol];
  __shared__ uint32_t s_nsurv, s_nkept;
  __shared__ uint32_t bhist[128];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const int64_t tile = tile0 + blockIdx.x;
  // tile -> (tx, ty, tz, b) in 32-bit arithmetic (ntiles < 2^32, checked in make_geom)
  uint32_t t = (uint32_t)tile, r;
  t = dx.divmod(t, r);
  const int64_t tx = r;
  t = dy.divmod(t, r);
  const int64_t ty = r;
  t = dz.divmod(t, r);
  const int64_t tz = r;
  const int64_t b = t;
  const int64_t z0 = tz * P::TZ - P::HZ, y0 = ty * P::TY - P::H, x0 = tx * kTX - P::HX;
  const uint32_t* Db = D + b * g.Z * g.Y * g.X;
  for (int k = tid; k < 128; k += 256) bhist[k] = 0;
  if (tid == 0) s_nsurv = 0;
  // halo staging with cp.async (zero-fill outside the grid), one warp per (z, y) row of the
  // padded tile.  Rows are 40 words starting at a multiple of 4, so when X % 4 == 0 every
  // 16-byte chunk lies entirely inside or outside the grid: 10 chunk copies per row.
  if constexpr (TMA) {
    // one tensor-memory-accelerator copy of the whole padded box; elements outside the grid
    // arrive as zeros (the tensor map's out-of-bounds fill), same as the cp.async path
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&s_bar);
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar),
                   "r"((unsigned)sizeof(s))
                   : "memory");
      const unsigned dst = (unsigned)__cvta_generic_to_shared(s);
      if constexpr (IS3D) {
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4, %5}], [%6];\n" ::"r"(dst),
            "l"(&tmap), "r"((int)x0), "r"((int)y0), "r"((int)z0), "r"((int)b), "r"(bar)
            : "memory");
        // round 2c: warm L2 with the halo box of the tile a CTA launched ~one residency later will
        // stage (CTAs start in index order), so its copy waits on L2 rather than on DRAM
        if (pf_ahead > 0 && blockIdx.x + pf_ahead < gridDim.x) {
          uint32_t pq = (uint32_t)(tile + pf_ahead), pr;
          pq = dx.divmod(pq, pr);
          const int px = (int)pr * kTX - P::HX;
          pq = dy.divmod(pq, pr);
          const int py = (int)pr * P::TY - P::H;
          pq = dz.divmod(pq, pr);
          const int pz = (int)pr * P::TZ - P::HZ;
          asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];\n" ::"l"(&tmap), "r"(px),
                       "r"(py), "r"(pz), "r"((int)pq)
                       : "memory");
        }
      } else
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4}], [%5];\n" ::"r"(dst),
            "l"(&tmap), "r"((int)x0), "r"((int)y0), "r"((int)b), "r"(bar)
            : "memory");
    }
    __syncthreads();  // the barrier is initialised before anyone polls it
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            bar)
        : "memory");
  } else {
    const int Zi = (int)g.Z, Yi = (int)g.Y, Xi = (int)g.X;
    constexpr int kRowsPZ = P::PZ * P::PY;
    if ((Xi & 3) == 0) {
      for (int i = tid; i < kRowsPZ * (P::PX / 4); i += 256) {
        const int r = i / (P::PX / 4), j = i - r * (P::PX / 4);
        const int lz = r / P::PY, ly = r - lz * P::PY;
        const int gz = (int)z0 + lz, gy = (int)y0 + ly, gx = (int)x0 + 4 * j;
        const bool ok = (unsigned)gz < (unsigned)Zi && (unsigned)gy < (unsigned)Yi && (unsigned)gx < (unsigned)Xi;
        const uint32_t* src = ok ? Db + ((int64_t)gz * Yi + gy) * Xi + gx : Db;
        cp_async16_zfill(&s[r * P::PX + 4 * j], src, ok);
      }
    } else {
      for (int r = warp; r < kRowsPZ; r += 8) {
        const int lz = r / P::PY, ly = r - lz * P::PY;
        const int gz = (int)z0 + lz, gy = (int)y0 + ly;
        const bool rowok = (unsigned)gz < (unsigned)Zi && (unsigned)gy < (unsigned)Yi;
        const uint32_t* src = Db + ((int64_t)(rowok ? gz : 0) * Yi + (rowok ? gy : 0)) * Xi;
#pragma unroll
        for (int k = 0; k < (P::PX + 31) / 32; ++k) {
          const int lx = lane + 32 * k;
          if (lx < P::PX) {
            const int gx = (int)x0 + lx;
            const bool ok = rowok && (unsigned)gx < (unsigned)Xi;
            cp_async4_zfill(&s[r * P::PX + lx], ok ? src + gx : Db, ok);
          }
        }
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  }
  __syncthreads();

  // Both staging paths zero-fill outside the grid, so "foreground" is D != 0 (cells of the
  // tile beyond the grid edge read 0), and neighbours outside the grid read 0 (never contain).
  constexpr int dcap = IS3D ? kDcap3 : kDcap2;
  {
    // a tile without foreground (C4: 21 % of the tiles) writes empty outputs and leaves
    bool any = false;
#pragma unroll
    for (int k = 0; k < kTileVol / 256; ++k) {
      const int v = tid + 256 * k;
      const int lx = v & 31, ly = (v >> 5) % P::TY, lz = v / (32 * P::TY);
      any |= s[((lz + P::HZ) * P::PY + (ly + P::H)) * P::PX + (lx + P::HX)] != 0u;
    }
    if (!__syncthreads_or(any)) {
      if (tid < kRows) {
        shm[tile * kRows + tid] = 0u;
        fgm[tile * kRows + tid] = 0u;
      } else if (tid < kRows + kOctPerTile) {
        oct[tile * kOctPerTile + (tid - kRows)] = 0;
      } else if (tid == kRows + kOctPerTile) {
        meta[tile] = TileMeta{0u, 0u, 0u, 0u};
      }
      return;
    }
  }
  uint32_t nfg = 0, maxd = 0;
  // stage-1 survivors are appended to the CTA-wide list (one shared atomic per warp row; the
  // list order does not matter: the output is sorted by D bucket, arbitrary inside a bucket)
  auto emit_row = [&](int row, uint32_t d, bool keep) {
    const bool fg = d != 0;
    const uint32_t fgb = __ballot_sync(kFullMask, fg);
    if (fgb == 0u) {  // a background row (C4: 43 % of the rows)
      if (lane == 0) {
        shm[tile * kRows + row] = 0u;
        fgm[tile * kRows + row] = 0u;
      }
      return;
    }
    // shell <=> D == 1 (a face neighbour or the flagged border is a site):
    // the per-row shell mask for the fused reductions of K5; the foreground mask for its coverage
    const uint32_t shb = __ballot_sync(kFullMask, d == 1u);
    const uint32_t kb = __ballot_sync(kFullMask, keep);
    uint32_t base = 0;
    if (lane == 0) {
      shm[tile * kRows + row] = shb;
      fgm[tile * kRows + row] = fgb;
      if (kb) base = atomicAdd(&s_nsurv, (uint32_t)__popc(kb));
    }
    base = __shfl_sync(kFullMask, base, 0);
    if (keep) surv[base + __popc(kb & lt_mask)] = (uint16_t)(row * 32 + lane);
    nfg += fg;
  };
  if constexpr (IS3D) {
    // ---- stage 1 (the 26-neighbourhood), warp = one y row of the tile, lane = x, a sliding
    // window over z.  The per-class maxima are separable: per layer z', over the 3x3 (x, y)
    // neighbourhood, a0 = centre, a1 = max of the 4 edge-adjacent, a2 = max of the 4 corners;
    // then over z: class (1,0,0) = max(a1(z), a0(z-1), a0(z+1)), class (1,1,0) = max(a2(z),
    // a1(z-1), a1(z+1)), class (1,1,1) = max(a2(z-1), a2(z+1)): 9 shared loads per layer, each
    // layer serving three rows, instead of 26 per row.
    constexpr int SZ = P::PY * P::PX;
    const int cb = (P::HZ * P::PY + (warp + P::H)) * P::PX + (lane + P::HX);  // (x=lane, y=warp, z=0)
    auto layer = [&](int lz, uint32_t& a0, uint32_t& a1, uint32_t& a2) {
      const uint32_t* q = s + cb + lz * SZ;
      a0 = q[0];
      a1 = max(max(q[-1], q[1]), max(q[-P::PX], q[P::PX]));
      a2 = max(max(q[-P::PX - 1], q[-P::PX + 1]), max(q[P::PX - 1], q[P::PX + 1]));
    };
    uint32_t p0, p1, p2, q0, q1, q2;
    layer(-1, p0, p1, p2);
    layer(0, q0, q1, q2);
    uint4 mq = (q0 != 0u && q0 <= (uint32_t)dcap) ? __ldg(M1 + q0) : make_uint4(~0u, ~0u, ~0u, ~0u);
#pragma unroll
    for (int lz = 0; lz < P::TZ; ++lz) {
      uint32_t n0, n1, n2;
      layer(lz + 1, n0, n1, n2);
      // the next row's thresholds, one row ahead (their latency overlaps this row)
      const uint4 mn = (lz + 1 < P::TZ && n0 != 0u && n0 <= (uint32_t)dcap) ? __ldg(M1 + n0)
                                                                            : make_uint4(~0u, ~0u, ~0u, ~0u);
      const uint32_t c0 = max(q1, max(p0, n0)), c1 = max(q2, max(p1, n1)), c2 = max(p2, n2);
      const bool keep = q0 != 0u && c0 <= mq.x && c1 <= mq.y && c2 <= mq.z;
      emit_row(warp + 8 * lz, q0, keep);
      p0 = q0, p1 = q1, p2 = q2;
      q0 = n0, q1 = n1, q2 = n2;
      mq = mn;
    }
  } else {
    // ---- stage 1 (2D: the 8-neighbourhood), row-vectorised; thresholds fetched first
    constexpr int kRowsPerWarp = kRows / 8;
    uint32_t dr[kRowsPerWarp], m0r[kRowsPerWarp], m1r[kRowsPerWarp];
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
      const int row = warp + 8 * k;
      const int c = (row + P::H) * P::PX + (lane + P::HX);
      const uint32_t d = s[c];
      dr[k] = d;
      const bool test = d != 0u && d <= (uint32_t)dcap;
      m0r[k] = test ? __ldg(M + d) : 0xFFFFFFFFu;
      m1r[k] = test ? __ldg(M + (dcap + 1) + d) : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
      const int row = warp + 8 * k;
      const int c = (row + P::H) * P::PX + (lane + P::HX);
      const uint32_t d = dr[k];
      const uint32_t e1 = max(max(s[c - 1], s[c + 1]), max(s[c - P::PX], s[c + P::PX]));
      const uint32_t e2 = max(max(s[c - P::PX - 1], s[c - P::PX + 1]), max(s[c + P::PX - 1], s[c + P::PX + 1]));
      emit_row(row, d, d != 0u && e1 <= m0r[k] && e2 <= m1r[k]);
    }
  }
  __syncthreads();
  // ---- stage 2: the remaining offsets (|s|^2 <= 12 / 8) on the stage-1 survivors, lanes =
  // survivors (warp-uniform offset loop, early exit per class); the kept ones are counted in
  // the D-bucket histogram and compacted in place in the warp's stripe
  const int nsurv = (int)s_nsurv;
  int nk = 0;  // kept by this warp (warp-uniform)
#pragma unroll 1
  for (int j0 = 0; warp * 32 + j0 < nsurv; j0 += 256) {
    const int i = warp * 32 + j0 + lane;
    // (lanes without a survivor test the first core element: every offset stays inside the block)
    int v = 0, c = (P::HZ * P::PY + P::H) * P::PX + P::HX;
    uint32_t d = 0;
    bool keep = false;
    if (i < nsurv) {
      v = surv[i];
      const int lx = v & 31, ly = (v >> 5) % P::TY, lz = v / (32 * P::TY);
      c = ((lz + P::HZ) * P::PY + (ly + P::H)) * P::PX + (lx + P::HX);
      d = s[c];
      keep = true;
    }
    const bool test = keep && d <= (uint32_t)dcap;
    uint32_t mv[IS3D ? 12 : P::NC - P::C1];
    if constexpr (IS3D) {
      // the 9 stage-2 thresholds of D interleaved in three 16-byte words
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const uint4 m4 = test ? __ldg(M1 + (kDcap3 + 1) + 3 * d + j) : make_uint4(~0u, ~0u, ~0u, ~0u);
        mv[4 * j] = m4.x, mv[4 * j + 1] = m4.y, mv[4 * j + 2] = m4.z, mv[4 * j + 3] = m4.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < P::NC - P::C1; ++q) mv[q] = test ? __ldg(M + (P::C1 + q) * (dcap + 1) + d) : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int q = 0; q < P::NC - P::C1; ++q) {
      if (q >= nc2) break;  // (warp-uniform) the classes this launch tests
      if (!__any_sync(kFullMask, test && keep)) break;
      // all offsets of class `cls` (the class test folds at compile time after unrolling): their
      // max against the class threshold.  Only lanes still alive load (the stage is bound by
      // shared-memory wavefronts), and the classes go in the order that drops most centres
      // first (tools/prune_stats.py on C4; the kept set does not depend on the order).
      const int cls = IS3D ? stage2_order3(q) : P::C1 + q;
      if (test && keep) {
        uint32_t mxk = 0;
        if (IS3D) {
#pragma unroll
          for (int dz = -3; dz <= 3; ++dz)
#pragma unroll
            for (int dy = -3; dy <= 3; ++dy)
#pragma unroll
              for (int dx = -3; dx <= 3; ++dx)
                if (class3(dz, dy, dx) == cls) mxk = max(mxk, s[c + (dz * P::PY + dy) * P::PX + dx]);
        } else {
#pragma unroll
          for (int dy = -2; dy <= 2; ++dy)
#pragma unroll
            for (int dx = -2; dx <= 2; ++dx)
              if (class2(dy, dx) == cls) mxk = max(mxk, s[c + dy * P::PX + dx]);
        }
        keep = mxk <= mv[cls - P::C1];
      }
    }
    const uint32_t kb = __ballot_sync(kFullMask, keep);
    __syncwarp();  // every lane has read its slot before the compaction overwrites slots <= it
    if (keep) {
      surv[stripe_slot(warp, nk + __popc(kb & lt_mask))] = (uint16_t)v;
      atomicAdd(&bhist[dbucket(d)], 1u);
      maxd = max(maxd, d);
    }
    nk += __popc(kb);
  }
  // ---- compaction sorted by D bucket (descending; order inside a bucket is arbitrary): the
  // dilation's gather stops scanning a home tile once its remaining balls cannot reach the
  // output tile.  Histogram (stage 2) -> warp-0 descending exclusive scan -> scatter.
  auto centre_d = [&](int v) {
    const int lx = v & 31, ly = (v >> 5) % P::TY, lz = v / (32 * P::TY);
    return s[((lz + P::HZ) * P::PY + (ly + P::H)) * P::PX + (lx + P::HX)];
  };
  __syncthreads();
  if (warp == 0) {
    uint32_t h[4], sum = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      h[q] = bhist[127 - 4 * lane - q];
      sum += h[q];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(kFullMask, inc, o);
      if (lane >= o) inc += v;
    }
    uint32_t run = inc - sum;
    __syncwarp();
    // entries with bucket >= 4k (k = 1..31) = the exclusive prefix at lane 32-k (its first
    // bucket is 127-4(32-k) = 4k-1); k = 0: all
    if (lane >= 1) oct[tile * kOctPerTile + (32 - lane)] = (uint16_t)run;
    if (lane == 31) oct[tile * kOctPerTile] = (uint16_t)inc;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      bhist[127 - 4 * lane - q] = run;  // now: next free slot of each bucket
      run += h[q];
    }
    if (lane == 31) s_nkept = inc;  // total kept
  }
  __syncthreads();
  {
    uint2* out = cent + tile * kTileVol;
#pragma unroll 1
    for (int k = lane; k < nk; k += 32) {
      const int v = surv[warp * 32 + ((k >> 5) << 8) + lane];
      const uint32_t d = centre_d(v);
      out[atomicAdd(&bhist[dbucket(d)], 1u)] = make_uint2((uint32_t)v, d);
    }
  }
  nfg = __reduce_add_sync(kFullMask, nfg);
  maxd = __reduce_max_sync(kFullMask, maxd);
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
    const uint32_t cnt = s_nkept;
    meta[tile] = TileMeta{cnt, m, f, 0};
    if (cnt) atomicAdd(&hdr->n_kept, (unsigned long long)cnt);
  }
}

// The 3D thresholds interleaved per D for K4: [0, kDcap3] the stage-1 classes (1,0,0), (1,1,0),
// (1,1,1) (one 16-byte load per row); then three 16-byte words per D with the stage-2 classes
// 3..11 (and 3 unused words)
__global__ void k_mtable3_il(const uint32_t* __restrict__ M, uint4* __restrict__ M1) {
  const int D = blockIdx.x * blockDim.x + threadIdx.x;
  if (D > kDcap3) return;
  M1[D] = make_uint4(M[D], M[(kDcap3 + 1) + D], M[2 * (kDcap3 + 1) + D], 0u);
  auto m = [&](int c) { return c < kClasses3 ? M[c * (kDcap3 + 1) + D] : 0xFFFFFFFFu; };
  uint4* o = M1 + (kDcap3 + 1) + 3 * D;
  for (int j = 0; j < 3; ++j) o[j] = make_uint4(m(3 + 4 * j), m(4 + 4 * j), m(5 + 4 * j), m(6 + 4 * j));
}

}  // namespace

cudaError_t dilate_cover_setup();
cudaError_t dilate_atomic_setup();

cudaError_t ensure_mtables(int dev) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  DeviceTables& dt = g_tables[dev];
  if (dt.m3) return cudaSuccess;
  uint32_t *m3 = nullptr, *m2 = nullptr;
  uint4* m3s1 = nullptr;
  unsigned long long* fx = nullptr;
  cudaError_t e = cudaMalloc(&m3, sizeof(uint32_t) * kClasses3 * (kDcap3 + 1));
  if (e == cudaSuccess) e = cudaMalloc(&m3s1, sizeof(uint4) * 4 * (kDcap3 + 1));
  if (e == cudaSuccess) e = cudaMalloc(&m2, sizeof(uint32_t) * kClasses2 * (kDcap2 + 1));
  if (e == cudaSuccess) e = cudaMalloc(&fx, sizeof(unsigned long long) * kFxLut);
  if (e != cudaSuccess) {
    cudaFree(m3);
    cudaFree(m3s1);
    cudaFree(m2);
    cudaFree(fx);
    return e;
  }
  const int64_t n3 = (int64_t)kClasses3 * (kDcap3 + 1), n2 = (int64_t)kClasses2 * (kDcap2 + 1);
  k_mtable3<<<(unsigned)((n3 + 127) / 128), 128>>>(m3);
  k_mtable3_il<<<(unsigned)((kDcap3 + 1 + 127) / 128), 128>>>(m3, m3s1);
  k_mtable2<<<(unsigned)((n2 + 127) / 128), 128>>>(m2);
  k_fxtable<<<kFxLut / 256, 256>>>(fx);
  e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) e = dilate_cover_setup();
  if (e == cudaSuccess) e = dilate_atomic_setup();
  if (e != cudaSuccess) {
    cudaFree(m3);
    cudaFree(m3s1);
    cudaFree(m2);
    cudaFree(fx);
    return e;
  }
  dt.m3 = m3;
  dt.m3s1 = m3s1;
  dt.m2 = m2;
  dt.fx = fx;
  return cudaSuccess;
}

const unsigned long long* device_fxlut(int dev) { return (dev >= 0 && dev < 64) ? g_tables[dev].fx : nullptr; }

void release_mtables() {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& dt : g_tables) {
    if (dt.m3) cudaFree(dt.m3);
    if (dt.m3s1) cudaFree(dt.m3s1);
    if (dt.m2) cudaFree(dt.m2);
    if (dt.fx) cudaFree(dt.fx);
    dt.m3 = dt.m2 = nullptr;
    dt.m3s1 = nullptr;
    dt.fx = nullptr;
  }
}

// Tiled tensor map over D ([B][Z][Y][X] u32, x fastest) whose box is the padded K4 tile; false
// (-> cp.async staging) when the driver entry point is missing or the layout does not meet the
// copy engine's rules (16-byte aligned base and row pitch, coordinates and extents in int32).
static bool prune_tensor_map(CUtensorMap* m, const uint32_t* D, const Geom& g) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    cudaGetLastError();
    return reinterpret_cast<Encode>(fn);
  }();
  memset(m, 0, sizeof(*m));
  if (!encode || (g.X & 3) != 0 || (reinterpret_cast<uintptr_t>(D) & 15) != 0) return false;
  if (g.X > INT32_MAX / 2 || g.Y > INT32_MAX / 2 || g.Z > INT32_MAX / 2 || g.B > INT32_MAX) return false;
  const bool is3 = g.ndim == 3;
  const cuuint32_t rank = is3 ? 4 : 3;
  cuuint64_t dims[4], strides[3];
  cuuint32_t box[4], estr[4] = {1, 1, 1, 1};
  dims[0] = (cuuint64_t)g.X;
  dims[1] = (cuuint64_t)g.Y;
  strides[0] = (cuuint64_t)g.X * 4;
  if (is3) {
    dims[2] = (cuuint64_t)g.Z;
    dims[3] = (cuuint64_t)g.B;
    strides[1] = strides[0] * (cuuint64_t)g.Y;
    strides[2] = strides[1] * (cuuint64_t)g.Z;
    box[0] = PruneTile<true>::PX, box[1] = PruneTile<true>::PY, box[2] = PruneTile<true>::PZ, box[3] = 1;
  } else {
    dims[2] = (cuuint64_t)g.B;
    strides[1] = strides[0] * (cuuint64_t)g.Y;
    box[0] = PruneTile<false>::PX, box[1] = PruneTile<false>::PY, box[2] = 1;
  }
  for (cuuint32_t i = 0; i + 1 < rank; ++i)
    if (strides[i] >= (1ull << 40)) return false;
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, rank, const_cast<uint32_t*>(D), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

#ifndef FASTRS_PRUNE_PREFETCH
#define FASTRS_PRUNE_PREFETCH 0
#endif
constexpr int kPrunePrefetch = FASTRS_PRUNE_PREFETCH;  // L2 prefetch distance in CTAs per SM (0: off; 6 measured 4.11 vs 4.09 ms)

void launch_prune(const uint32_t* D, const Geom& g, TileMeta* meta, uint2* centres, uint32_t* fgm, uint32_t* shm,
                  uint16_t* oct, WsHeader* hdr, cudaStream_t st, int64_t tz_lo, int64_t tz_hi, bool exact_prune) {
  int dev = 0;
  cudaGetDevice(&dev);
  // tile layers [tz_lo, tz_hi) of item 0 (batch 1), or every tile
  const bool part = tz_hi > tz_lo && g.B == 1;
  const int64_t tile0 = part ? tz_lo * g.nty * g.ntx : 0;
  const int64_t n = part ? (tz_hi - tz_lo) * g.nty * g.ntx : g.ntiles;
  if (n <= 0) return;
  CUtensorMap tmap;
  const bool tma = prune_tensor_map(&tmap, D, g);
  const FastDiv fdx((uint32_t)g.ntx), fdy((uint32_t)g.nty), fdz((uint32_t)g.ntz);
  // stage-2 classes: 3D tests the five that drop centres on C4 unless the exact |s|^2 <= 12 set
  // is asked for (FASTRS_EXACT_PRUNE); the skipped four only ever keep more (contained) balls,
  // which LT^2 = max over covering balls ignores.  2D: all three classes.
  const int nc2 = g.ndim == 3 ? (exact_prune ? kClasses3 - 3 : kPruneFastClasses3) : kClasses2 - 2;
  int pf = 0;
  if (kPrunePrefetch) {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    pf = nsm * kPrunePrefetch;  // resident CTAs (6 per SM) x the knob / 6
    pf = pf / 6 * 6 > 0 ? pf : 0;
  }
  if (g.ndim == 3) {
    if (tma)
      k_prune<true, true><<<(unsigned)n, 256, 0, st>>>(D, g, meta, centres, fgm, shm, oct, g_tables[dev].m3, g_tables[dev].m3s1, tile0, hdr, tmap, fdx, fdy, fdz, nc2, pf);
    else
      k_prune<true, false><<<(unsigned)n, 256, 0, st>>>(D, g, meta, centres, fgm, shm, oct, g_tables[dev].m3, g_tables[dev].m3s1, tile0, hdr, tmap, fdx, fdy, fdz, nc2, pf);
  } else {
    if (tma)
      k_prune<false, true><<<(unsigned)n, 256, 0, st>>>(D, g, meta, centres, fgm, shm, oct, g_tables[dev].m2, nullptr, tile0, hdr, tmap, fdx, fdy, fdz, nc2, pf);
    else
      k_prune<false, false><<<(unsigned)n, 256, 0, st>>>(D, g, meta, centres, fgm, shm, oct, g_tables[dev].m2, nullptr, tile0, hdr, tmap, fdx, fdy, fdz, nc2, pf);
  }
}

}  // namespace fastrs
