// Analysis-protocol kernels around the hot path:
//   NEXT-4  connected-component labelling of a binary mask ("segmenting and
//           labeling each fat component") and Eq. 3 width/length
//           sphericity (SPEC.md:355-361 covariance reading);
//   NEXT-2  the S_MC baseline: per-object marching-squares perimeter (2D) / marching-cubes
//           surface area (3D) and the sphericity from it (§5.2).
// The readings are listed in DESIGN.md "Readings" (r1-r4).
#include <cmath>
#include <mutex>

#include "common.cuh"
#include "fastrs.h"

namespace fastrs {
namespace {

constexpr unsigned kAll = 0xFFFFFFFFu;
constexpr uint32_t kNoParent = 0xFFFFFFFFu;

// ============================================================================================
// Connected components: union-find with atomicMin linking.  Every union links the larger root
// under the smaller, so a component's root is its smallest (row-major first) element; roots
// numbered in index order give exactly the first-encounter labelling (canonical, independent
// of thread scheduling).
// ============================================================================================
__device__ __forceinline__ uint32_t uf_find(uint32_t* P, uint32_t x) {
  uint32_t p = P[x];
  while (p != x) {
    const uint32_t gp = P[p];
    if (gp != p) P[x] = gp;  // path halving: parents only ever move to ancestors
    x = p;
    p = gp;
  }
  return x;
}

__device__ __forceinline__ void uf_union(uint32_t* P, uint32_t a, uint32_t b) {
  for (;;) {
    a = uf_find(P, a);
    b = uf_find(P, b);
    if (a == b) return;
    if (a < b) {
      const uint32_t t = a;
      a = b;
      b = t;
    }
    const uint32_t old = atomicMin(P + a, b);  // link root a under b (a > b)
    if (old == a) return;
    a = old;  // a gained another parent meanwhile: retry from there
  }
}

struct CclGeom {
  int ndim, conn;
  int64_t B, Z, Y, X, vol;
};

__global__ void k_ccl_init(const uint8_t* __restrict__ mask, uint32_t* __restrict__ P, CclGeom g) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.B * g.vol) return;
  P[i] = mask[i] ? (uint32_t)(i % g.vol) : kNoParent;  // item-relative indices
}

__global__ void k_ccl_merge(uint32_t* __restrict__ P, CclGeom g) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.B * g.vol) return;
  if (P[i] == kNoParent) return;
  const int64_t b = i / g.vol, r = i % g.vol;
  uint32_t* Pb = P + b * g.vol;
  const int64_t x = r % g.X, y = (r / g.X) % g.Y, z = r / (g.X * g.Y);
  const int maxsum = g.ndim == 2 ? (g.conn == 4 ? 1 : 2) : (g.conn == 6 ? 1 : (g.conn == 18 ? 2 : 3));
  // backward neighbours (linear offset < 0) of the connectivity: each pair is united once
  for (int dz = (g.ndim == 3 ? -1 : 0); dz <= 0; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const bool back = dz < 0 || (dz == 0 && (dy < 0 || (dy == 0 && dx < 0)));
        if (!back || abs(dz) + abs(dy) + abs(dx) > maxsum) continue;
        const int64_t zz = z + dz, yy = y + dy, xx = x + dx;
        if (zz < 0 || yy < 0 || yy >= g.Y || xx < 0 || xx >= g.X) continue;
        const int64_t j = (zz * g.Y + yy) * g.X + xx;
        if (Pb[j] != kNoParent) uf_union(Pb, (uint32_t)r, (uint32_t)j);
      }
}

constexpr int kScanBlock = 1024;  // elements per scan block (256 threads x 4)

// read-only find (the flatten pass: each thread writes only its own parent, so no ancestor
// pointer of another element is ever replaced by a stale one)
__device__ __forceinline__ uint32_t uf_root(const uint32_t* P, uint32_t x) {
  uint32_t p = P[x];
  while (p != x) {
    x = p;
    p = P[x];
  }
  return x;
}

// flatten every tree and count the roots of each scan block of each item
__global__ void k_ccl_flatten_count(uint32_t* __restrict__ P, CclGeom g, int64_t nblk, uint32_t* __restrict__ bsum) {
  const int64_t b = blockIdx.y, blk = blockIdx.x;
  uint32_t* Pb = P + b * g.vol;
  uint32_t c = 0;
  for (int k = 0; k < kScanBlock / 256; ++k) {
    const int64_t r = blk * kScanBlock + k * 256 + threadIdx.x;
    if (r < g.vol && Pb[r] != kNoParent) {
      const uint32_t root = uf_root(Pb, (uint32_t)r);
      Pb[r] = root;
      c += root == (uint32_t)r;
    }
  }
  c = __reduce_add_sync(kAll, c);
  __shared__ uint32_t ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < 8; ++w) t += ws[w];
    bsum[b * nblk + blk] = t;
  }
}

// per item: exclusive scan of the block counts (one CTA per item), total = components
__global__ void k_ccl_scan_blocks(uint32_t* __restrict__ bsum, int64_t nblk, int64_t* __restrict__ counts) {
  const int64_t b = blockIdx.x;
  uint32_t* s = bsum + b * nblk;
  const int64_t per = (nblk + 1023) / 1024, lo = threadIdx.x * per, hi = min(nblk, lo + per);
  unsigned long long loc = 0;
  for (int64_t i = lo; i < hi; ++i) loc += s[i];
  __shared__ unsigned long long part[1024];
  part[threadIdx.x] = loc;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {  // inclusive Hillis-Steele scan of the per-thread sums
    const unsigned long long v = threadIdx.x >= o ? part[threadIdx.x - o] : 0ull;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  unsigned long long run = part[threadIdx.x] - loc;
  for (int64_t i = lo; i < hi; ++i) {
    const uint32_t v = s[i];
    s[i] = (uint32_t)run;
    run += v;
  }
  if (threadIdx.x == 1023 && counts) counts[b] = (int64_t)part[1023];
}

// roots get their dense label (1 + number of roots before them in the item)
__global__ void k_ccl_root_labels(const uint32_t* __restrict__ P, CclGeom g, int64_t nblk,
                                  const uint32_t* __restrict__ boff, int32_t* __restrict__ out) {
  const int64_t b = blockIdx.y, blk = blockIdx.x;
  const uint32_t* Pb = P + b * g.vol;
  __shared__ uint32_t ws[8];
  uint32_t base = boff[b * nblk + blk];
  for (int k = 0; k < kScanBlock / 256; ++k) {
    const int64_t r = blk * kScanBlock + k * 256 + threadIdx.x;
    const bool root = r < g.vol && Pb[r] == (uint32_t)r;
    const uint32_t m = __ballot_sync(kAll, root);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) ws[w] = __popc(m);
    __syncthreads();
    uint32_t before = 0, tot = 0;
    for (int v = 0; v < 8; ++v) {
      if (v < w) before += ws[v];
      tot += ws[v];
    }
    if (root) out[b * g.vol + r] = (int32_t)(base + before + __popc(m & ((1u << lane) - 1u)) + 1);
    base += tot;
    __syncthreads();
  }
}

__global__ void k_ccl_relabel(const uint32_t* __restrict__ P, CclGeom g, int32_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.B * g.vol) return;
  const uint32_t p = P[i];
  const int64_t b = i / g.vol;
  if (p == kNoParent) out[i] = 0;
  else if (p != (uint32_t)(i % g.vol)) out[i] = out[b * g.vol + p];  // (roots are not written here)
}

// ============================================================================================
// Eq. 3 width / length sphericity: exact integer moments per label, then the covariance axes
// ============================================================================================
struct Moments {
  unsigned long long* n;
  unsigned long long* sx;
  unsigned long long* sy;
  unsigned long long* sxx;
  unsigned long long* syy;
  unsigned long long* sxy;
  int32_t max_label;
};

// sum of a per-lane value v < 2^28 over the lanes of `grp` (two 16-bit pieces: no u32 overflow)
__device__ __forceinline__ unsigned long long group_sum28(uint32_t v, bool in) {
  const uint32_t hi = __reduce_add_sync(kAll, in ? v >> 16 : 0u), lo = __reduce_add_sync(kAll, in ? v & 0xFFFFu : 0u);
  return ((unsigned long long)hi << 16) + lo;
}

__global__ void k_wl_moments(const int32_t* __restrict__ lab, int64_t B, int64_t Y, int64_t X, Moments m) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);  // one warp per row
  if (row >= B * Y) return;
  const int64_t b = row / Y, y = row % Y;
  for (int64_t x0 = 0; x0 < X; x0 += 32) {
    const int64_t x = x0 + lane;
    int32_t L = x < X ? __ldg(lab + row * X + x) : 0;
    if ((uint32_t)L > (uint32_t)m.max_label) L = 0;
    uint32_t act = __ballot_sync(kAll, L != 0);
    while (act) {
      const int leader = __ffs(act) - 1;
      const int32_t key = __shfl_sync(kAll, L, leader);
      const uint32_t grp = __ballot_sync(kAll, L == key);
      const bool in = (grp >> lane) & 1u;
      const uint32_t xi = (uint32_t)x, yi = (uint32_t)y;
      const unsigned long long n = __popc(grp), sx = group_sum28(xi, in), sy = group_sum28(yi, in);
      const unsigned long long sxx = group_sum28(xi * xi, in), syy = group_sum28(yi * yi, in),
                               sxy = group_sum28(xi * yi, in);
      if (lane == leader) {
        const int64_t id = b * m.max_label + key - 1;
        atomicAdd(m.n + id, n);
        atomicAdd(m.sx + id, sx);
        atomicAdd(m.sy + id, sy);
        atomicAdd(m.sxx + id, sxx);
        atomicAdd(m.syy + id, syy);
        atomicAdd(m.sxy + id, sxy);
      }
      act &= ~grp;
    }
  }
}

__global__ void k_wl_metrics(Moments m, int64_t M, double* __restrict__ swl, double* __restrict__ d1,
                             double* __restrict__ d2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  const unsigned long long n = m.n[i];
  double s = nan(""), a = nan(""), c = nan("");
  if (n > 0) {
    // population covariance from exact integer numerators: n^2 var_x = n sxx - sx^2, ...
    const __int128 N = (__int128)n;
    const __int128 nx = N * (__int128)m.sxx[i] - (__int128)m.sx[i] * (__int128)m.sx[i];
    const __int128 ny = N * (__int128)m.syy[i] - (__int128)m.sy[i] * (__int128)m.sy[i];
    const __int128 nxy = N * (__int128)m.sxy[i] - (__int128)m.sx[i] * (__int128)m.sy[i];
    const double n2 = (double)n * (double)n;
    const double vx = (double)nx / n2, vy = (double)ny / n2, vxy = (double)nxy / n2;
    const double h = 0.5 * (vx + vy), r = sqrt(0.25 * (vx - vy) * (vx - vy) + vxy * vxy);
    const double l1 = h + r, l2 = fmax(h - r, 0.0);
    a = 4.0 * sqrt(l1);
    c = 4.0 * sqrt(l2);
    s = l1 > 0 ? c / a : 1.0;  // a single pixel: 1
  }
  if (swl) swl[i] = s;
  if (d1) d1[i] = a;
  if (d2) d2[i] = c;
}

// ============================================================================================
// S_MC: per-label iso-0.5 perimeter (2D marching squares) / surface area (3D marching cubes)
// ============================================================================================
constexpr double kMcScale = 4294967296.0;  // fixed-point 2^-32: the per-label sums are exact

// 3D case table (cube corner q = x | y << 1 | z << 2 inside when bit q of the case is set): the
// iso-surface is built from its definition -- per face the midpoint crossings joined into
// segments (two diagonal inside corners: one segment around each inside corner), the face
// segments closed into loops through the shared crossings, each loop's area the fan of
// triangles (loop centroid, v_i, v_i+1).  Computed once per device.
__device__ double3 edge_mid(int e) {  // e = a * 8 + b: the midpoint of cube edge (a, b)
  const int a = e >> 3, b = e & 7;
  return make_double3(0.5 * ((a & 1) + (b & 1)), 0.5 * (((a >> 1) & 1) + ((b >> 1) & 1)),
                      0.5 * (((a >> 2) & 1) + ((b >> 2) & 1)));
}

__global__ void k_mc_table3(double* __restrict__ tab) {
  const int cs = threadIdx.x;  // 256 cases
  const int F[6][4] = {{0, 1, 3, 2}, {4, 5, 7, 6}, {0, 1, 5, 4}, {2, 3, 7, 6}, {0, 2, 6, 4}, {1, 3, 7, 5}};
  int sa[12], sb[12], ns = 0;  // segments as pairs of edge ids
  auto ek = [](int a, int b) { return a < b ? a * 8 + b : b * 8 + a; };
  for (int f = 0; f < 6; ++f) {
    bool in[4];
    int cnt = 0;
    for (int i = 0; i < 4; ++i) cnt += (in[i] = (cs >> F[f][i]) & 1);
    if (cnt == 0 || cnt == 4) continue;
    if (cnt == 2 && in[0] == in[2]) {
      for (int i = 0; i < 4; ++i)
        if (in[i]) {
          sa[ns] = ek(F[f][i], F[f][(i + 3) & 3]);
          sb[ns++] = ek(F[f][i], F[f][(i + 1) & 3]);
        }
    } else {
      int e[2], k = 0;
      for (int i = 0; i < 4; ++i)
        if (in[i] != in[(i + 1) & 3]) e[k++] = ek(F[f][i], F[f][(i + 1) & 3]);
      sa[ns] = e[0];
      sb[ns++] = e[1];
    }
  }
  bool used[12] = {false};
  double area = 0;
  for (int s0 = 0; s0 < ns; ++s0) {
    if (used[s0]) continue;
    int loop[12], nl = 0;
    used[s0] = true;
    loop[nl++] = sa[s0];
    int cur = sb[s0];
    while (cur != loop[0]) {
      loop[nl++] = cur;
      for (int t = 0; t < ns; ++t)
        if (!used[t] && (sa[t] == cur || sb[t] == cur)) {
          used[t] = true;
          cur = sa[t] == cur ? sb[t] : sa[t];
          break;
        }
    }
    double3 c = make_double3(0, 0, 0);
    for (int i = 0; i < nl; ++i) {
      const double3 v = edge_mid(loop[i]);
      c.x += v.x;
      c.y += v.y;
      c.z += v.z;
    }
    c.x /= nl;
    c.y /= nl;
    c.z /= nl;
    for (int i = 0; i < nl; ++i) {
      const double3 p = edge_mid(loop[i]), q = edge_mid(loop[(i + 1) % nl]);
      const double ux = p.x - c.x, uy = p.y - c.y, uz = p.z - c.z, vx = q.x - c.x, vy = q.y - c.y, vz = q.z - c.z;
      const double cx = uy * vz - uz * vy, cy = uz * vx - ux * vz, cz = ux * vy - uy * vx;
      area += 0.5 * sqrt(cx * cx + cy * cy + cz * cz);
    }
  }
  tab[cs] = area;
}

// 2D: corners in cyclic order (y, x), (y, x+1), (y+1, x+1), (y+1, x) -> bits 0..3; every
// crossing is an edge midpoint: one corner cut off sqrt(1/2), two adjacent corners a straight
// unit segment, two diagonal corners two cuts, three corners one cut
__device__ __forceinline__ double ms_length(int cs) {
  const int n = __popc(cs);
  if (n == 1 || n == 3) return 0.70710678118654752440;
  if (n == 2) return (cs == 5 || cs == 10) ? 1.41421356237309504880 : 1.0;
  return 0.0;
}

struct McArgs {
  int ndim;
  int64_t B, Z, Y, X;
  int32_t max_label;
  unsigned long long* sum;  // fixed-point measure per label
  unsigned long long* vol;  // elements per label
};

// one thread per cell; cells have origins (z, y, x) in [-1, Z) x [-1, Y) x [-1, X) (2D: z = 0);
// each distinct label among the cell's corners adds its case's measure; the voxel at the
// cell's corner (1,1,1) (i.e. (z+1, y+1, x+1), when inside the grid) is counted in vol
__global__ void __launch_bounds__(256) k_mc_cells(const int32_t* __restrict__ lab, McArgs a,
                                                  const unsigned long long* __restrict__ tab) {
  const int64_t nx = a.X + 1, ny = a.Y + 1, nz = a.ndim == 3 ? a.Z + 1 : 1;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = nx * ny * nz;
  const bool valid = t < a.B * per;
  const int lane = threadIdx.x & 31;
  int64_t b = 0, z = 0, y = 0, x = 0;
  if (valid) {
    b = t / per;
    const int64_t r = t % per;
    x = r % nx - 1;
    y = (r / nx) % ny - 1;
    z = a.ndim == 3 ? r / (nx * ny) - 1 : 0;
  }
  const int32_t* Lb = lab + b * a.Z * a.Y * a.X;
  auto at = [&](int64_t zz, int64_t yy, int64_t xx) -> int32_t {
    if (!valid || zz < 0 || zz >= a.Z || yy < 0 || yy >= a.Y || xx < 0 || xx >= a.X) return 0;
    const int32_t v = __ldg(Lb + (zz * a.Y + yy) * a.X + xx);
    return (uint32_t)v > (uint32_t)a.max_label ? 0 : v;
  };
  int32_t c[8];
  int ncorner;
  if (a.ndim == 3) {
    for (int q = 0; q < 8; ++q) c[q] = at(z + ((q >> 2) & 1), y + ((q >> 1) & 1), x + (q & 1));
    ncorner = 8;
  } else {
    c[0] = at(0, y, x);
    c[1] = at(0, y, x + 1);
    c[2] = at(0, y + 1, x + 1);
    c[3] = at(0, y + 1, x);
    ncorner = 4;
  }
  for (int i = 0; i < ncorner; ++i) {
    const int32_t k = c[i];
    if (k == 0) continue;
    bool seen = false;
    for (int j = 0; j < i; ++j) seen |= c[j] == k;
    if (seen) continue;
    int cs = 0;
    for (int j = 0; j < ncorner; ++j) cs |= (c[j] == k) << j;
    const unsigned long long v = a.ndim == 3 ? tab[cs] : (unsigned long long)__double2ull_rn(ms_length(cs) * kMcScale);
    if (v) atomicAdd(a.sum + b * a.max_label + k - 1, v);
  }
  // the element at the cell's far corner, counted once per element: warp-aggregated
  const int32_t e = a.ndim == 3 ? c[7] : c[2];
  const bool own = valid && e != 0 && x + 1 < a.X && y + 1 < a.Y && (a.ndim == 2 || z + 1 < a.Z);
  const int32_t key = own ? e : 0;
  uint32_t act = __ballot_sync(kAll, key != 0);
  while (act) {
    const int leader = __ffs(act) - 1;
    const int32_t kk = __shfl_sync(kAll, key, leader);
    const int64_t bb = __shfl_sync(kAll, b, leader);
    const uint32_t grp = __ballot_sync(kAll, key == kk && b == bb);
    if (lane == leader) atomicAdd(a.vol + bb * a.max_label + kk - 1, (unsigned long long)__popc(grp));
    act &= ~grp;
  }
}

__global__ void k_mc_finish(McArgs a, int64_t M, double* __restrict__ measure, double* __restrict__ smc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  const double V = (double)a.vol[i], m = (double)a.sum[i] / kMcScale;
  double s = nan("");
  if (V > 0)
    s = a.ndim == 3 ? cbrt(3.14159265358979323846) * pow(6.0 * V, 2.0 / 3.0) / m  // Eq. 1
                    : 2.0 * sqrt(3.14159265358979323846 * V) / m;               // Eq. 2, P_c / P_o
  if (measure) measure[i] = V > 0 ? m : nan("");
  if (smc) smc[i] = s;
}

__global__ void k_mc_fixed(const double* __restrict__ d, unsigned long long* __restrict__ f) {
  f[threadIdx.x] = (unsigned long long)__double2ull_rn(d[threadIdx.x] * kMcScale);
}

std::mutex g_mc_mu;
unsigned long long* g_mc_tab[64];

int api_err(int code, const char* msg) { return set_error(code, msg); }

}  // namespace
}  // namespace fastrs

using namespace fastrs;

extern "C" {

int fastrs_ccl_workspace_bytes(const int64_t* dims, int ndim, int64_t batch, size_t* bytes) {
  if (!dims || !bytes || (ndim != 2 && ndim != 3) || batch < 1) return api_err(FASTRS_EINVAL, "bad arguments");
  int64_t vol = 1;
  for (int i = 0; i < ndim; ++i) vol *= dims[i];
  const int64_t nblk = (vol + kScanBlock - 1) / kScanBlock;
  *bytes = (size_t)(batch * vol * 4 + 256 + batch * nblk * 4 + 256);
  return FASTRS_OK;
}

int fastrs_label_components(const uint8_t* mask, const int64_t* dims, int ndim, int64_t batch, int connectivity,
                            int32_t* labels_out, int64_t* counts_out, void* ws, size_t ws_bytes, void* stream) {
  if (!mask || !dims || !labels_out || !ws) return api_err(FASTRS_EINVAL, "NULL pointer");
  if (ndim != 2 && ndim != 3) return api_err(FASTRS_EINVAL, "ndim must be 2 or 3");
  const bool ok = ndim == 2 ? (connectivity == 4 || connectivity == 8)
                            : (connectivity == 6 || connectivity == 18 || connectivity == 26);
  if (!ok) return api_err(FASTRS_EINVAL, "connectivity must be 4/8 (2D) or 6/18/26 (3D)");
  CclGeom g{};
  g.ndim = ndim;
  g.conn = connectivity;
  g.B = batch;
  g.Z = ndim == 3 ? dims[0] : 1;
  g.Y = dims[ndim - 2];
  g.X = dims[ndim - 1];
  if (batch < 1 || g.Z < 1 || g.Y < 1 || g.X < 1) return api_err(FASTRS_EINVAL, "empty geometry");
  g.vol = g.Z * g.Y * g.X;
  if (g.vol >= (int64_t)kNoParent) return api_err(FASTRS_EINVAL, "an item has 2^32 or more elements");
  size_t need = 0;
  fastrs_ccl_workspace_bytes(dims, ndim, batch, &need);
  if (ws_bytes < need) return api_err(FASTRS_ENOMEM, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* P = (uint32_t*)ws;
  const int64_t nblk = (g.vol + kScanBlock - 1) / kScanBlock;
  uint32_t* bsum = (uint32_t*)((char*)ws + ((batch * g.vol * 4 + 255) & ~(int64_t)255));
  const int64_t n = batch * g.vol;
  const unsigned grid = (unsigned)((n + 255) / 256);
  k_ccl_init<<<grid, 256, 0, st>>>(mask, P, g);
  k_ccl_merge<<<grid, 256, 0, st>>>(P, g);
  k_ccl_flatten_count<<<dim3((unsigned)nblk, (unsigned)batch), 256, 0, st>>>(P, g, nblk, bsum);
  k_ccl_scan_blocks<<<(unsigned)batch, 1024, 0, st>>>(bsum, nblk, counts_out);
  k_ccl_root_labels<<<dim3((unsigned)nblk, (unsigned)batch), 256, 0, st>>>(P, g, nblk, bsum, labels_out);
  k_ccl_relabel<<<grid, 256, 0, st>>>(P, g, labels_out);
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return api_err(FASTRS_ECUDA, cudaGetErrorString(e));
  return FASTRS_OK;
}

int fastrs_wl_workspace_bytes(int64_t batch, int32_t max_label, size_t* bytes) {
  if (!bytes || batch < 1 || max_label < 1) return api_err(FASTRS_EINVAL, "bad arguments");
  *bytes = (size_t)(6 * batch * (int64_t)max_label * 8);
  return FASTRS_OK;
}

int fastrs_sphericity_wl(const int32_t* labels, const int64_t* dims, int ndim, int64_t batch, int32_t max_label,
                         double* swl, double* d1, double* d2, void* ws, size_t ws_bytes, void* stream) {
  if (!labels || !dims || !ws) return api_err(FASTRS_EINVAL, "NULL pointer");
  if (ndim != 2) return api_err(FASTRS_EINVAL, "Eq. 3 width/length sphericity is defined for 2D images");
  if (batch < 1 || max_label < 1 || dims[0] < 1 || dims[1] < 1 || dims[1] > 16384 || dims[0] > 16384)
    return api_err(FASTRS_EINVAL, "bad geometry");
  size_t need = 0;
  fastrs_wl_workspace_bytes(batch, max_label, &need);
  if (ws_bytes < need) return api_err(FASTRS_ENOMEM, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t M = batch * (int64_t)max_label;
  unsigned long long* w = (unsigned long long*)ws;
  Moments m{w, w + M, w + 2 * M, w + 3 * M, w + 4 * M, w + 5 * M, max_label};
  cudaMemsetAsync(ws, 0, need, st);
  const int64_t rows = batch * dims[0];
  k_wl_moments<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(labels, batch, dims[0], dims[1], m);
  k_wl_metrics<<<(unsigned)((M + 255) / 256), 256, 0, st>>>(m, M, swl, d1, d2);
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return api_err(FASTRS_ECUDA, cudaGetErrorString(e));
  return FASTRS_OK;
}

int fastrs_mc_workspace_bytes(int64_t batch, int32_t max_label, size_t* bytes) {
  if (!bytes || batch < 1 || max_label < 1) return api_err(FASTRS_EINVAL, "bad arguments");
  *bytes = (size_t)(2 * batch * (int64_t)max_label * 8);
  return FASTRS_OK;
}

int fastrs_mc_measure(const int32_t* labels, const int64_t* dims, int ndim, int64_t batch, int32_t max_label,
                      double* measure, double* sphericity_mc, void* ws, size_t ws_bytes, void* stream) {
  if (!labels || !dims || !ws) return api_err(FASTRS_EINVAL, "NULL pointer");
  if ((ndim != 2 && ndim != 3) || batch < 1 || max_label < 1) return api_err(FASTRS_EINVAL, "bad arguments");
  for (int i = 0; i < ndim; ++i)
    if (dims[i] < 1 || dims[i] > 16384) return api_err(FASTRS_EINVAL, "dims outside [1, 16384]");
  size_t need = 0;
  fastrs_mc_workspace_bytes(batch, max_label, &need);
  if (ws_bytes < need) return api_err(FASTRS_ENOMEM, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(g_mc_mu);
    if (!g_mc_tab[dev]) {  // the 256-case area table, once per device
      double* d = nullptr;
      unsigned long long* f = nullptr;
      cudaError_t e = cudaMalloc(&d, 256 * sizeof(double));
      if (e == cudaSuccess) e = cudaMalloc(&f, 256 * sizeof(unsigned long long));
      if (e == cudaSuccess) {
        k_mc_table3<<<1, 256>>>(d);
        k_mc_fixed<<<1, 256>>>(d, f);
        e = cudaDeviceSynchronize();
      }
      cudaFree(d);
      if (e != cudaSuccess) {
        cudaFree(f);
        return api_err(FASTRS_ECUDA, cudaGetErrorString(e));
      }
      g_mc_tab[dev] = f;
    }
  }
  const int64_t M = batch * (int64_t)max_label;
  McArgs a{};
  a.ndim = ndim;
  a.B = batch;
  a.Z = ndim == 3 ? dims[0] : 1;
  a.Y = dims[ndim - 2];
  a.X = dims[ndim - 1];
  a.max_label = max_label;
  a.sum = (unsigned long long*)ws;
  a.vol = a.sum + M;
  cudaMemsetAsync(ws, 0, need, st);
  const int64_t cells = batch * (a.X + 1) * (a.Y + 1) * (ndim == 3 ? a.Z + 1 : 1);
  k_mc_cells<<<(unsigned)((cells + 255) / 256), 256, 0, st>>>(labels, a, g_mc_tab[dev]);
  k_mc_finish<<<(unsigned)((M + 255) / 256), 256, 0, st>>>(a, M, measure, sphericity_mc);
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return api_err(FASTRS_ECUDA, cudaGetErrorString(e));
  return FASTRS_OK;
}

}  // extern "C"
