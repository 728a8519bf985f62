// The paper's object filters (the label-level part):
//  - edge objects: a label with an element on the grid boundary ("Edge cells are
//    removed for preservation of realistic shapes"; SPEC.md:212 remove_edge_objects);
//  - small objects: volume below a threshold ("the smallest objects are filtered
//    out (V < 10^3)"; SPEC.md:219 filter_small).
// Connected-component labelling stays out of scope: inputs are label grids.
#include "common.cuh"

namespace fastrs {
namespace {

// one thread per boundary element of one item: 3D faces z = 0, Z-1 (Y*X each), y = 0, Y-1
// (Z*X), x = 0, X-1 (Z*Y); 2D edges y = 0, Y-1 (X each), x = 0, X-1 (Y each).  Elements on
// several faces are visited more than once (harmless: every write stores 1).
__global__ void k_touch_edge(const int32_t* __restrict__ lab, Geom g, int32_t max_label, int64_t per_item,
                             int skip_zlo, int skip_zhi, uint8_t* __restrict__ touch) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= per_item * g.B) return;
  const int64_t b = t / per_item;
  int64_t r = t - b * per_item;
  const int64_t X = g.X, Y = g.Y, Z = g.Z;
  int64_t x, y, z = 0;
  if (g.ndim == 3) {
    if (r < 2 * Y * X) {
      z = r < Y * X ? 0 : Z - 1;
      if ((r < Y * X && skip_zlo) || (r >= Y * X && skip_zhi)) return;  // a slab's inner face
      r %= Y * X;
      y = r / X;
      x = r % X;
    } else if ((r -= 2 * Y * X) < 2 * Z * X) {
      y = r < Z * X ? 0 : Y - 1;
      r %= Z * X;
      z = r / X;
      x = r % X;
    } else {
      r -= 2 * Z * X;
      x = r < Z * Y ? 0 : X - 1;
      r %= Z * Y;
      z = r / Y;
      y = r % Y;
    }
  } else {
    if (r < 2 * X) {
      y = r < X ? 0 : Y - 1;
      x = r % X;
    } else {
      r -= 2 * X;
      x = r < Y ? 0 : X - 1;
      y = r % Y;
    }
  }
  const int32_t L = lab[((b * Z + z) * Y + y) * X + x];
  if (L > 0 && L <= max_label) touch[b * max_label + (L - 1)] = 1;
}

__global__ void k_filter(double* __restrict__ sph, double* __restrict__ rnd, const int64_t* __restrict__ vol,
                         const uint8_t* __restrict__ touch, int64_t n, int64_t min_volume) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool drop = (vol && vol[i] < min_volume) || (touch && touch[i]);
  if (drop) {
    const double nan = __longlong_as_double(0x7FF8000000000000ll);
    if (sph) sph[i] = nan;
    if (rnd) rnd[i] = nan;
  }
}

}  // namespace

cudaError_t launch_touch_edge(const int32_t* labels, const Geom& g, int32_t max_label, uint8_t* touch,
                              bool skip_zlo, bool skip_zhi, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(touch, 0, (size_t)g.B * (size_t)max_label, st);
  if (e != cudaSuccess) return e;
  const int64_t per_item = g.ndim == 3 ? 2 * (g.Y * g.X + g.Z * g.X + g.Z * g.Y) : 2 * (g.X + g.Y);
  const int64_t n = per_item * g.B;
  if (n > 0)
    k_touch_edge<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(labels, g, max_label, per_item, skip_zlo ? 1 : 0,
                                                             skip_zhi ? 1 : 0, touch);
  return cudaGetLastError();
}

cudaError_t launch_filter(double* sph, double* rnd, const int64_t* vol, const uint8_t* touch, int64_t n,
                          int64_t min_volume, cudaStream_t st) {
  if (n > 0) k_filter<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(sph, rnd, vol, touch, n, min_volume);
  return cudaGetLastError();
}

}  // namespace fastrs
