// Seeded synthetic label-image generators: test and benchmark scaffolding only.
//
// This module holds NONE of the method's arithmetic (no distance transform, no local
// thickness, no sphericity/roundness).  It only rasterises randomly drawn ellipses,
// spheroids, rough grains and touching cells into int32 label grids, standing in for
// the paper's datasets, which are not available (PAPER.md:160 Krumbein charts,
// PAPER.md:179 microscopy, PAPER.md:199 mozzarella uCT).  The recipe is stated in
// DESIGN.md ("Input recipe").  Both the CPU oracle tests and the GPU parity tests /
// bench consume its output; neither side's code lives here.
//
// Shapes.  An object is an ellipsoid with semi-axes (a0,a1,a2) in a body frame given
// by a rotation matrix, optionally roughened: a body-frame point b is inside iff
//     sum_i b_i^2 / a_i^2  <=  (1 + A * n(b/|b|))^2 ,
// where n is a smooth function on the unit sphere (3D) or circle (2D) with |n| <= 1.
// Rasterisation is by element-centre inclusion.
//
// Placement (non-touching scenes).  Objects are placed in the given order (the caller
// sorts them large-first) by rejection sampling of integer centres: a placement is
// accepted iff every element of the object's footprint dilated by one element
// (26-/8-neighbourhood) is inside the grid and free.  After `max_tries` failures the
// object is shrunk by 0.85 and retried (at most 12 times), then dropped.
//
// Touching scenes (C5 cells).  Every cell claims the elements where its normalised
// radius is <= 1; an element claimed by several cells goes to the smallest normalised
// radius (ties: the lower label).

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

struct SplitMix {
  uint64_t s;
  explicit SplitMix(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return (next() >> 11) * (1.0 / 9007199254740992.0); }
  double normal() {
    double u1 = uniform(), u2 = uniform();
    if (u1 < 1e-300) u1 = 1e-300;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
};

constexpr int kRoughTerms3D = 6;
constexpr int kRoughTerms2D = 8;

// Per-object description as passed from Python (13 doubles per object):
//   [0..2] semi-axes a0,a1,a2 (a2 unused in 2D)
//   [3..6] unit quaternion (w,x,y,z) (3D) | [3] = angle theta (2D)
//   [7]    roughness amplitude A (0 = smooth)
//   [8]    roughness seed (as double, integer-valued)
//   [9..11] fixed centre (z,y,x) if [12] != 0
//   [12]   has fixed centre
constexpr int kParams = 13;

struct Shape {
  bool is2d;
  double ax[3];
  double R[9];  // world->body: b = R * d   (d = (dz,dy,dx) offsets)
  double A;
  // rough terms
  double v[kRoughTerms3D][3], f[kRoughTerms3D], ph[kRoughTerms3D], c[kRoughTerms3D];
  double c2[kRoughTerms2D], ph2[kRoughTerms2D];
  double bound;  // max extent (elements) from the centre

  void init(const double* p, bool two_d) {
    is2d = two_d;
    ax[0] = p[0]; ax[1] = p[1]; ax[2] = two_d ? 1.0 : p[2];
    if (two_d) {
      double t = p[3], ct = std::cos(t), st = std::sin(t);
      // d = (dy,dx) -> body (b0,b1)
      R[0] = ct; R[1] = st; R[2] = 0; R[3] = -st; R[4] = ct; R[5] = 0; R[6] = 0; R[7] = 0; R[8] = 1;
    } else {
      double w = p[3], x = p[4], y = p[5], z = p[6];
      double n = std::sqrt(w * w + x * x + y * y + z * z);
      w /= n; x /= n; y /= n; z /= n;
      // rotation matrix of the quaternion (body->world); we store its transpose
      double M[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w),
                     2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w),
                     2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)};
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) R[i * 3 + j] = M[j * 3 + i];
    }
    A = p[7];
    SplitMix rng((uint64_t)p[8] * 0x2545F4914F6CDD1Dull + 17);
    if (!two_d) {
      double tot = 0;
      for (int j = 0; j < kRoughTerms3D; ++j) {
        double a = rng.normal(), b = rng.normal(), cc = rng.normal();
        double nn = std::sqrt(a * a + b * b + cc * cc) + 1e-300;
        v[j][0] = a / nn; v[j][1] = b / nn; v[j][2] = cc / nn;
        f[j] = 1.0 + 2.0 * rng.uniform();
        ph[j] = 6.283185307179586 * rng.uniform();
        c[j] = rng.normal() / f[j];
        tot += std::fabs(c[j]);
      }
      for (int j = 0; j < kRoughTerms3D; ++j) c[j] /= (tot > 0 ? tot : 1);
    } else {
      double tot = 0;
      for (int k = 0; k < kRoughTerms2D; ++k) {
        c2[k] = rng.normal() / (k + 1);
        ph2[k] = 6.283185307179586 * rng.uniform();
        tot += std::fabs(c2[k]);
      }
      for (int k = 0; k < kRoughTerms2D; ++k) c2[k] /= (tot > 0 ? tot : 1);
    }
    double amax = std::max(ax[0], std::max(ax[1], two_d ? 0.0 : ax[2]));
    bound = amax * (1.0 + std::fabs(A));
  }

  // normalised radius^2 relative to the (rough) surface: inside iff <= 1
  double nrad2(double dz, double dy, double dx) const {
    double b0, b1, b2;
    if (is2d) {
      b0 = R[0] * dy + R[1] * dx;
      b1 = R[3] * dy + R[4] * dx;
      b2 = 0;
    } else {
      b0 = R[0] * dz + R[1] * dy + R[2] * dx;
      b1 = R[3] * dz + R[4] * dy + R[5] * dx;
      b2 = R[6] * dz + R[7] * dy + R[8] * dx;
    }
    double q = b0 * b0 / (ax[0] * ax[0]) + b1 * b1 / (ax[1] * ax[1]);
    if (!is2d) q += b2 * b2 / (ax[2] * ax[2]);
    if (A == 0.0) return q;
    double r2 = b0 * b0 + b1 * b1 + b2 * b2;
    double s;
    if (r2 == 0.0) {
      s = 1.0;
    } else if (is2d) {
      double phi = std::atan2(b1, b0), n = 0;
      for (int k = 0; k < kRoughTerms2D; ++k) n += c2[k] * std::cos((k + 1) * phi + ph2[k]);
      s = 1.0 + A * n;
    } else {
      double ir = 1.0 / std::sqrt(r2), n = 0;
      for (int j = 0; j < kRoughTerms3D; ++j) {
        double dotp = (b0 * v[j][0] + b1 * v[j][1] + b2 * v[j][2]) * ir;
        n += c[j] * std::cos(f[j] * 3.141592653589793 * dotp + ph[j]);
      }
      s = 1.0 + A * n;
    }
    return q / (s * s);
  }
};

struct Run {
  int16_t dz, dy, x0, x1;  // inclusive x range, offsets from centre
};

// Element-centre rasterisation of the shape around an integer centre, as x-runs.
void rasterise(const Shape& sh, double scale, std::vector<Run>& runs) {
  runs.clear();
  int B = (int)std::ceil(sh.bound * scale) + 1;
  int bz = sh.is2d ? 0 : B;
  double is2 = 1.0 / (scale * scale);
  for (int dz = -bz; dz <= bz; ++dz)
    for (int dy = -B; dy <= B; ++dy) {
      int start = INT32_MIN;
      for (int dx = -B; dx <= B + 1; ++dx) {
        bool in = dx <= B && sh.nrad2(dz, dy, dx) * is2 <= 1.0;
        if (in && start == INT32_MIN) start = dx;
        if (!in && start != INT32_MIN) {
          runs.push_back(Run{(int16_t)dz, (int16_t)dy, (int16_t)start, (int16_t)(dx - 1)});
          start = INT32_MIN;
        }
      }
    }
}

struct Grid {
  int32_t* g;
  int64_t Z, Y, X;
  int32_t* row(int64_t z, int64_t y) { return g + (z * Y + y) * X; }
};

bool fits(Grid& G, const std::vector<Run>& runs, int64_t cz, int64_t cy, int64_t cx, bool is2d) {
  // footprint dilated by one element must be in-grid and free
  int dzr = is2d ? 0 : 1;
  for (const Run& r : runs) {
    int64_t x0 = cx + r.x0 - 1, x1 = cx + r.x1 + 1;
    if (x0 < 0 || x1 >= G.X) return false;
    for (int dz = -dzr; dz <= dzr; ++dz)
      for (int dy = -1; dy <= 1; ++dy) {
        int64_t z = cz + r.dz + dz, y = cy + r.dy + dy;
        if (z < 0 || z >= G.Z || y < 0 || y >= G.Y) return false;
        const int32_t* row = G.row(z, y);
        for (int64_t x = x0; x <= x1; ++x)
          if (row[x]) return false;
      }
  }
  return true;
}

void paint(Grid& G, const std::vector<Run>& runs, int64_t cz, int64_t cy, int64_t cx, int32_t label) {
  for (const Run& r : runs) {
    int32_t* row = G.row(cz + r.dz, cy + r.dy);
    for (int64_t x = cx + r.x0; x <= cx + r.x1; ++x) row[x] = label;
  }
}

int n_threads() {
  unsigned h = std::thread::hardware_concurrency();
  return h ? (int)std::min(h, 64u) : 4;
}

}  // namespace

extern "C" {

// Place `nobj` objects (params: nobj x 13 doubles, see kParams) into a zeroed grid
// [Z][Y][X] (Z = 1 for 2D), in the given order, labels label_of[i].
// placed[i] receives 1 if object i was placed (0 if dropped), scale_out[i] the shrink
// factor finally used.  Returns the number of placed objects.
int synth_place(int32_t* grid, int64_t Z, int64_t Y, int64_t X, int is2d, int nobj,
                const double* params, const int32_t* label_of, uint64_t seed, int max_tries,
                int32_t* placed, double* scale_out) {
  std::vector<Shape> shapes(nobj);
  for (int i = 0; i < nobj; ++i) shapes[i].init(params + (size_t)i * kParams, is2d != 0);
  // rasterise all objects in parallel at scale 1 (the common case)
  std::vector<std::vector<Run>> runs(nobj);
  {
    std::atomic<int> next(0);
    int nt = n_threads();
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&]() {
        for (int i; (i = next.fetch_add(1)) < nobj;) rasterise(shapes[i], 1.0, runs[i]);
      });
    for (auto& t : th) t.join();
  }
  Grid G{grid, Z, Y, X};
  SplitMix rng(seed ^ 0xA5A5A5A5DEADBEEFull);
  int count = 0;
  for (int i = 0; i < nobj; ++i) {
    const double* p = params + (size_t)i * kParams;
    double scale = 1.0;
    bool ok = false;
    std::vector<Run> local;
    const std::vector<Run>* rr = &runs[i];
    for (int attempt = 0; attempt < 13 && !ok; ++attempt) {
      if (attempt > 0) {
        scale *= 0.85;
        rasterise(shapes[i], scale, local);
        rr = &local;
      }
      if (rr->empty()) break;
      int mz = 0, my = 0, mx = 0;
      for (const Run& r : *rr) {
        mz = std::max(mz, std::abs((int)r.dz));
        my = std::max(my, std::abs((int)r.dy));
        mx = std::max(mx, std::max(std::abs((int)r.x0), std::abs((int)r.x1)));
      }
      if (p[12] != 0.0) {
        int64_t cz = (int64_t)p[9], cy = (int64_t)p[10], cx = (int64_t)p[11];
        if (fits(G, *rr, cz, cy, cx, is2d != 0)) {
          paint(G, *rr, cz, cy, cx, label_of[i]);
          ok = true;
        }
        continue;
      }
      int64_t lz = is2d ? 0 : mz + 1, hz = is2d ? 0 : Z - mz - 2;
      int64_t ly = my + 1, hy = Y - my - 2, lx = mx + 1, hx = X - mx - 2;
      if (hz < lz || hy < ly || hx < lx) continue;
      for (int t = 0; t < max_tries; ++t) {
        int64_t cz = lz + (int64_t)(rng.uniform() * (hz - lz + 1));
        int64_t cy = ly + (int64_t)(rng.uniform() * (hy - ly + 1));
        int64_t cx = lx + (int64_t)(rng.uniform() * (hx - lx + 1));
        if (fits(G, *rr, cz, cy, cx, is2d != 0)) {
          paint(G, *rr, cz, cy, cx, label_of[i]);
          ok = true;
          break;
        }
      }
    }
    placed[i] = ok ? 1 : 0;
    scale_out[i] = scale;
    count += ok;
  }
  return count;
}

// Touching 2D cells, one image per batch item: grid [B][Y][X]; params: B*ncell x 13
// (fixed centre fields used as the centre); labels 1..ncell per image.
void synth_cells(int32_t* grid, int64_t B, int64_t Y, int64_t X, int ncell, const double* params) {
  std::atomic<int64_t> next(0);
  int nt = n_threads();
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&]() {
      std::vector<float> best((size_t)(Y * X));
      for (int64_t b; (b = next.fetch_add(1)) < B;) {
        int32_t* img = grid + b * Y * X;
        std::fill(best.begin(), best.end(), 2.0f);
        std::memset(img, 0, sizeof(int32_t) * Y * X);
        for (int k = 0; k < ncell; ++k) {
          const double* p = params + ((size_t)b * ncell + k) * kParams;
          Shape sh;
          sh.init(p, true);
          double cy = p[10], cx = p[11];
          int Bd = (int)std::ceil(sh.bound) + 1;
          int64_t y0 = std::max<int64_t>(0, (int64_t)std::floor(cy) - Bd);
          int64_t y1 = std::min<int64_t>(Y - 1, (int64_t)std::ceil(cy) + Bd);
          int64_t x0 = std::max<int64_t>(0, (int64_t)std::floor(cx) - Bd);
          int64_t x1 = std::min<int64_t>(X - 1, (int64_t)std::ceil(cx) + Bd);
          for (int64_t y = y0; y <= y1; ++y)
            for (int64_t x = x0; x <= x1; ++x) {
              double r2 = sh.nrad2(0, (double)y - cy, (double)x - cx);
              if (r2 > 1.0) continue;
              float r = (float)std::sqrt(r2);
              size_t o = (size_t)(y * X + x);
              if (r < best[o]) {
                best[o] = r;
                img[o] = k + 1;
              }
            }
        }
      }
    });
  for (auto& t : th) t.join();
}

}  // extern "C"
