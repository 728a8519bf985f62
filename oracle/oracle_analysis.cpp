// ORACLE, analysis protocol part — plain CPU definitions of the SURVEY.md §8(f) rows around the
// hot path.  *** TEST INFRASTRUCTURE ONLY *** (same rules as oracle.cpp: only tests/,
// __graft_entry__.smoke() and bench.py's CPU legs load it; it shares nothing with csrc/).
//
//   label_components   connected-component labelling of a binary mask (SPEC.md:205-211
//                      label_components; "segmenting and labeling each fat
//                      component"): per batch item, labels 1..K in the order of first encounter
//                      in a row-major scan; connectivity 4 / 8 (2D), 6 / 18 / 26 (3D).  Plain
//                      breadth-first flood fill from each first-encountered element.
//   sphericity_wl      Eq. 3 width-to-length sphericity S = d2 / d1, 2D, with
//                      SPEC.md:355-361's reading: d1, d2 = 4 sqrt(eigenvalues) of the object's
//                      pixel-coordinate covariance (population, 1/n; exact for a continuum
//                      ellipse: 4 sqrt(lambda) = the full axis); a single pixel gives 1.0.
//                      Two-pass mean / covariance in double.
//   mc_measure         the S_MC baseline of PAPER.md:211 (§5.2) and PAPER.md:274 (Fig. 6a):
//                      2D perimeter of the iso-0.5 contour of each object's binary mask by
//                      marching squares with linear interpolation (every crossing of a binary
//                      field is an edge midpoint; the saddle cases give two segments of
//                      sqrt(2)/2 either way, so the length needs no saddle convention); 3D
//                      surface area of the iso-0.5 surface by marching cubes built from its
//                      definition rather than a case table: on each cube face the edge-midpoint
//                      crossings are joined into segments (a face with two diagonal inside
//                      corners gets one segment around each inside corner -- the same rule in
//                      the two cubes sharing the face, so the surface is watertight), the
//                      segments of the 6 faces close into loops, and each loop's area is the
//                      fan of triangles (centroid, v_i, v_i+1).  (Reading: the paper used
//                      scikit-image's marching cubes; its case table and interior-ambiguity
//                      resolution are not reproduced -- DESIGN.md "Readings".)
//                      Outside the grid counts as background, so every object is closed.
//                      sphericity_mc = Eq. 1 with S = area (3D) / Eq. 2 with P_o = perimeter.
// Pins: tests/test_oracle_analysis.py (scipy.ndimage.label, SPEC.md examples, closed forms for
// rectangles, single pixel / voxel, squares; convergence to the analytic circle / sphere).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <deque>
#include <vector>

namespace {

constexpr double kPiA = 3.14159265358979323846;

struct G {
  int ndim;
  int64_t B, Z, Y, X;
};

bool geom(const int64_t* dims, int ndim, int64_t batch, G& g) {
  if (!dims || (ndim != 2 && ndim != 3) || batch < 1) return false;
  g.ndim = ndim;
  g.B = batch;
  g.Z = ndim == 3 ? dims[0] : 1;
  g.Y = dims[ndim - 2];
  g.X = dims[ndim - 1];
  return g.Z >= 1 && g.Y >= 1 && g.X >= 1;
}

}  // namespace

extern "C" {

// labels_out: int32 like mask; counts_out: batch entries (number of components per item)
int fastrs_oracle_label_components(const uint8_t* mask, const int64_t* dims, int ndim, int64_t batch,
                                   int connectivity, int32_t* labels_out, int64_t* counts_out) {
  G g;
  if (!mask || !labels_out || !geom(dims, ndim, batch, g)) return 1;
  const bool ok = ndim == 2 ? (connectivity == 4 || connectivity == 8)
                            : (connectivity == 6 || connectivity == 18 || connectivity == 26);
  if (!ok) return 1;
  // neighbour offsets of the connectivity (|dz| + |dy| + |dx| bounded: 1 face, 2 edge, 3 corner)
  std::vector<int> off;
  const int maxsum = (ndim == 2) ? (connectivity == 4 ? 1 : 2) : (connectivity == 6 ? 1 : connectivity == 18 ? 2 : 3);
  for (int dz = (ndim == 3 ? -1 : 0); dz <= (ndim == 3 ? 1 : 0); ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int s = std::abs(dz) + std::abs(dy) + std::abs(dx);
        if (s == 0 || s > maxsum) continue;
        off.push_back(dz);
        off.push_back(dy);
        off.push_back(dx);
      }
  const int64_t vol = g.Z * g.Y * g.X;
  for (int64_t b = 0; b < g.B; ++b) {
    const uint8_t* m = mask + b * vol;
    int32_t* L = labels_out + b * vol;
    for (int64_t i = 0; i < vol; ++i) L[i] = 0;
    int32_t next = 0;
    std::deque<int64_t> q;
    for (int64_t i = 0; i < vol; ++i) {  // row-major scan: the first unlabelled element starts a component
      if (!m[i] || L[i]) continue;
      L[i] = ++next;
      q.push_back(i);
      while (!q.empty()) {
        const int64_t p = q.front();
        q.pop_front();
        const int64_t z = p / (g.Y * g.X), y = (p / g.X) % g.Y, x = p % g.X;
        for (size_t k = 0; k < off.size(); k += 3) {
          const int64_t zz = z + off[k], yy = y + off[k + 1], xx = x + off[k + 2];
          if (zz < 0 || zz >= g.Z || yy < 0 || yy >= g.Y || xx < 0 || xx >= g.X) continue;
          const int64_t j = (zz * g.Y + yy) * g.X + xx;
          if (m[j] && !L[j]) {
            L[j] = next;
            q.push_back(j);
          }
        }
      }
    }
    if (counts_out) counts_out[b] = next;
  }
  return 0;
}

// 2D only.  swl, d1, d2: batch*max_label (nullable each); absent labels NaN.
int fastrs_oracle_sphericity_wl(const int32_t* labels, const int64_t* dims, int ndim, int64_t batch,
                                int32_t max_label, double* swl, double* d1, double* d2) {
  G g;
  if (!labels || ndim != 2 || !geom(dims, ndim, batch, g) || max_label < 1) return 1;
  const int64_t M = max_label, area = g.Y * g.X;
  for (int64_t b = 0; b < g.B; ++b) {
    std::vector<double> n(M, 0), sx(M, 0), sy(M, 0);
    const int32_t* Lb = labels + b * area;
    for (int64_t y = 0; y < g.Y; ++y)
      for (int64_t x = 0; x < g.X; ++x) {
        const int32_t L = Lb[y * g.X + x];
        if (L < 1 || L > max_label) continue;
        n[L - 1] += 1;
        sx[L - 1] += (double)x;
        sy[L - 1] += (double)y;
      }
    std::vector<double> cxx(M, 0), cyy(M, 0), cxy(M, 0);
    for (int64_t y = 0; y < g.Y; ++y)  // second pass: deviations from the mean
      for (int64_t x = 0; x < g.X; ++x) {
        const int32_t L = Lb[y * g.X + x];
        if (L < 1 || L > max_label) continue;
        const double mx = sx[L - 1] / n[L - 1], my = sy[L - 1] / n[L - 1];
        cxx[L - 1] += (x - mx) * (x - mx);
        cyy[L - 1] += (y - my) * (y - my);
        cxy[L - 1] += (x - mx) * (y - my);
      }
    for (int64_t k = 0; k < M; ++k) {
      double s = NAN, a = NAN, c = NAN;
      if (n[k] > 0) {
        const double vx = cxx[k] / n[k], vy = cyy[k] / n[k], vxy = cxy[k] / n[k];
        const double h = 0.5 * (vx + vy), r = std::sqrt(0.25 * (vx - vy) * (vx - vy) + vxy * vxy);
        const double l1 = h + r, l2 = std::max(h - r, 0.0);
        a = 4.0 * std::sqrt(l1);
        c = 4.0 * std::sqrt(l2);
        s = l1 > 0 ? c / a : 1.0;  // a single pixel: 1 by convention
      }
      const int64_t i = b * M + k;
      if (swl) swl[i] = s;
      if (d1) d1[i] = a;
      if (d2) d2[i] = c;
    }
  }
  return 0;
}

namespace {

struct V3 {
  double x, y, z;
};
V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
V3 mid(V3 a, V3 b) { return {0.5 * (a.x + b.x), 0.5 * (a.y + b.y), 0.5 * (a.z + b.z)}; }
double cross_norm(V3 a, V3 b) {
  const double cx = a.y * b.z - a.z * b.y, cy = a.z * b.x - a.x * b.z, cz = a.x * b.y - a.y * b.x;
  return std::sqrt(cx * cx + cy * cy + cz * cz);
}

// cube corner q = (x, y, z) bits (x = q & 1, y = (q >> 1) & 1, z = (q >> 2) & 1)
V3 corner(int q) { return {(double)(q & 1), (double)((q >> 1) & 1), (double)((q >> 2) & 1)}; }

// iso-0.5 surface area inside one unit cube with binary corner values in[8] (see the header)
double cube_area(const bool in[8]) {
  // the 6 faces, corners in cyclic order
  static const int faces[6][4] = {{0, 1, 3, 2}, {4, 5, 7, 6}, {0, 1, 5, 4}, {2, 3, 7, 6}, {0, 2, 6, 4}, {1, 3, 7, 5}};
  // crossing points are identified by their edge (corner pair a < b); segments join two of them
  std::vector<std::pair<int, int>> seg;  // edge keys a * 8 + b
  auto key = [](int a, int b) { return a < b ? a * 8 + b : b * 8 + a; };
  for (const auto& f : faces) {
    int ninside = 0;
    for (int i = 0; i < 4; ++i) ninside += in[f[i]];
    if (ninside == 0 || ninside == 4) continue;
    const bool saddle = ninside == 2 && in[f[0]] == in[f[2]];
    if (saddle) {  // one segment around each inside corner
      for (int i = 0; i < 4; ++i)
        if (in[f[i]]) seg.push_back({key(f[i], f[(i + 3) % 4]), key(f[i], f[(i + 1) % 4])});
    } else {  // exactly two crossings on the face
      int e[2], n = 0;
      for (int i = 0; i < 4; ++i)
        if (in[f[i]] != in[f[(i + 1) % 4]]) e[n++] = key(f[i], f[(i + 1) % 4]);
      seg.push_back({e[0], e[1]});
    }
  }
  // close the segments into loops and sum the loops' centroid-fan areas
  std::vector<bool> used(seg.size(), false);
  double area = 0;
  for (size_t s0 = 0; s0 < seg.size(); ++s0) {
    if (used[s0]) continue;
    std::vector<int> loop;
    used[s0] = true;
    loop.push_back(seg[s0].first);
    int cur = seg[s0].second;
    while (cur != loop[0]) {
      loop.push_back(cur);
      for (size_t t = 0; t < seg.size(); ++t)
        if (!used[t] && (seg[t].first == cur || seg[t].second == cur)) {
          used[t] = true;
          cur = seg[t].first == cur ? seg[t].second : seg[t].first;
          break;
        }
    }
    std::vector<V3> v;
    V3 c = {0, 0, 0};
    for (int k : loop) {
      v.push_back(mid(corner(k / 8), corner(k % 8)));
      c.x += v.back().x;
      c.y += v.back().y;
      c.z += v.back().z;
    }
    c = {c.x / v.size(), c.y / v.size(), c.z / v.size()};
    for (size_t i = 0; i < v.size(); ++i) area += 0.5 * cross_norm(sub(v[i], c), sub(v[(i + 1) % v.size()], c));
  }
  return area;
}

}  // namespace

// measure: batch*max_label (perimeter in 2D, surface area in 3D); smc (nullable): S_MC
int fastrs_oracle_mc_measure(const int32_t* labels, const int64_t* dims, int ndim, int64_t batch, int32_t max_label,
                             double* measure, double* smc) {
  G g;
  if (!labels || !measure || !geom(dims, ndim, batch, g) || max_label < 1) return 1;
  const int64_t M = max_label, vol = g.Z * g.Y * g.X;
  for (int64_t b = 0; b < g.B; ++b) {
    const int32_t* Lb = labels + b * vol;
    auto lab = [&](int64_t z, int64_t y, int64_t x) -> int32_t {  // outside the grid: background
      if (z < 0 || z >= g.Z || y < 0 || y >= g.Y || x < 0 || x >= g.X) return 0;
      return Lb[(z * g.Y + y) * g.X + x];
    };
    std::vector<double> meas(M, 0.0), count(M, 0.0);
    for (int64_t i = 0; i < vol; ++i)
      if (Lb[i] >= 1 && Lb[i] <= max_label) count[Lb[i] - 1] += 1;
    if (ndim == 2) {
      for (int64_t y = -1; y < g.Y; ++y)
        for (int64_t x = -1; x < g.X; ++x) {
          const int32_t c[4] = {lab(0, y, x), lab(0, y, x + 1), lab(0, y + 1, x + 1), lab(0, y + 1, x)};  // cyclic
          for (int t = 0; t < 4; ++t) {
            const int32_t k = c[t];
            bool seen = false;
            for (int u = 0; u < t; ++u) seen |= c[u] == k;
            if (k < 1 || k > max_label || seen) continue;
            bool in[4];
            int n = 0;
            for (int u = 0; u < 4; ++u) n += (in[u] = c[u] == k);
            double len = 0;
            if (n == 1 || n == 3) len = std::sqrt(0.5);                   // one corner cut off
            else if (n == 2) len = (in[0] == in[2]) ? 2 * std::sqrt(0.5)  // diagonal: two corners cut
                                                    : 1.0;                // a straight segment
            meas[k - 1] += len;
          }
        }
    } else {
      for (int64_t z = -1; z < g.Z; ++z)
        for (int64_t y = -1; y < g.Y; ++y)
          for (int64_t x = -1; x < g.X; ++x) {
            int32_t c[8];  // corner (i,j,k) at index i + 2j + 4k (x, y, z bits)
            for (int q = 0; q < 8; ++q) c[q] = lab(z + ((q >> 2) & 1), y + ((q >> 1) & 1), x + (q & 1));
            for (int t = 0; t < 8; ++t) {
              const int32_t k = c[t];
              bool seen = false;
              for (int u = 0; u < t; ++u) seen |= c[u] == k;
              if (k < 1 || k > max_label || seen) continue;
              bool in[8];
              for (int q = 0; q < 8; ++q) in[q] = c[q] == k;
              meas[k - 1] += cube_area(in);
            }
          }
    }
    for (int64_t k = 0; k < M; ++k) {
      const int64_t i = b * M + k;
      measure[i] = count[k] > 0 ? meas[k] : NAN;
      if (smc) {
        double s = NAN;
        if (count[k] > 0) {
          if (ndim == 3) s = std::cbrt(kPiA) * std::pow(6.0 * count[k], 2.0 / 3.0) / meas[k];  // Eq. 1
          else s = 2.0 * std::sqrt(kPiA * count[k]) / meas[k];                                  // Eq. 2, P_c / P_o
        }
        smc[i] = s;
      }
    }
  }
  return 0;
}

}  // extern "C"
