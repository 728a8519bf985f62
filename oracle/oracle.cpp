// ORACLE — plain, slow, obviously-correct CPU implementation of the paper's definitions.
//
// *** TEST INFRASTRUCTURE ONLY. ***  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library.  It shares no code, headers,
// tables or helpers with the CUDA path (paper_2504_05808_b200/csrc), and neither side
// includes or links the other.
//
// What it computes (readings c1..c17 listed in DESIGN.md "Readings"):
// per batch item and per label k >= 1 with V_k > 0
//   sites    S_k = every element whose label != k, plus (flag BORDER_BACKGROUND) the virtual
//            layer just outside the grid                         [reading c6, c7]
//   EDT      D(p) = min_{s in S_k} |p - s|^2, centre-to-centre    [SPEC.md:88; reading c4]
//   LT       LT^2(p) = max{ D(q) : label(q)=k, |p-q|^2 < D(q) }  [PAPER.md:11,85; reading c5]
//            lt(p) = sqrt((double)LT^2(p))                        [reading c3: a radius]
//   shell    p has a face neighbour (4-conn 2D / 6-conn 3D) with label != k, or outside the
//            grid when BORDER_BACKGROUND                          [PAPER.md:148,150; c8, c9]
//   V        = #elements                                          [PAPER.md:124]
//   a        = mean lt over the object                            [PAPER.md:124,133; c10]
//   R_max    = max lt; r_bar = mean lt over the shell             [PAPER.md:142,148; c11]
//   3D       c = 3V/(4 pi a^2) (Eq. 8), S_area = Eqs. 6-7 with e = sqrt(1-c^2/a^2) or
//            sqrt(1-a^2/c^2) (reading c1), sphericity = pi^(1/3)(6V)^(2/3)/S_area (Eq. 1)
//   2D       b = A/(pi a) (Eq. 10), P_o = Ramanujan I (Eq. 9), P_c = 2 sqrt(pi A) (Eq. 11),
//            sphericity = P_c / P_o (Eq. 2)
//   roundness = r_bar / R_max                                     [PAPER.md:142-152]
//
// Algorithm, deliberately plain: bounding boxes by one scan; then per object (thread pool
// over objects) crop bbox +- 1 ("crop exactness"); EDT by brute force over
// every site of the crop when the crop has <= 4096 elements, else the textbook separable
// squared EDT with an O(len^2) minimum over ALL positions of each line; LT by painting EVERY
// object element's ball (no pruning); shell by the neighbour definition (NOT via D == 1);
// sums in float64 with Neumaier compensation; closed forms in float64.
//
// Parity pins (tests/test_oracle_*.py): brute-force EDT and brute-force all-balls LT on
// tiny random grids, scipy's EDT on separated labels, SPEC worked examples, digital
// disk r=20 / sphere r=15 closed forms, numeric-integral spheroid areas, elliptic-integral
// perimeters, invariants.  No function here is "parity unpinned".

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

namespace {

constexpr uint32_t kFlagBorderBackground = 1u;
constexpr uint64_t kInf = std::numeric_limits<uint64_t>::max() / 4;
constexpr double kPi = 3.14159265358979323846;

enum { OK = 0, EINVAL_ = 1, ENOSITE_ = 2, EINTERNAL_ = 6 };

struct Geometry {
  int ndim;
  int64_t batch, Z, Y, X;  // 2D: Z = 1
  int64_t plane() const { return Y * X; }
  int64_t volume() const { return Z * Y * X; }
};

bool make_geometry(const int64_t* dims, int ndim, int64_t batch, Geometry& g) {
  if (!dims || (ndim != 2 && ndim != 3) || batch < 1) return false;
  g.ndim = ndim;
  g.batch = batch;
  g.Z = ndim == 3 ? dims[0] : 1;
  g.Y = dims[ndim - 2];
  g.X = dims[ndim - 1];
  return g.Z >= 1 && g.Y >= 1 && g.X >= 1;
}

struct BBox {
  int64_t lo[3] = {INT64_MAX, INT64_MAX, INT64_MAX};
  int64_t hi[3] = {INT64_MIN, INT64_MIN, INT64_MIN};
  int64_t count = 0;
};

// One object's crop: bbox +- 1 on every axis (clamped to [-1, dim] with the border flag,
// to [0, dim-1] without: elements outside the grid exist only as border sites).
struct Crop {
  int64_t o[3];  // origin (z,y,x) in grid coordinates
  int64_t n[3];  // extent
  int64_t size() const { return n[0] * n[1] * n[2]; }
};

enum Cell : uint8_t { VOID = 0, SITE = 1, OBJ = 2 };

struct Object {
  int64_t b;
  int32_t label;
  BBox box;
};

// ---------------------------------------------------------------------------------------
// closed forms (§2.1, §4.1, §4.2)
// ---------------------------------------------------------------------------------------

// Eqs. 6-7 with reading c1: e is the eccentricity sqrt(1-c^2/a^2) /
// sqrt(1-a^2/c^2); reading c12: branch as printed, 1-e^2 taken as c^2/a^2, e == 0 -> sphere.
double spheroid_area(double a, double c) {
  if (c < a) {
    double one_minus_e2 = (c * c) / (a * a);
    double e = std::sqrt(1.0 - one_minus_e2);
    if (e == 0.0) return 4.0 * kPi * a * a;
    return 2.0 * kPi * a * a * (1.0 + one_minus_e2 / e * std::atanh(e));  // Eq. 6
  }
  double e = std::sqrt(1.0 - (a * a) / (c * c));
  if (e == 0.0) return 4.0 * kPi * a * a;
  return 2.0 * kPi * a * a * (1.0 + c / (a * e) * std::asin(e));  // Eq. 7
}

// Eq. 9, Ramanujan's first approximation.
double ramanujan_perimeter(double a, double b) {
  return kPi * (3.0 * (a + b) - std::sqrt((3.0 * a + b) * (a + 3.0 * b)));
}

// Eq. 1 with Eq. 8: a_s = mean LT, c_s = 3V/(4 pi a_s^2).
double sphericity_3d(double V, double mean_lt) {
  double a = mean_lt;
  double c = 3.0 * V / (4.0 * kPi * a * a);
  return std::pow(kPi, 1.0 / 3.0) * std::pow(6.0 * V, 2.0 / 3.0) / spheroid_area(a, c);
}

// Eq. 2 with Eqs. 9-11: a_e = mean LT, b_e = A/(pi a_e).
double sphericity_2d(double A, double mean_lt) {
  double a = mean_lt;
  double b = A / (kPi * a);
  double Pc = 2.0 * std::sqrt(kPi * A);
  double Po = ramanujan_perimeter(a, b);
  return Pc / Po;
}

// Neumaier-compensated float64 sum.
struct KSum {
  double s = 0.0, c = 0.0;
  void add(double x) {
    double t = s + x;
    if (std::fabs(s) >= std::fabs(x))
      c += (s - t) + x;
    else
      c += (x - t) + s;
    s = t;
  }
  double value() const { return s + c; }
};

// ---------------------------------------------------------------------------------------
// per-object work
// ---------------------------------------------------------------------------------------

struct ObjectResult {
  int64_t volume = 0, n_shell = 0;
  uint32_t max_lt2 = 0;
  double sum_lt = 0, sum_shell_lt = 0;
  int status = OK;
};

struct Ctx {
  const int32_t* labels;
  Geometry g;
  uint32_t flags;
  uint32_t* d2_out;   // nullable, full grid
  uint32_t* lt2_out;  // nullable, full grid
  uint8_t* shell_out; // nullable, full grid
};

inline int32_t label_at(const Ctx& C, int64_t b, int64_t z, int64_t y, int64_t x) {
  return C.labels[((b * C.g.Z + z) * C.g.Y + y) * C.g.X + x];
}

ObjectResult process_object(const Ctx& C, const Object& ob) {
  ObjectResult res;
  const Geometry& g = C.g;
  const bool border = (C.flags & kFlagBorderBackground) != 0;
  const int64_t dims[3] = {g.Z, g.Y, g.X};
  const int nax = g.ndim;  // number of real axes; in 2D the z axis has extent 1, no crop
  Crop cr;
  for (int a = 0; a < 3; ++a) {
    bool real_axis = (a > 0) || nax == 3;
    int64_t lo = ob.box.lo[a], hi = ob.box.hi[a];
    if (real_axis) {
      lo -= 1;
      hi += 1;
      int64_t mn = border ? -1 : 0, mx = border ? dims[a] : dims[a] - 1;
      lo = std::max(lo, mn);
      hi = std::min(hi, mx);
    }
    cr.o[a] = lo;
    cr.n[a] = hi - lo + 1;
  }
  const int64_t n0 = cr.n[0], n1 = cr.n[1], n2 = cr.n[2], N = cr.size();
  auto idx = [&](int64_t i, int64_t j, int64_t k) { return (i * n1 + j) * n2 + k; };

  // classify the crop
  std::vector<uint8_t> cell(N);
  for (int64_t i = 0; i < n0; ++i)
    for (int64_t j = 0; j < n1; ++j)
      for (int64_t k = 0; k < n2; ++k) {
        int64_t z = cr.o[0] + i, y = cr.o[1] + j, x = cr.o[2] + k;
        uint8_t c;
        if (z < 0 || z >= g.Z || y < 0 || y >= g.Y || x < 0 || x >= g.X)
          c = border ? SITE : VOID;
        else
          c = label_at(C, ob.b, z, y, x) == ob.label ? OBJ : SITE;
        cell[idx(i, j, k)] = c;
      }

  // ---- EDT ------------------------------------------------------------------------------
  std::vector<uint64_t> D(N, kInf);
  if (N <= 4096) {
    // brute force over every site of the crop
    std::vector<int64_t> sites;
    for (int64_t t = 0; t < N; ++t)
      if (cell[t] == SITE) sites.push_back(t);
    for (int64_t t = 0; t < N; ++t) {
      if (cell[t] != OBJ) continue;
      int64_t i = t / (n1 * n2), j = (t / n2) % n1, k = t % n2;
      uint64_t best = kInf;
      for (int64_t s : sites) {
        int64_t si = s / (n1 * n2), sj = (s / n2) % n1, sk = s % n2;
        uint64_t d = (uint64_t)((i - si) * (i - si) + (j - sj) * (j - sj) + (k - sk) * (k - sk));
        best = std::min(best, d);
      }
      D[t] = best;
    }
  } else {
    // textbook separable squared EDT: f = 0 on sites, inf elsewhere; per axis
    // h(i) = min over ALL j of f(j) + (i-j)^2, in O(len^2).
    for (int64_t t = 0; t < N; ++t) D[t] = cell[t] == SITE ? 0 : kInf;
    const int64_t ext[3] = {n0, n1, n2};
    const int64_t stride[3] = {n1 * n2, n2, 1};
    std::vector<uint64_t> line, outl;
    for (int a = 2; a >= 0; --a) {
      int64_t len = ext[a];
      if (len == 1) continue;
      line.resize(len);
      outl.resize(len);
      int b1 = (a + 1) % 3, b2 = (a + 2) % 3;
      for (int64_t u = 0; u < ext[b1]; ++u)
        for (int64_t v = 0; v < ext[b2]; ++v) {
          int64_t base = u * stride[b1] + v * stride[b2];
          for (int64_t i = 0; i < len; ++i) line[i] = D[base + i * stride[a]];
          for (int64_t i = 0; i < len; ++i) {
            uint64_t best = kInf;
            for (int64_t j = 0; j < len; ++j) {
              if (line[j] >= kInf) continue;
              uint64_t d = line[j] + (uint64_t)((i - j) * (i - j));
              best = std::min(best, d);
            }
            outl[i] = best;
          }
          for (int64_t i = 0; i < len; ++i) D[base + i * stride[a]] = outl[i];
        }
    }
  }
  for (int64_t t = 0; t < N; ++t)
    if (cell[t] == OBJ && D[t] >= kInf) res.status = ENOSITE_;
  if (res.status != OK) return res;

  // ---- LT: paint every object element's ball, strict |p-q|^2 < D(q) -----------------------
  std::vector<uint32_t> lt2(N, 0);
  for (int64_t i = 0; i < n0; ++i)
    for (int64_t j = 0; j < n1; ++j)
      for (int64_t k = 0; k < n2; ++k) {
        int64_t t = idx(i, j, k);
        if (cell[t] != OBJ) continue;
        int64_t Dq = (int64_t)D[t];
        int64_t r = (int64_t)std::sqrt((double)(Dq - 1));
        while (r * r > Dq - 1) --r;
        while ((r + 1) * (r + 1) <= Dq - 1) ++r;
        for (int64_t di = -r; di <= r; ++di) {
          int64_t ii = i + di;
          if (ii < 0 || ii >= n0) continue;
          for (int64_t dj = -r; dj <= r; ++dj) {
            int64_t jj = j + dj;
            if (jj < 0 || jj >= n1) continue;
            int64_t rem = Dq - 1 - di * di - dj * dj;
            if (rem < 0) continue;
            for (int64_t kk = std::max<int64_t>(0, k - r); kk <= std::min<int64_t>(n2 - 1, k + r); ++kk) {
              int64_t dk = kk - k;
              if (dk * dk > rem) continue;
              int64_t p = idx(ii, jj, kk);
              if (cell[p] != OBJ) {  // a ball inside the object never reaches a site
                res.status = EINTERNAL_;
                return res;
              }
              if ((uint32_t)Dq > lt2[p]) lt2[p] = (uint32_t)Dq;
            }
          }
        }
      }

  // ---- shell (neighbour definition) and aggregates ----------------------------------------
  KSum s_all, s_shell;
  for (int64_t i = 0; i < n0; ++i)
    for (int64_t j = 0; j < n1; ++j)
      for (int64_t k = 0; k < n2; ++k) {
        int64_t t = idx(i, j, k);
        if (cell[t] != OBJ) continue;
        int64_t z = cr.o[0] + i, y = cr.o[1] + j, x = cr.o[2] + k;
        bool shell = false;
        const int64_t pos[3] = {z, y, x};
        for (int a = 0; a < 3 && !shell; ++a) {
          if (a == 0 && nax == 2) continue;
          for (int sgn = -1; sgn <= 1; sgn += 2) {
            int64_t q[3] = {pos[0], pos[1], pos[2]};
            q[a] += sgn;
            if (q[a] < 0 || q[a] >= dims[a]) {
              if (border) shell = true;
            } else if (label_at(C, ob.b, q[0], q[1], q[2]) != ob.label) {
              shell = true;
            }
          }
        }
        double lt = std::sqrt((double)lt2[t]);
        res.volume += 1;
        s_all.add(lt);
        res.max_lt2 = std::max(res.max_lt2, lt2[t]);
        if (shell) {
          res.n_shell += 1;
          s_shell.add(lt);
        }
        int64_t gi = ((ob.b * g.Z + z) * g.Y + y) * g.X + x;
        if (C.d2_out) C.d2_out[gi] = (uint32_t)D[t];
        if (C.lt2_out) C.lt2_out[gi] = lt2[t];
        if (C.shell_out) C.shell_out[gi] = shell ? 1 : 0;
      }
  res.sum_lt = s_all.value();
  res.sum_shell_lt = s_shell.value();
  return res;
}

int run(const Ctx& C, int32_t max_label, const uint8_t* label_mask, int nthreads,
        std::vector<Object>& objs, std::vector<ObjectResult>& results) {
  const Geometry& g = C.g;
  // bounding boxes, one scan
  std::vector<BBox> boxes((size_t)g.batch * max_label);
  for (int64_t b = 0; b < g.batch; ++b)
    for (int64_t z = 0; z < g.Z; ++z)
      for (int64_t y = 0; y < g.Y; ++y)
        for (int64_t x = 0; x < g.X; ++x) {
          int32_t L = label_at(C, b, z, y, x);
          if (L == 0) continue;
          if (L < 0 || L > max_label) return EINVAL_;
          BBox& bb = boxes[(size_t)b * max_label + (L - 1)];
          const int64_t p[3] = {z, y, x};
          for (int a = 0; a < 3; ++a) {
            bb.lo[a] = std::min(bb.lo[a], p[a]);
            bb.hi[a] = std::max(bb.hi[a], p[a]);
          }
          bb.count += 1;
        }
  for (int64_t b = 0; b < g.batch; ++b)
    for (int32_t L = 1; L <= max_label; ++L) {
      size_t id = (size_t)b * max_label + (L - 1);
      if (boxes[id].count == 0) continue;
      if (label_mask && !label_mask[id]) continue;
      objs.push_back(Object{b, L, boxes[id]});
    }
  // big objects first for load balance
  std::vector<size_t> order(objs.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::sort(order.begin(), order.end(),
            [&](size_t a, size_t b) { return objs[a].box.count > objs[b].box.count; });
  results.assign(objs.size(), ObjectResult{});
  std::atomic<size_t> next(0);
  int nt = nthreads > 0 ? nthreads : (int)std::max(1u, std::thread::hardware_concurrency());
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&]() {
      for (size_t i; (i = next.fetch_add(1)) < order.size();)
        results[order[i]] = process_object(C, objs[order[i]]);
    });
  for (auto& t : th) t.join();
  int status = OK;
  for (auto& r : results)
    if (r.status != OK) status = std::max(status, r.status);
  return status;
}

}  // namespace

extern "C" {

// Full-grid squared EDT (0 on background).  Returns 0 / 1 EINVAL / 2 ENOSITE.
int fastrs_oracle_edt_sq(const int32_t* labels, const int64_t* dims, int ndim, int64_t batch,
                         uint32_t flags, uint32_t* d2_out, int nthreads) {
  Geometry g;
  if (!labels || !d2_out || !make_geometry(dims, ndim, batch, g)) return EINVAL_;
  size_t n = (size_t)(g.batch * g.volume());
  std::memset(d2_out, 0, sizeof(uint32_t) * n);
  int32_t max_label = 0;
  for (size_t i = 0; i < n; ++i) {
    if (labels[i] < 0) return EINVAL_;
    max_label = std::max(max_label, labels[i]);
  }
  if (max_label == 0) return OK;
  Ctx C{labels, g, flags, d2_out, nullptr, nullptr};
  std::vector<Object> objs;
  std::vector<ObjectResult> res;
  return run(C, max_label, nullptr, nthreads, objs, res);
}

// Full-grid LT^2 and (optionally) D and shell mask.  max_label bounds the labels.
int fastrs_oracle_fields(const int32_t* labels, const int64_t* dims, int ndim, int64_t batch,
                         int32_t max_label, uint32_t flags, uint32_t* d2_out, uint32_t* lt2_out,
                         uint8_t* shell_out, int nthreads) {
  Geometry g;
  if (!labels || !make_geometry(dims, ndim, batch, g) || max_label < 0) return EINVAL_;
  size_t n = (size_t)(g.batch * g.volume());
  if (d2_out) std::memset(d2_out, 0, 4 * n);
  if (lt2_out) std::memset(lt2_out, 0, 4 * n);
  if (shell_out) std::memset(shell_out, 0, n);
  Ctx C{labels, g, flags, d2_out, lt2_out, shell_out};
  std::vector<Object> objs;
  std::vector<ObjectResult> res;
  return run(C, max_label, nullptr, nthreads, objs, res);
}

// Per-object sphericity and roundness (and stats).  Output arrays have batch*max_label
// entries, index b*max_label + (label-1); labels with V = 0, or not selected by the
// optional label_mask, get NaN metrics and zero counts.  Any output pointer may be null.
int fastrs_oracle_sphericity_roundness(const int32_t* labels, const int64_t* dims, int ndim,
                                       int64_t batch, int32_t max_label, uint32_t flags,
                                       double* sphericity, double* roundness, int64_t* volume,
                                       int64_t* n_shell, uint32_t* max_lt2, double* mean_lt,
                                       double* shell_mean_lt, double* axis_a, double* axis_cb,
                                       const uint8_t* label_mask, int nthreads) {
  Geometry g;
  if (!labels || !make_geometry(dims, ndim, batch, g) || max_label < 1) return EINVAL_;
  size_t M = (size_t)g.batch * max_label;
  const double nan = std::numeric_limits<double>::quiet_NaN();
  for (size_t i = 0; i < M; ++i) {
    if (sphericity) sphericity[i] = nan;
    if (roundness) roundness[i] = nan;
    if (volume) volume[i] = 0;
    if (n_shell) n_shell[i] = 0;
    if (max_lt2) max_lt2[i] = 0;
    if (mean_lt) mean_lt[i] = nan;
    if (shell_mean_lt) shell_mean_lt[i] = nan;
    if (axis_a) axis_a[i] = nan;
    if (axis_cb) axis_cb[i] = nan;
  }
  Ctx C{labels, g, flags, nullptr, nullptr, nullptr};
  std::vector<Object> objs;
  std::vector<ObjectResult> res;
  int st = run(C, max_label, label_mask, nthreads, objs, res);
  if (st != OK) return st;
  for (size_t i = 0; i < objs.size(); ++i) {
    const ObjectResult& r = res[i];
    size_t id = (size_t)objs[i].b * max_label + (objs[i].label - 1);
    double V = (double)r.volume;
    double a = r.sum_lt / V;
    double Rmax = std::sqrt((double)r.max_lt2);
    double rbar = r.sum_shell_lt / (double)r.n_shell;
    double cb = g.ndim == 3 ? 3.0 * V / (4.0 * kPi * a * a) : V / (kPi * a);
    if (sphericity) sphericity[id] = g.ndim == 3 ? sphericity_3d(V, a) : sphericity_2d(V, a);
    if (roundness) roundness[id] = rbar / Rmax;
    if (volume) volume[id] = r.volume;
    if (n_shell) n_shell[id] = r.n_shell;
    if (max_lt2) max_lt2[id] = r.max_lt2;
    if (mean_lt) mean_lt[id] = a;
    if (shell_mean_lt) shell_mean_lt[id] = rbar;
    if (axis_a) axis_a[id] = a;
    if (axis_cb) axis_cb[id] = cb;
  }
  return OK;
}

double fastrs_oracle_spheroid_area(double a, double c) { return spheroid_area(a, c); }
double fastrs_oracle_ramanujan_perimeter(double a, double b) { return ramanujan_perimeter(a, b); }
double fastrs_oracle_sphericity_3d(double V, double mean_lt) { return sphericity_3d(V, mean_lt); }
double fastrs_oracle_sphericity_2d(double A, double mean_lt) { return sphericity_2d(A, mean_lt); }

}  // extern "C"
