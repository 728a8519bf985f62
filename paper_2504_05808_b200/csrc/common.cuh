// Internal declarations shared by the libfastrs.so translation units (NOT the oracle).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fastrs {

// ---- packed EDT word (S2): [b31 y-run start][b30 z-run start][b29..0 partial D] -----
constexpr uint32_t kInf = 0x3FFFFFFFu;   // "no site yet"; also the D mask
constexpr uint32_t kMask = 0x3FFFFFFFu;
constexpr uint32_t kBitY = 0x80000000u;  // element is the first of its y-run
constexpr uint32_t kBitZ = 0x40000000u;  // element is the first of its z-run

// ---- status bits in the workspace header ---------------------------------------------
constexpr uint32_t kStBadLabel = 1u, kStNoSite = 2u, kStInternal = 4u, kStShell = 8u;

constexpr uint32_t kFlagBorder = 1u, kFlagAsync = 4u, kFlagHostIO = 8u, kFlagForceFallback = 16u;
constexpr uint32_t kFlagNoListStaging = 1024u;  // test hook: K5a list overflow regathers instead of staging
constexpr uint32_t kFlagNoCoverCut = 2048u;     // test hook: K5a without the cover cut
constexpr uint32_t kFlagExactPrune = 4096u;     // K4: every stage-2 class (the exact |s|^2 <= 12 kept set)
// launch_dilate_gather mode bits
constexpr int kGatherForceFallback = 1, kGatherNoStaging = 2, kGatherNoCoverCut = 4;
__host__ inline int gather_mode_of(uint32_t flags) {
  return ((flags & kFlagForceFallback) ? kGatherForceFallback : 0) | ((flags & kFlagNoListStaging) ? kGatherNoStaging : 0) |
         ((flags & kFlagNoCoverCut) ? kGatherNoCoverCut : 0);
}
constexpr uint32_t kFlagEdgeSkipZlo = 32u, kFlagEdgeSkipZhi = 64u, kFlagSlabTranspose = 128u, kFlagApproxLt = 256u;

// ---- dilation / pruning tiles ---------------------------------------------------------
// 3D tile 32 x 8 x 8 (x fastest), 2D tile 32 x 64; both 64 rows of 32 = 2048 elements.
constexpr int kTX = 32;
constexpr int kTileVol = 2048;
// per tile: counts of the kept centres with D bucket >= 4k, k = 0..31 (K4 writes, K5a cuts each
// home tile's bucket-sorted list with them)
constexpr int kOctPerTile = 32;
constexpr int kRows = 64;
constexpr int kTZ3 = 8;                 // 3D tile extent along z (slab alignment unit)
constexpr int kLevels = 6;              // sparse-table levels for 32-wide rows: 1..32
constexpr int kRowStride = kLevels * 32 + 1;  // +1: rows start in different banks

// ---- lattice containment table (S4) ---------------------------------------------------
constexpr int kDcap3 = 8192;   // 3D: centres with D > kDcap3 are always kept
constexpr int kDcap2 = 32768;  // 2D
constexpr int kClasses3 = 12;  // offset classes with |s|^2 <= 12 (178 offsets; first 3 = 26-nbhd)
constexpr int kClasses2 = 5;   // offset classes with |s|^2 <= 8 (24 offsets; first 2 = 8-nbhd)

// Division of 32-bit unsigned values by a runtime-invariant divisor d >= 1 (Granlund-Montgomery:
// one multiply-high, an add and two shifts instead of a ~20-instruction integer division);
// kernels split flat tile / group indices into coordinates with it.
struct FastDiv {
  uint32_t d = 1, m = 0, s = 0;
  FastDiv() = default;
  __host__ explicit FastDiv(uint32_t div) : d(div) {
    if (d <= 1) {
      d = 1;
      return;
    }
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    m = (uint32_t)(((((unsigned long long)1 << l) - d) << 32) / d + 1);
    s = l - 1;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    if (d == 1) return n;
    const uint32_t t = __umulhi(n, m);
    return (t + ((n - t) >> 1)) >> s;
  }
  // n = q * d + r
  __device__ __forceinline__ uint32_t divmod(uint32_t n, uint32_t& r) const {
    const uint32_t q = div(n);
    r = n - q * d;
    return q;
  }
};

struct Geom {
  int ndim;
  int64_t B, Z, Y, X;  // 2D: Z = 1
  int64_t N;           // B*Z*Y*X
  int TY, TZ;          // tile extents (3D: 8,8; 2D: 64,1)
  int64_t ntx, nty, ntz, ntiles;  // tile grid per item: ntz*nty*ntx, ntiles includes B
  int64_t tz_lo, tz_hi;           // tile layers whose LT / reductions are produced (slab path)
  int64_t nscale;                 // elements per item for the fixed-point scale (global volume)
};

struct WsHeader {
  uint32_t status;
  uint32_t dmax;
  unsigned long long n_fg;
  unsigned long long n_kept;
  unsigned long long n_intervals;
  int32_t scale_log2;   // fixed-point scale of the LT sums (always 32)
  uint32_t n_fallback;  // tile groups handed to the atomic fallback dilation
  uint32_t dxymax;      // max partial D after the y pass (slab path: the z halo width)
  uint32_t n_fb;        // tiles listed for the atomic fallback dilation
  uint32_t n_rounds_extra;  // K5 groups x rounds beyond the first
  uint32_t n_regathers;     // K5 list overflows that needed a second gather pass
  uint32_t max_group_list;  // K5 longest per-group candidate list
  uint32_t n_staged;        // K5 list overflows staged in the pool's top half (no second pass)
  unsigned long long sum_group_list;  // K5 candidates summed over groups
  unsigned long long pool_used;       // K5 candidate pool entries allocated
  unsigned long long stage_used;      // K5a: list-overflow staging entries (reset per gather launch)
  uint32_t paint_next;   // K5b work counter (reset before each launch)
  uint32_t sat_n;        // K2/K3: CTAs listed for the exact 32-bit column pass (reset per launch)
  uint32_t pad3;
  unsigned long long n_painted;   // K5b: balls painted (lanes over rows) after the screens
  unsigned long long n_covering;  // K5b: painted balls that covered at least one cell
  unsigned long long g_stats[3];  // K5a statistics (FASTRS_GATHER_STATS builds only): examined, D-cut, taken
  uint32_t n_defer[4];            // K5 waves: groups wave w deferred to wave w + 1 (the pool was full)
  uint32_t slow_n;                // K2/K3: elements listed for the batched 32-bit scan (reset per launch)
  uint32_t pad4;
};
static_assert(sizeof(WsHeader) <= 256, "header");

// per-tile metadata written by the pruning kernel
struct TileMeta {
  uint32_t count;  // kept centres
  uint32_t maxD;   // max D over kept centres
  uint32_t nfg;    // foreground elements of the tile
  uint32_t pad;
};

// per-label accumulators (SoA).  The LT sums are exact fixed-point integers with the fixed
// scale 2^32: every term is fx(c) = round(sqrt(c) * 2^32) (c = LT^2), and each sum is kept as
// two u64 words, hi = sum of (term >> 32) pieces and lo = sum of (term & (2^32-1)) pieces, so
// the value is hi * 2^32 + lo with no overflow for objects below 2^32 elements.  Integer adds
// are order-independent: the result is bit-identical for any launch order, chunking or
// z-slab split, and no scale depends on Dmax.
struct Accum {
  unsigned long long* vol;
  unsigned long long* nshell;
  unsigned long long* sum;       // hi words (M), lo words at sum + M
  unsigned long long* sumshell;  // hi words (M), lo words at sumshell + M
  uint32_t* maxlt2;
  int64_t M;                     // batch*max_label
  int32_t max_label;
};
constexpr double kFxScale = 4294967296.0;  // 2^32
constexpr uint32_t kFxLut = 65536;         // entries of the per-device fixed-point sqrt table

struct Outputs {
  double* sphericity;
  double* roundness;
  int64_t* volume;
  int64_t* n_shell;
  uint32_t* max_lt2;
  double* mean_lt;
  double* max_lt;
  double* shell_mean_lt;
  double* axis_a;
  double* axis_cb;
};

__host__ __device__ inline int ceil_log2_u64(unsigned long long v) {
  int r = 0;
  while ((1ull << r) < v && r < 63) ++r;
  return r;
}

// Monotone bucket of a squared radius D: 8 buckets per octave, 0..126 for D < 65536; every
// D >= 65536 shares the saturated bucket 127 (K4's 128-entry histograms stay in range).
// Kept-centre lists are sorted by it (descending) and K5 walks it downwards.
constexpr int kBucketTop = 127;
__host__ __device__ inline int dbucket(uint32_t D) {
  int msb = 31;
  while (msb > 0 && !((D >> msb) & 1u)) --msb;
#ifdef __CUDA_ARCH__
  msb = 31 - __clz(D);
#endif
  const int frac = msb >= 3 ? (int)((D >> (msb - 3)) & 7u) : (int)((D << (3 - msb)) & 7u);
  const int b = msb * 8 + frac;
  return b < kBucketTop ? b : kBucketTop;
}
// Largest D with dbucket(D) <= b (D >= 1): one less than the smallest D of bucket b+1 or above.
__host__ __device__ inline uint32_t dbucket_max(int b) {
  if (b >= kBucketTop) return 0xFFFFFFFFu;  // the saturated bucket is unbounded
  const int b1 = b + 1;
  if (b1 >= 24) return ((uint32_t)(8 + (b1 & 7)) << ((b1 >> 3) - 3)) - 1u;
  // smallest D with dbucket(D) >= b1 for b1 < 24 (dbucket: 1->0, 2->8, 3->12, 4->16, 5->18, 6->20, 7->22, 8->24)
  const uint32_t dmin = b1 <= 0 ? 1u : b1 <= 8 ? 2u : b1 <= 12 ? 3u : b1 <= 16 ? 4u : b1 <= 18 ? 5u : b1 <= 20 ? 6u : b1 <= 22 ? 7u : 8u;
  return dmin - 1u;
}

// ---- kernel launchers (stream-ordered) -----------------------------------------------
void launch_edt_x(const int32_t* labels, const int32_t* labels_below, uint32_t* out, const Geom& g,
                  int32_t max_label, bool border, WsHeader* hdr, cudaStream_t st);
// Column pass along axis 1 (y) or 2 (z) of g.  Positions [p_lo, p_hi) of the axis are written,
// to out + (p - p_lo) * stride; gofs / Lg: global position of local 0 and the global axis length
// (the border convention applies at global 0 and Lg).  Default: p_lo = 0, p_hi = L, gofs = 0.
// satlist: workspace list of col_blocks(g) u32 for the CTAs the 16-bit kernel hands to the exact
// 32-bit kernel (NULL: the 32-bit kernel everywhere).
// scratch (nullable): device memory idle during the pass (the K5 candidate pool) for the exact
// lower-envelope fix-up of the CTAs the 16-bit kernel lists (else the windowed 32-bit kernel)
void launch_edt_col(const uint32_t* in, uint32_t* out, const Geom& g, int axis, bool final_pass,
                    bool border, WsHeader* hdr, uint32_t* satlist, cudaStream_t st, int64_t p_lo = 0,
                    int64_t p_hi = -1, int64_t gofs = 0, int64_t Lg = -1, void* scratch = nullptr,
                    size_t scratch_bytes = 0);
int64_t col_blocks(const Geom& g);  // column-pass CTAs of the larger of the y / z passes
cudaError_t ensure_mtables(int device);  // builds the per-device lattice tables (sync, once)
const unsigned long long* device_fxlut(int device);  // fx(c) for c < kFxLut (after ensure_mtables)
// K4; also writes per tile the foreground and shell (D == 1) row masks (fgm, shm: kRows u32 each)
// and the number of kept entries with D bucket >= 8o for o = 0..15 (oct: 16 u16) used by K5's gather
void launch_prune(const uint32_t* D, const Geom& g, TileMeta* meta, uint2* centres, uint32_t* fgm, uint32_t* shm,
                  uint16_t* oct, WsHeader* hdr, cudaStream_t st, int64_t tz_lo = 0, int64_t tz_hi = 0,
                  bool exact_prune = false);
int64_t dilate_groups(const Geom& g);        // K5 tile groups (gcount / goff entries)
// K5b.  acc == NULL: LT^2 of every painted tile -> the LT plane ltp (u16).  acc != NULL (fused):
// no LT plane; every ball that covers cells adds (count, shell count, D) of those cells to the
// per-label accumulators of the label of the cells it covers (labels read once per covering ball)
// approx (FASTRS_APPROX_LT, needs D): each tile stops once <= 4 % of its foreground is uncovered;
// those cells take LT^2 = D
void launch_dilate_paint(const uint32_t* fgm, const uint32_t* shm, const TileMeta* meta,
                         const unsigned long long* pool, const uint32_t* gcount, const uint32_t* goff, const Geom& g,
                         uint32_t* ltp, const int32_t* labels, const Accum* acc, const uint32_t* D, bool approx,
                         WsHeader* hdr, cudaStream_t st, int wave = 0);
void launch_dilate_fallback(TileMeta* meta, const uint2* centres, const uint32_t* fbl, const Geom& g, uint32_t* ltp,
                            WsHeader* hdr, cudaStream_t st);
// K5a: per tile group, gather the kept balls that reach it and write them sorted by D
// (descending) to the candidate pool; groups that cannot be handled are listed in fbl.
// Waves: the pool is reused by kDilateWaves gather + paint rounds; wave w > 0 takes only the
// groups the previous wave deferred because the pool was full (the last wave lists such groups
// for the atomic fallback).  Call gather(w) then paint(w) for w = 0 .. kDilateWaves - 1.
constexpr int kDilateWaves = 3;
void launch_dilate_gather(const uint32_t* fgm, TileMeta* meta, const uint2* centres, const uint16_t* oct, uint32_t* fbl,
                          unsigned long long* pool, uint32_t* gcount, uint32_t* goff, const Geom& g, int gather_mode,
                          WsHeader* hdr, cudaStream_t st, int wave, uint32_t* deflists);
// workspace of the deferred-group lists of the waves: 2 * dilate_groups(g) u32
int64_t dilate_pool_entries(const Geom& g);  // K5 candidate pool (sorted per-group lists), u64 entries
// K5 epilogue: shell, per-label reductions (acc nullable) and LT outputs from the LT plane ltp
void launch_epilogue(const int32_t* labels, const uint32_t* D, const Geom& g, const Accum* acc, uint32_t* lt2_out,
                     float* lt_out, const uint32_t* ltp, WsHeader* hdr, cudaStream_t st);
// per-label reductions of the tiles the atomic fallback kernel painted (every tile when
// Dmax > 65535, else the n_fb tiles listed in fbl); the fused paint covers all the others
void launch_epilogue_fallback(const int32_t* labels, const uint32_t* D, const TileMeta* meta, const uint32_t* fbl,
                              const Geom& g, const Accum& acc, const uint32_t* ltp, WsHeader* hdr, cudaStream_t st);
cudaError_t launch_touch_edge(const int32_t* labels, const Geom& g, int32_t max_label, uint8_t* touch,
                              bool skip_zlo, bool skip_zhi, cudaStream_t st);
cudaError_t launch_filter(double* sph, double* rnd, const int64_t* vol, const uint8_t* touch, int64_t n,
                          int64_t min_volume, cudaStream_t st);
void launch_metrics(const Accum& acc, const Geom& g, const Outputs& o, WsHeader* hdr,
                    cudaStream_t st);
void release_mtables();
int set_error(int code, const char* msg);  // sets the fastrs_last_error message, returns code

}  // namespace fastrs
