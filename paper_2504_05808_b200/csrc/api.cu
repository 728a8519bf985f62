// C ABI of libfastrs.so (include/fastrs.h): argument checks, workspace carving, the
// stream-ordered launch sequence K1..K6 and the single status read at the end.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include "fastrs.h"

namespace fastrs {
namespace {

// NVTX range per stage of a call (host-side launch ranges; visible to Nsight tools, no cost
// without an attached tool)
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

thread_local std::string t_err = "";

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(FASTRS_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

constexpr int64_t kMaxDim = 16384;

int make_geom(const int64_t* dims, int ndim, int64_t batch, Geom& g) {
  if (!dims) return fail(FASTRS_EINVAL, "dims is NULL");
  if (ndim != 2 && ndim != 3) return fail(FASTRS_EINVAL, "ndim must be 2 or 3 (got %d)", ndim);
  if (batch < 1) return fail(FASTRS_EINVAL, "batch must be >= 1");
  for (int i = 0; i < ndim; ++i)
    if (dims[i] < 1 || dims[i] > kMaxDim) return fail(FASTRS_EINVAL, "dims[%d] = %lld outside [1, 16384]", i, (long long)dims[i]);
  g.ndim = ndim;
  g.B = batch;
  g.Z = ndim == 3 ? dims[0] : 1;
  g.Y = dims[ndim - 2];
  g.X = dims[ndim - 1];
  g.N = g.B * g.Z * g.Y * g.X;
  g.TY = ndim == 3 ? 8 : 64;
  g.TZ = ndim == 3 ? 8 : 1;
  g.ntx = (g.X + kTX - 1) / kTX;
  g.nty = (g.Y + g.TY - 1) / g.TY;
  g.ntz = (g.Z + g.TZ - 1) / g.TZ;
  g.ntiles = g.B * g.ntz * g.nty * g.ntx;
  g.tz_lo = 0;
  g.tz_hi = g.ntz;
  g.nscale = g.Z * g.Y * g.X;
  if (g.ntiles >= (1ll << 32)) return fail(FASTRS_EINVAL, "grid too large");
  return FASTRS_OK;
}

inline size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

struct Layout {
  size_t hdr, A, B, meta, fgm, shm, oct, fbl, gcount, goff, defl, pool, sat, cent, vol, nsh, sum, sumsh, mx, h_labels, h_sph, h_rnd,
      total;
};

Layout make_layout(const Geom& g, int32_t max_label, uint32_t flags) {
  Layout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align256(bytes);
    return o;
  };
  const size_t M = (size_t)g.B * (size_t)(max_label > 0 ? max_label : 0);
  L.hdr = take(256);
  L.A = take((size_t)g.N * 4);
  L.B = take((size_t)g.N * 4);
  L.meta = take((size_t)g.ntiles * sizeof(TileMeta));
  L.fgm = take((size_t)g.ntiles * kRows * 4);
  L.shm = take((size_t)g.ntiles * kRows * 4);
  L.oct = take((size_t)g.ntiles * kOctPerTile * 2);
  L.fbl = take((size_t)g.ntiles * 4);
  L.gcount = take((size_t)dilate_groups(g) * 4);
  L.goff = take((size_t)dilate_groups(g) * 4);
  L.defl = take((size_t)dilate_groups(g) * 8);  // K5 waves: two deferred-group lists
  L.pool = take((size_t)dilate_pool_entries(g) * 8);
  L.sat = take((size_t)col_blocks(g) * 4);
  L.cent = take((size_t)g.ntiles * kTileVol * sizeof(uint2));
  L.vol = take(M * 8);
  L.nsh = take(M * 8);
  L.sum = take(2 * M * 8);    // hi | lo words (common.cuh "Accum")
  L.sumsh = take(2 * M * 8);
  L.mx = take(M * 4);
  if (flags & kFlagHostIO) {
    L.h_labels = take((size_t)g.N * 4);
    L.h_sph = take(M * 8);
    L.h_rnd = take(M * 8);
  }
  L.total = off;
  return L;
}

// ---- profiling -------------------------------------------------------------------------
constexpr int kStages = 8;
std::mutex g_prof_mu;
bool g_prof = false;
double g_prof_ms[kStages];
int64_t g_prof_calls = 0;
cudaEvent_t g_ev[64][kStages + 1];
bool g_ev_init[64];

struct StageTimer {
  bool on = false;
  int dev = 0;
  cudaStream_t st = nullptr;
  int order[kStages];  // stages in the order their end events were recorded
  int nmarks = 0;
  void begin(cudaStream_t s) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    on = g_prof;
    st = s;
    if (!on) return;
    cudaGetDevice(&dev);
    if (!g_ev_init[dev]) {
      for (auto& e : g_ev[dev]) cudaEventCreate(&e);
      g_ev_init[dev] = true;
    }
    cudaEventRecord(g_ev[dev][0], st);
  }
  // mark the end of stage k (each stage's time runs from the previous mark)
  void mark(int k) {
    if (!on || nmarks >= kStages) return;
    cudaEventRecord(g_ev[dev][k + 1], st);
    order[nmarks++] = k;
  }
  void finish() {
    if (!on || nmarks == 0) return;
    cudaEventSynchronize(g_ev[dev][order[nmarks - 1] + 1]);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    int prev = 0;
    for (int i = 0; i < nmarks; ++i) {
      const int k = order[i];
      float ms = 0;
      cudaEventElapsedTime(&ms, g_ev[dev][prev], g_ev[dev][k + 1]);
      g_prof_ms[k] += ms;
      prev = k + 1;
    }
    g_prof_calls += 1;
  }
};

enum Stage { kEdtOnly, kLtOnly, kFull };

int run(const int32_t* labels, const Geom& g, int32_t max_label, uint32_t flags, Stage stage, uint32_t* d2_out,
        uint32_t* lt2_out, float* lt_out, const Outputs* outs, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (!labels) return fail(FASTRS_EINVAL, "labels is NULL");
  if (!ws) return fail(FASTRS_EINVAL, "workspace is NULL");
  if (((uintptr_t)ws & 255) != 0) return fail(FASTRS_EINVAL, "workspace must be 256-byte aligned");
  const Layout L = make_layout(g, stage == kFull ? max_label : 0, 0);
  if (ws_bytes < L.total)
    return fail(FASTRS_ENOMEM, "workspace too small: %zu < %zu bytes", ws_bytes, L.total);
  char* w = (char*)ws;
  WsHeader* hdr = (WsHeader*)(w + L.hdr);
  uint32_t* A = (uint32_t*)(w + L.A);
  uint32_t* B = (uint32_t*)(w + L.B);
  TileMeta* meta = (TileMeta*)(w + L.meta);
  uint2* cent = (uint2*)(w + L.cent);
  uint32_t* sat = (uint32_t*)(w + L.sat);
  // the candidate pool is idle during the EDT passes: scratch of the column passes' envelope fix-up
  void* scr = w + L.pool;
  const size_t scr_bytes = (size_t)dilate_pool_entries(g) * 8;
  const bool border = (flags & kFlagBorder) != 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (stage != kEdtOnly) {
    e = ensure_mtables(dev);
    if (e != cudaSuccess) return cuda_fail(e, "building the lattice containment table");
  }
  StageTimer tm;
  tm.begin(st);
  e = cudaMemsetAsync(hdr, 0, 256, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  Accum acc{};
  if (stage == kFull) {
    acc.vol = (unsigned long long*)(w + L.vol);
    acc.nshell = (unsigned long long*)(w + L.nsh);
    acc.sum = (unsigned long long*)(w + L.sum);
    acc.sumshell = (unsigned long long*)(w + L.sumsh);
    acc.maxlt2 = (uint32_t*)(w + L.mx);
    acc.M = g.B * (int64_t)max_label;
    acc.max_label = max_label;
    cudaMemsetAsync(w + L.vol, 0, (L.mx - L.vol) + align256((size_t)acc.M * 4), st);
  }
  if (lt2_out) cudaMemsetAsync(lt2_out, 0, (size_t)g.N * 4, st);
  if (lt_out) cudaMemsetAsync(lt_out, 0, (size_t)g.N * 4, st);

  // K1..K3: EDT
  Nvtx call_range(stage == kFull ? "fastrs_sphericity_roundness" : stage == kLtOnly ? "fastrs_local_thickness"
                                                                                   : "fastrs_edt_sq");
  {
    Nvtx r("K1 edt_x");
    launch_edt_x(labels, nullptr, A, g, stage == kFull ? max_label : INT32_MAX, border, hdr, st);
  }
  tm.mark(0);
  uint32_t* D;
  if (g.ndim == 2) {
    D = stage == kEdtOnly ? d2_out : B;
    Nvtx r("K2 edt_y (final)");
    launch_edt_col(A, D, g, 1, true, border, hdr, sat, st, 0, -1, 0, -1, scr, scr_bytes);
    tm.mark(1);
  } else {
    {
      Nvtx r("K2 edt_y");
      launch_edt_col(A, B, g, 1, false, border, hdr, sat, st, 0, -1, 0, -1, scr, scr_bytes);
    }
    tm.mark(1);
    D = stage == kEdtOnly ? d2_out : A;
    Nvtx r("K3 edt_z");
    launch_edt_col(B, D, g, 2, true, border, hdr, sat, st, 0, -1, 0, -1, scr, scr_bytes);
    tm.mark(2);
  }
  if (stage != kEdtOnly) {
    uint32_t* fgm = (uint32_t*)(w + L.fgm);
    uint32_t* shm = (uint32_t*)(w + L.shm);
    uint16_t* oct = (uint16_t*)(w + L.oct);
    {
      Nvtx r("K4 prune");
      launch_prune(D, g, meta, cent, fgm, shm, oct, hdr, st, 0, 0, (flags & kFlagExactPrune) != 0);
    }
    tm.mark(3);
    uint32_t* ltp = D == A ? B : A;  // the plane the EDT no longer needs holds LT^2 (fallback / LT outputs)
    uint32_t* fbl = (uint32_t*)(w + L.fbl);
    unsigned long long* pool = (unsigned long long*)(w + L.pool);
    uint32_t* gcount = (uint32_t*)(w + L.gcount);
    uint32_t* goff = (uint32_t*)(w + L.goff);
    // K5a + K5b in waves over the candidate pool (wave w > 0: the groups the pool could not
    // hold in wave w - 1; its kernels leave at once when there are none); K5b with the
    // reductions fused (S&R) or writing the LT plane (LT outputs); K5' for the tiles K5a handed
    // over (every tile when Dmax > 65535)
    for (int wv = 0; wv < kDilateWaves; ++wv) {
      {
        Nvtx r("K5a gather");
        launch_dilate_gather(fgm, meta, cent, oct, fbl, pool, gcount, goff, g, gather_mode_of(flags), hdr, st, wv,
                             (uint32_t*)(w + L.defl));
      }
      if (wv == 0) tm.mark(7);
      Nvtx r("K5b paint");
      launch_dilate_paint(fgm, shm, meta, pool, gcount, goff, g, ltp, labels, stage == kFull ? &acc : nullptr, D,
                          (flags & kFlagApproxLt) != 0, hdr, st, wv);
    }
    {
      Nvtx r("K5' fallback");
      launch_dilate_fallback(meta, cent, fbl, g, ltp, hdr, st);
    }
    tm.mark(4);
    if (stage == kFull) {
      {
        Nvtx r("K5e fallback-tile reductions");
        launch_epilogue_fallback(labels, D, meta, fbl, g, acc, ltp, hdr, st);
      }
      tm.mark(6);
      Nvtx r("K6 metrics");
      launch_metrics(acc, g, *outs, hdr, st);
      tm.mark(5);
    } else {
      Nvtx r("K5e LT outputs");
      launch_epilogue(labels, D, g, nullptr, lt2_out, lt_out, ltp, hdr, st);
      tm.mark(6);
    }
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  if (flags & kFlagAsync) return FASTRS_OK;
  uint32_t status = 0;
  e = cudaMemcpyAsync(&status, &hdr->status, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "status read");
  tm.finish();
  if (status & kStBadLabel) return fail(FASTRS_EINVAL, "a label is < 0 or > max_label");
  if (status & kStNoSite)
    return fail(FASTRS_ENOSITE, "an object element has no site (no other label and the border is not background)");
  if (status & kStInternal) return fail(FASTRS_EINTERNAL, "device invariant violated: LT^2 < D");
  if (status & kStShell) return fail(FASTRS_EINTERNAL, "device invariant violated: shell mean LT > max LT or empty shell");
  return FASTRS_OK;
}

__global__ void k_set_dmax(WsHeader* hdr, uint32_t v) { hdr->dmax = v; }

// copy one u32 of the header to a caller-owned device word
int header_word_out(const WsHeader* hdr, const uint32_t* field, uint32_t* dst, cudaStream_t st) {
  if (!dst) return FASTRS_OK;
  (void)hdr;
  cudaError_t e = cudaMemcpyAsync(dst, field, 4, cudaMemcpyDeviceToDevice, st);
  return e == cudaSuccess ? FASTRS_OK : cuda_fail(e, "header copy");
}

// end of a call: optional sync + status mapping (shared by the slab phases)
int finish_call(WsHeader* hdr, uint32_t flags, cudaStream_t st) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  if (flags & kFlagAsync) return FASTRS_OK;
  uint32_t status = 0;
  e = cudaMemcpyAsync(&status, &hdr->status, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "status read");
  if (status & kStBadLabel) return fail(FASTRS_EINVAL, "a label is < 0 or > max_label");
  if (status & kStNoSite)
    return fail(FASTRS_ENOSITE, "an object element has no site (no other label and the border is not background)");
  if (status & kStInternal) return fail(FASTRS_EINTERNAL, "device invariant violated: LT^2 < D");
  if (status & kStShell) return fail(FASTRS_EINTERNAL, "device invariant violated: shell mean LT > max LT or empty shell");
  return FASTRS_OK;
}

struct SlabLayout {
  size_t hdr, P, meta, fgm, shm, oct, fbl, gcount, goff, defl, pool, sat, poff, cent, total;
};
SlabLayout make_slab_layout(const Geom& g) {
  SlabLayout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align256(bytes);
    return o;
  };
  L.hdr = take(256);
  L.P = take((size_t)g.N * 4);
  L.meta = take((size_t)g.ntiles * sizeof(TileMeta));
  L.fgm = take((size_t)g.ntiles * kRows * 4);
  L.shm = take((size_t)g.ntiles * kRows * 4);
  L.oct = take((size_t)g.ntiles * kOctPerTile * 2);
  L.fbl = take((size_t)g.ntiles * 4);
  L.gcount = take((size_t)dilate_groups(g) * 4);
  L.goff = take((size_t)dilate_groups(g) * 4);
  L.defl = take((size_t)dilate_groups(g) * 8);  // K5 waves: two deferred-group lists
  L.pool = take((size_t)dilate_pool_entries(g) * 8);
  L.sat = take((size_t)col_blocks(g) * 4);
  L.poff = take((size_t)g.ntiles * 4 + 16);
  L.cent = take((size_t)g.ntiles * kTileVol * sizeof(uint2));
  L.total = off;
  return L;
}

// ---- kept-centre halo (N4): pack / unpack the K4 outputs of whole tile layers ----------------
// record per tile: TileMeta (4 u32) + the 16 octave counts (8 u32) = 12 u32; entries: the tile's
// kept centres (uint2), tiles in index order
constexpr int kRecWords = FASTRS_TILE_RECORD_WORDS;
static_assert(kRecWords == 4 + kOctPerTile / 2, "tile record: 4 meta words + the bucket counts");

// exclusive prefix of the tiles' centre counts (one CTA; counts from meta or from records)
__global__ void k_tile_prefix(const TileMeta* __restrict__ meta, const uint32_t* __restrict__ rec, int64_t t0,
                              int64_t n, uint32_t* __restrict__ off, unsigned long long* __restrict__ total) {
  const int64_t per = (n + blockDim.x - 1) / blockDim.x, lo = threadIdx.x * per, hi = lo + per < n ? lo + per : n;
  unsigned long long loc = 0;
  for (int64_t i = lo; i < hi; ++i) loc += rec ? rec[i * kRecWords] : meta[t0 + i].count;
  __shared__ unsigned long long part[1024];
  part[threadIdx.x] = loc;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {
    const unsigned long long v = (int)threadIdx.x >= o ? part[threadIdx.x - o] : 0ull;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  unsigned long long run = part[threadIdx.x] - loc;
  for (int64_t i = lo; i < hi; ++i) {
    off[i] = (uint32_t)run;
    run += rec ? rec[i * kRecWords] : meta[t0 + i].count;
  }
  if (threadIdx.x == blockDim.x - 1 && total) *total = part[threadIdx.x];
}

__global__ void k_tile_pack(const TileMeta* __restrict__ meta, const uint16_t* __restrict__ oct,
                            const uint2* __restrict__ cent, int64_t t0, const uint32_t* __restrict__ off,
                            uint32_t* __restrict__ rec, uint2* __restrict__ ent) {
  const int64_t i = blockIdx.x, t = t0 + i;
  const TileMeta m = meta[t];
  if (threadIdx.x < 4) rec[i * kRecWords + threadIdx.x] = threadIdx.x == 0 ? m.count : threadIdx.x == 1 ? m.maxD
                                                                              : threadIdx.x == 2 ? m.nfg : 0u;
  if (threadIdx.x < kOctPerTile / 2)
    rec[i * kRecWords + 4 + threadIdx.x] = (uint32_t)oct[t * kOctPerTile + 2 * threadIdx.x] |
                                           ((uint32_t)oct[t * kOctPerTile + 2 * threadIdx.x + 1] << 16);
  for (uint32_t k = threadIdx.x; k < m.count; k += blockDim.x) ent[off[i] + k] = cent[t * kTileVol + k];
}

__global__ void k_tile_unpack(TileMeta* __restrict__ meta, uint16_t* __restrict__ oct, uint2* __restrict__ cent,
                              int64_t t0, const uint32_t* __restrict__ off, const uint32_t* __restrict__ rec,
                              const uint2* __restrict__ ent) {
  const int64_t i = blockIdx.x, t = t0 + i;
  const uint32_t cnt = rec[i * kRecWords];
  if (threadIdx.x == 0) meta[t] = TileMeta{cnt, rec[i * kRecWords + 1], rec[i * kRecWords + 2], 0u};
  if (threadIdx.x < kOctPerTile / 2) {
    const uint32_t w = rec[i * kRecWords + 4 + threadIdx.x];
    oct[t * kOctPerTile + 2 * threadIdx.x] = (uint16_t)(w & 0xFFFFu);
    oct[t * kOctPerTile + 2 * threadIdx.x + 1] = (uint16_t)(w >> 16);
  }
  for (uint32_t k = threadIdx.x; k < cnt; k += blockDim.x) cent[t * kTileVol + k] = ent[off[i] + k];
}

int slab_prologue(const int64_t* dims, Geom& g, SlabLayout& L, void* ws, size_t ws_bytes, WsHeader*& hdr,
                  cudaStream_t st) {
  int rc = make_geom(dims, 3, 1, g);
  if (rc) return rc;
  if (!ws) return fail(FASTRS_EINVAL, "workspace is NULL");
  if (((uintptr_t)ws & 255) != 0) return fail(FASTRS_EINVAL, "workspace must be 256-byte aligned");
  L = make_slab_layout(g);
  if (ws_bytes < L.total) return fail(FASTRS_ENOMEM, "workspace too small: %zu < %zu bytes", ws_bytes, L.total);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = ensure_mtables(dev);
  if (e != cudaSuccess) return cuda_fail(e, "per-device setup");
  hdr = (WsHeader*)((char*)ws + L.hdr);
  e = cudaMemsetAsync(hdr, 0, 256, st);
  return e == cudaSuccess ? FASTRS_OK : cuda_fail(e, "cudaMemsetAsync");
}

// ---- host entry point: the host->device copy overlapped with the computation -------------
// The label volume is copied in z-chunks of kChunkZ slices on a copy stream; the compute stream
// runs each stage on a chunk as soon as the chunks it depends on are in: K1+K2 on chunk c
// (per-slice work), K3 on chunk c-1 (reads up to h = ceil(sqrt(max D_xy)) slices away), K4 on
// chunk c-2 (3-voxel halo), K5a+K5b on chunk c-3 (balls of radius R = isqrt(Dmax-1)); K5's
// fallback tiles, the epilogue (it needs the final Dmax for the fixed-point scale) and K6 run
// after the last chunk.  Exact whenever h <= kChunkZ and R <= kChunkZ, which is checked at the
// end; otherwise the call recomputes everything with the plain path from the resident labels.
constexpr int64_t kChunkZ = 64;  // a multiple of the 16-slice K5 tile group

std::mutex g_cs_mu;
cudaStream_t g_copy_stream[64];

cudaStream_t copy_stream(int dev) {
  std::lock_guard<std::mutex> lk(g_cs_mu);
  if (!g_copy_stream[dev]) cudaStreamCreateWithFlags(&g_copy_stream[dev], cudaStreamNonBlocking);
  return g_copy_stream[dev];
}

// returns FASTRS_OK with *exact = false when the halo check failed (the caller reruns)
int run_host_pipelined(const int32_t* labels_host, int32_t* dlab, const Geom& g, int32_t max_label, uint32_t flags,
                       const Outputs& outs, void* ws, cudaStream_t st, bool* exact) {
  *exact = false;
  const Layout L = make_layout(g, max_label, 0);
  char* w = (char*)ws;
  WsHeader* hdr = (WsHeader*)(w + L.hdr);
  uint32_t* A = (uint32_t*)(w + L.A);
  uint32_t* B = (uint32_t*)(w + L.B);
  TileMeta* meta = (TileMeta*)(w + L.meta);
  uint2* cent = (uint2*)(w + L.cent);
  uint32_t* fgm = (uint32_t*)(w + L.fgm);
  uint32_t* shm = (uint32_t*)(w + L.shm);
  uint16_t* oct = (uint16_t*)(w + L.oct);
  uint32_t* fbl = (uint32_t*)(w + L.fbl);
  unsigned long long* pool = (unsigned long long*)(w + L.pool);
  uint32_t* gcount = (uint32_t*)(w + L.gcount);
  uint32_t* goff = (uint32_t*)(w + L.goff);
  uint32_t* sat = (uint32_t*)(w + L.sat);
  // the candidate pool is idle during the EDT passes: scratch of the column passes' envelope fix-up
  void* scr = w + L.pool;
  const size_t scr_bytes = (size_t)dilate_pool_entries(g) * 8;
  const bool border = (flags & kFlagBorder) != 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = ensure_mtables(dev);
  if (e != cudaSuccess) return cuda_fail(e, "per-device setup");
  Accum acc{};
  acc.vol = (unsigned long long*)(w + L.vol);
  acc.nshell = (unsigned long long*)(w + L.nsh);
  acc.sum = (unsigned long long*)(w + L.sum);
  acc.sumshell = (unsigned long long*)(w + L.sumsh);
  acc.maxlt2 = (uint32_t*)(w + L.mx);
  acc.M = (int64_t)max_label;
  acc.max_label = max_label;
  cudaMemsetAsync(hdr, 0, 256, st);
  cudaMemsetAsync(w + L.vol, 0, (L.mx - L.vol) + align256((size_t)acc.M * 4), st);
  cudaMemsetAsync(meta, 0, (size_t)g.ntiles * sizeof(TileMeta), st);  // unpruned tiles read as empty
  const int64_t YX = g.Y * g.X, Z = g.Z;
  const int nc = (int)((Z + kChunkZ - 1) / kChunkZ);
  cudaStream_t cs = copy_stream(dev);
  std::vector<cudaEvent_t> ev(nc + 1);
  for (auto& x : ev) cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
  cudaEventRecord(ev[nc], st);  // the copies wait for earlier work on the caller's stream
  cudaStreamWaitEvent(cs, ev[nc], 0);
  for (int c = 0; c < nc; ++c) {
    const int64_t z0 = c * kChunkZ, nz = (z0 + kChunkZ < Z ? kChunkZ : Z - z0);
    e = cudaMemcpyAsync(dlab + z0 * YX, labels_host + z0 * YX, (size_t)(nz * YX) * 4, cudaMemcpyHostToDevice, cs);
    if (e != cudaSuccess) return cuda_fail(e, "H2D labels chunk");
    cudaEventRecord(ev[c], cs);
  }
  auto zr = [&](int c, int64_t& z0, int64_t& z1) {
    z0 = c * kChunkZ;
    z1 = z0 + kChunkZ < Z ? z0 + kChunkZ : Z;
  };
  for (int step = 0; step < nc + 3; ++step) {
    int64_t z0, z1;
    if (step < nc) {  // K1 + K2 on chunk `step`
      zr(step, z0, z1);
      cudaStreamWaitEvent(st, ev[step], 0);
      const int64_t cd[3] = {z1 - z0, g.Y, g.X};
      Geom gc;
      make_geom(cd, 3, 1, gc);
      launch_edt_x(dlab + z0 * YX, z0 > 0 ? dlab + (z0 - 1) * YX : nullptr, A + z0 * YX, gc, max_label, border, hdr,
                   st);
      launch_edt_col(A + z0 * YX, B + z0 * YX, gc, 1, false, border, hdr, sat, st, 0, -1, 0, -1, scr, scr_bytes);
    }
    if (step >= 1 && step - 1 < nc) {  // K3 on chunk step-1: D into A
      zr(step - 1, z0, z1);
      launch_edt_col(B, A + z0 * YX, g, 2, true, border, hdr, sat, st, z0, z1, 0, -1, scr, scr_bytes);
    }
    if (step >= 2 && step - 2 < nc) {  // K4 on chunk step-2
      zr(step - 2, z0, z1);
      launch_prune(A, g, meta, cent, fgm, shm, oct, hdr, st, z0 / kTZ3, (z1 + kTZ3 - 1) / kTZ3,
                   (flags & kFlagExactPrune) != 0);
    }
    if (step >= 3 && step - 3 < nc) {  // K5a + K5b (reductions fused) on chunk step-3
      zr(step - 3, z0, z1);
      Geom gg = g;
      gg.tz_lo = z0 / kTZ3;
      gg.tz_hi = (z1 + kTZ3 - 1) / kTZ3;
      for (int wv = 0; wv < kDilateWaves; ++wv) {
        launch_dilate_gather(fgm, meta, cent, oct, fbl, pool, gcount, goff, gg, 0, hdr, st, wv, (uint32_t*)(w + L.defl));
        launch_dilate_paint(fgm, shm, meta, pool, gcount, goff, gg, B, dlab, &acc, A, (flags & kFlagApproxLt) != 0, hdr,
                            st, wv);
      }
    }
  }
  // tiles handed to the atomic kernel (LT^2 into B, whose y-pass words are consumed) and their
  // reductions; then the closed forms.  The fixed-point scale does not depend on Dmax, so the
  // per-chunk sums are final.
  launch_dilate_fallback(meta, cent, fbl, g, B, hdr, st);
  launch_epilogue_fallback(dlab, A, meta, fbl, g, acc, B, hdr, st);
  launch_metrics(acc, g, outs, hdr, st);
  // halo check: the chunked z pass and dilation were exact iff both halos fit in one chunk.
  // Decided first: the status bits of an inexact pass are not trusted (the caller reruns).
  WsHeader h;
  e = cudaMemcpyAsync(&h, hdr, sizeof h, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  for (auto& x : ev) cudaEventDestroy(x);
  if (e != cudaSuccess) return cuda_fail(e, "pipelined pass");
  uint64_t hz = 0;
  while (hz * hz < h.dxymax && hz <= (uint64_t)kChunkZ) ++hz;
  uint64_t rr = 0;
  while ((rr + 1) * (rr + 1) <= (h.dmax ? h.dmax - 1 : 0) && rr <= (uint64_t)kChunkZ) ++rr;
  if (hz > (uint64_t)kChunkZ || rr > (uint64_t)kChunkZ || h.dxymax >= kInf) return FASTRS_OK;  // not exact: rerun
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  *exact = true;
  return FASTRS_OK;
}

}  // namespace

// shared with the slab driver (slab.cu): the thread-local message of fastrs_last_error
int set_error(int code, const char* msg) {
  t_err = msg;
  return code;
}
}  // namespace fastrs

using namespace fastrs;

extern "C" {

int fastrs_workspace_bytes(const int64_t* dims, int ndim, int64_t batch, int32_t max_label, uint32_t flags,
                           size_t* bytes) {
  Geom g;
  int rc = make_geom(dims, ndim, batch, g);
  if (rc) return rc;
  if (!bytes) return fail(FASTRS_EINVAL, "bytes is NULL");
  if (max_label < 0) return fail(FASTRS_EINVAL, "max_label < 0");
  *bytes = make_layout(g, max_label, flags).total;
  return FASTRS_OK;
}

int fastrs_edt_sq(const int32_t* labels, const int64_t* dims, int ndim, int64_t batch, uint32_t flags,
                  uint32_t* d2_out, void* ws, size_t ws_bytes, void* stream) {
  Geom g;
  int rc = make_geom(dims, ndim, batch, g);
  if (rc) return rc;
  if (!d2_out) return fail(FASTRS_EINVAL, "d2_out is NULL");
  return run(labels, g, 0, flags, kEdtOnly, d2_out, nullptr, nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream);
}

int fastrs_local_thickness(const int32_t* labels, const int64_t* dims, int ndim, int64_t batch, uint32_t flags,
                           uint32_t* lt2_out, float* lt_out, void* ws, size_t ws_bytes, void* stream) {
  Geom g;
  int rc = make_geom(dims, ndim, batch, g);
  if (rc) return rc;
  if (!lt2_out && !lt_out) return fail(FASTRS_EINVAL, "both lt2_out and lt_out are NULL");
  return run(labels, g, 0, flags, kLtOnly, nullptr, lt2_out, lt_out, nullptr, ws, ws_bytes, (cudaStream_t)stream);
}

int fastrs_sphericity_roundness(const int32_t* labels, const int64_t* dims, int ndim, int64_t batch,
                                int32_t max_label, uint32_t flags, double* sphericity, double* roundness,
                                const fastrs_object_stats* stats, void* ws, size_t ws_bytes, void* stream) {
  Geom g;
  int rc = make_geom(dims, ndim, batch, g);
  if (rc) return rc;
  if (max_label < 1) return fail(FASTRS_EINVAL, "max_label must be >= 1");
  Outputs o{};
  o.sphericity = sphericity;
  o.roundness = roundness;
  if (stats) {
    o.volume = stats->volume;
    o.n_shell = stats->n_shell;
    o.max_lt2 = stats->max_lt2;
    o.mean_lt = stats->mean_lt;
    o.max_lt = stats->max_lt;
    o.shell_mean_lt = stats->shell_mean_lt;
    o.axis_a = stats->axis_a;
    o.axis_cb = stats->axis_cb;
  }
  return run(labels, g, max_label, flags, kFull, nullptr, nullptr, nullptr, &o, ws, ws_bytes, (cudaStream_t)stream);
}

int fastrs_sphericity_roundness_host(const int32_t* labels_host, const int64_t* dims, int ndim, int64_t batch,
                                     int32_t max_label, uint32_t flags, double* sphericity_host,
                                     double* roundness_host, void* ws, size_t ws_bytes, void* stream) {
  Geom g;
  int rc = make_geom(dims, ndim, batch, g);
  if (rc) return rc;
  if (max_label < 1) return fail(FASTRS_EINVAL, "max_label must be >= 1");
  if (!labels_host || !ws) return fail(FASTRS_EINVAL, "NULL pointer");
  const Layout L = make_layout(g, max_label, kFlagHostIO);
  if (ws_bytes < L.total) return fail(FASTRS_ENOMEM, "workspace too small for HOST_IO: %zu < %zu", ws_bytes, L.total);
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)ws;
  int32_t* dlab = (int32_t*)(w + L.h_labels);
  double* dsph = (double*)(w + L.h_sph);
  double* drnd = (double*)(w + L.h_rnd);
  Outputs o{};
  o.sphericity = dsph;
  o.roundness = drnd;
  bool done = false;
  if (g.ndim == 3 && g.B == 1 && g.Z >= 4 * kChunkZ && !(flags & kFlagForceFallback)) {
    rc = run_host_pipelined(labels_host, dlab, g, max_label, flags, o, ws, st, &done);
    if (rc) return rc;
  } else {
    cudaError_t e0 = cudaMemcpyAsync(dlab, labels_host, (size_t)g.N * 4, cudaMemcpyHostToDevice, st);
    if (e0 != cudaSuccess) return cuda_fail(e0, "H2D labels");
  }
  if (!done) {  // plain path (labels resident in dlab)
    rc = run(dlab, g, max_label, flags | kFlagAsync, kFull, nullptr, nullptr, nullptr, &o, ws, ws_bytes, st);
    if (rc) return rc;
  }
  cudaError_t e = cudaSuccess;
  const size_t M = (size_t)g.B * max_label;
  uint32_t status = 0;
  e = cudaMemcpyAsync(&status, w + make_layout(g, max_label, 0).hdr, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && sphericity_host) e = cudaMemcpyAsync(sphericity_host, dsph, M * 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && roundness_host) e = cudaMemcpyAsync(roundness_host, drnd, M * 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "D2H results");
  if (status & kStBadLabel) return fail(FASTRS_EINVAL, "a label is < 0 or > max_label");
  if (status & kStNoSite) return fail(FASTRS_ENOSITE, "an object element has no site");
  if (status & (kStInternal | kStShell)) return fail(FASTRS_EINTERNAL, "device invariant violated (bits %u)", status);
  return FASTRS_OK;
}

int fastrs_touches_edge(const int32_t* labels, const int64_t* dims, int ndim, int64_t batch, int32_t max_label,
                        uint8_t* touches_edge, uint32_t flags, void* stream) {
  Geom g;
  int rc = make_geom(dims, ndim, batch, g);
  if (rc) return rc;
  if (!labels || !touches_edge) return fail(FASTRS_EINVAL, "NULL pointer");
  if (max_label < 1) return fail(FASTRS_EINVAL, "max_label must be >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = launch_touch_edge(labels, g, max_label, touches_edge, (flags & kFlagEdgeSkipZlo) && g.ndim == 3,
                                    (flags & kFlagEdgeSkipZhi) && g.ndim == 3, st);
  if (e == cudaSuccess && !(flags & kFlagAsync)) e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? FASTRS_OK : cuda_fail(e, "touches_edge");
}

int fastrs_filter_objects(double* sphericity, double* roundness, const int64_t* volume, const uint8_t* touches_edge,
                          int64_t n_labels, int64_t min_volume, uint32_t flags, void* stream) {
  if (n_labels < 0) return fail(FASTRS_EINVAL, "n_labels < 0");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = launch_filter(sphericity, roundness, volume, touches_edge, n_labels, min_volume, st);
  if (e == cudaSuccess && !(flags & kFlagAsync)) e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? FASTRS_OK : cuda_fail(e, "filter_objects");
}

int fastrs_read_diagnostics(const void* ws, fastrs_diagnostics* out, void* stream) {
  if (!ws || !out) return fail(FASTRS_EINVAL, "NULL pointer");
  WsHeader h;
  cudaError_t e = cudaMemcpyAsync(&h, ws, sizeof h, cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "read diagnostics");
  out->status_bits = h.status;
  out->dmax = h.dmax;
  out->n_fg = h.n_fg;
  out->n_kept = h.n_kept;
  out->n_intervals = h.n_intervals;
  out->sum_scale_log2 = 32;
  out->n_fallback = h.n_fallback;
  out->n_rounds_extra = h.n_rounds_extra;
  out->n_regathers = h.n_regathers;
  out->n_staged = h.n_staged;
  out->max_group_list = h.max_group_list;
  out->sum_group_list = h.sum_group_list;
  out->n_painted = h.n_painted;
  out->n_covering = h.n_covering;
  out->n_deferred = h.n_defer[0] + h.n_defer[1] + h.n_defer[2] + h.n_defer[3];
  out->n_col_slow = h.slow_n;
  out->reserved = 0;
  return FASTRS_OK;
}

void fastrs_profile(int enable) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof = enable != 0;
  if (g_prof) {
    for (double& v : g_prof_ms) v = 0;
    g_prof_calls = 0;
  }
}

int fastrs_profile_read(double* ms_out, int64_t* calls_out, int n_stages) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (int k = 0; k < n_stages && k < kStages; ++k) ms_out[k] = g_prof_ms[k];
  if (calls_out) *calls_out = g_prof_calls;
  return kStages;
}

const char* fastrs_last_error(void) { return t_err.c_str(); }

void fastrs_release(void) { release_mtables(); }

// ---- z-slab multi-GPU path -----------------------------------------------------------------
int fastrs_slab_workspace_bytes(const int64_t* dims_ext, size_t* bytes) {
  Geom g;
  int rc = make_geom(dims_ext, 3, 1, g);
  if (rc) return rc;
  if (!bytes) return fail(FASTRS_EINVAL, "bytes is NULL");
  *bytes = make_slab_layout(g).total;
  return FASTRS_OK;
}

int fastrs_slab_edt_xy(const int32_t* labels, const int32_t* labels_below, const int64_t* dims, int32_t max_label,
                       uint32_t flags, uint32_t* packed_out, uint32_t* dxy_max, void* ws, size_t ws_bytes,
                       void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  Geom g;
  SlabLayout L{};
  WsHeader* hdr = nullptr;
  int rc = slab_prologue(dims, g, L, ws, ws_bytes, hdr, st);
  if (rc) return rc;
  if (!labels || !packed_out) return fail(FASTRS_EINVAL, "NULL pointer");
  uint32_t* tmp = (uint32_t*)((char*)ws + L.P);
  const bool border = (flags & kFlagBorder) != 0;
  launch_edt_x(labels, labels_below, tmp, g, max_label > 0 ? max_label : INT32_MAX, border, hdr, st);
  launch_edt_col(tmp, packed_out, g, 1, false, border, hdr, (uint32_t*)((char*)ws + L.sat), st, 0, -1, 0, -1,
                 (char*)ws + L.pool, (size_t)dilate_pool_entries(g) * 8);
  rc = header_word_out(hdr, &hdr->dxymax, dxy_max, st);
  if (rc) return rc;
  return finish_call(hdr, flags, st);
}

int fastrs_slab_edt_z(const uint32_t* packed_ext, const int64_t* dims_ext, int64_t own_lo, int64_t own_hi,
                      int64_t z_ext0, int64_t Z, uint32_t flags, uint32_t* d_out, uint32_t* dmax_out, void* ws,
                      size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  Geom g;
  SlabLayout L{};
  WsHeader* hdr = nullptr;
  int rc = slab_prologue(dims_ext, g, L, ws, ws_bytes, hdr, st);
  if (rc) return rc;
  if (!packed_ext || !d_out) return fail(FASTRS_EINVAL, "NULL pointer");
  if (own_lo < 0 || own_hi > g.Z || own_lo >= own_hi || z_ext0 < 0 || z_ext0 + g.Z > Z)
    return fail(FASTRS_EINVAL, "slab range outside the extended slab / the grid");
  launch_edt_col(packed_ext, d_out, g, 2, true, (flags & kFlagBorder) != 0, hdr, (uint32_t*)((char*)ws + L.sat), st, own_lo,
                 own_hi, z_ext0, Z, (char*)ws + L.pool, (size_t)dilate_pool_entries(g) * 8);
  rc = header_word_out(hdr, &hdr->dmax, dmax_out, st);
  if (rc) return rc;
  return finish_call(hdr, flags, st);
}

}  // extern "C"

namespace fastrs {
namespace {
// K5 (gather, paint with fused reductions, fallback) of the own tiles of an extended slab whose
// K4 outputs are in the workspace (own layers from K4, halo layers from K4 or unpacked)
int slab_dilate_impl(const int32_t* labels, const uint32_t* d_ext, Geom g, const SlabLayout& L, WsHeader* hdr,
                     int64_t own_lo, int64_t own_hi, int64_t Z, uint32_t dmax_global, int32_t max_label,
                     uint32_t flags, uint64_t* vol, uint64_t* n_shell, uint64_t* sum_lt, uint64_t* sum_shell_lt,
                     uint32_t* max_lt2, void* ws, cudaStream_t st) {
  g.tz_lo = own_lo / kTZ3;
  g.tz_hi = (own_hi + kTZ3 - 1) / kTZ3;
  g.nscale = Z * g.Y * g.X;
  const int64_t M = max_label;
  cudaError_t e = cudaSuccess;
  for (void* a : {(void*)vol, (void*)n_shell})
    if (e == cudaSuccess) e = cudaMemsetAsync(a, 0, (size_t)M * 8, st);
  for (void* a : {(void*)sum_lt, (void*)sum_shell_lt})
    if (e == cudaSuccess) e = cudaMemsetAsync(a, 0, (size_t)M * 16, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(max_lt2, 0, (size_t)M * 4, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  k_set_dmax<<<1, 1, 0, st>>>(hdr, dmax_global);
  TileMeta* meta = (TileMeta*)((char*)ws + L.meta);
  uint2* cent = (uint2*)((char*)ws + L.cent);
  uint32_t* fgm = (uint32_t*)((char*)ws + L.fgm);
  uint32_t* shm = (uint32_t*)((char*)ws + L.shm);
  uint16_t* oct = (uint16_t*)((char*)ws + L.oct);
  Accum acc{};
  acc.vol = (unsigned long long*)vol;
  acc.nshell = (unsigned long long*)n_shell;
  acc.sum = (unsigned long long*)sum_lt;
  acc.sumshell = (unsigned long long*)sum_shell_lt;
  acc.maxlt2 = max_lt2;
  acc.M = M;
  acc.max_label = max_label;
  // labels are indexed in the extended layout: shift the own-slab pointer (only own elements
  // are ever read: the fused paint reads labels at covered cells of own tiles)
  const int32_t* lab_ext = labels - own_lo * g.Y * g.X;
  uint32_t* ltp = (uint32_t*)((char*)ws + L.P);
  uint32_t* fbl = (uint32_t*)((char*)ws + L.fbl);
  unsigned long long* pool = (unsigned long long*)((char*)ws + L.pool);
  uint32_t* gcount = (uint32_t*)((char*)ws + L.gcount);
  uint32_t* goff = (uint32_t*)((char*)ws + L.goff);
  for (int wv = 0; wv < kDilateWaves; ++wv) {
    launch_dilate_gather(fgm, meta, cent, oct, fbl, pool, gcount, goff, g, gather_mode_of(flags), hdr, st, wv,
                         (uint32_t*)((char*)ws + L.defl));
    launch_dilate_paint(fgm, shm, meta, pool, gcount, goff, g, ltp, lab_ext, &acc, d_ext, (flags & kFlagApproxLt) != 0,
                        hdr, st, wv);
  }
  launch_dilate_fallback(meta, cent, fbl, g, ltp, hdr, st);
  launch_epilogue_fallback(lab_ext, d_ext, meta, fbl, g, acc, ltp, hdr, st);
  return FASTRS_OK;
}

int check_own(const Geom& g, int64_t own_lo, int64_t own_hi) {
  if (own_lo < 0 || own_hi > g.Z || own_lo >= own_hi || (own_lo % kTZ3) != 0 || ((own_hi % kTZ3) != 0 && own_hi != g.Z))
    return fail(FASTRS_EINVAL, "own slab range must be tile aligned (multiples of 8 slices) inside the extended slab");
  return FASTRS_OK;
}
}  // namespace
}  // namespace fastrs

extern "C" {

int fastrs_slab_reduce(const int32_t* labels, const uint32_t* d_ext, const int64_t* dims_ext, int64_t own_lo,
                       int64_t own_hi, int64_t Z, uint32_t dmax_global, int32_t max_label, uint32_t flags,
                       uint64_t* vol, uint64_t* n_shell, uint64_t* sum_lt, uint64_t* sum_shell_lt, uint32_t* max_lt2,
                       void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  Geom g;
  SlabLayout L{};
  WsHeader* hdr = nullptr;
  int rc = slab_prologue(dims_ext, g, L, ws, ws_bytes, hdr, st);
  if (rc) return rc;
  if (!labels || !d_ext || !vol || !n_shell || !sum_lt || !sum_shell_lt || !max_lt2 || max_label < 1)
    return fail(FASTRS_EINVAL, "NULL pointer or max_label < 1");
  if ((rc = check_own(g, own_lo, own_hi))) return rc;
  // K4 on every tile of the extended slab (the halo tiles from the D halo), then K5 on the own tiles
  launch_prune(d_ext, g, (TileMeta*)((char*)ws + L.meta), (uint2*)((char*)ws + L.cent), (uint32_t*)((char*)ws + L.fgm),
               (uint32_t*)((char*)ws + L.shm), (uint16_t*)((char*)ws + L.oct), hdr, st);
  rc = slab_dilate_impl(labels, d_ext, g, L, hdr, own_lo, own_hi, Z, dmax_global, max_label, flags, vol, n_shell,
                        sum_lt, sum_shell_lt, max_lt2, ws, st);
  if (rc) return rc;
  return finish_call(hdr, flags, st);
}

int fastrs_slab_prune(const uint32_t* d_ext, const int64_t* dims_ext, int64_t own_lo, int64_t own_hi, uint32_t flags,
                      void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  Geom g;
  SlabLayout L{};
  WsHeader* hdr = nullptr;
  int rc = slab_prologue(dims_ext, g, L, ws, ws_bytes, hdr, st);
  if (rc) return rc;
  if (!d_ext) return fail(FASTRS_EINVAL, "NULL pointer");
  if ((rc = check_own(g, own_lo, own_hi))) return rc;
  TileMeta* meta = (TileMeta*)((char*)ws + L.meta);
  // halo layers read as empty until fastrs_slab_unpack_tiles fills them
  cudaError_t e = cudaMemsetAsync(meta, 0, (size_t)g.ntiles * sizeof(TileMeta), st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  launch_prune(d_ext, g, meta, (uint2*)((char*)ws + L.cent), (uint32_t*)((char*)ws + L.fgm),
               (uint32_t*)((char*)ws + L.shm), (uint16_t*)((char*)ws + L.oct), hdr, st, own_lo / kTZ3,
               (own_hi + kTZ3 - 1) / kTZ3);
  return finish_call(hdr, flags, st);
}

int fastrs_slab_pack_tiles(void* ws, const int64_t* dims_ext, int64_t tz_a, int64_t tz_b, uint32_t* rec_out,
                           void* ent_out, uint64_t* n_entries, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  Geom g;
  int rc = make_geom(dims_ext, 3, 1, g);
  if (rc) return rc;
  if (!ws || !rec_out || !ent_out || !n_entries || tz_a < 0 || tz_b > g.ntz || tz_a >= tz_b)
    return fail(FASTRS_EINVAL, "bad pack arguments");
  const SlabLayout L = make_slab_layout(g);
  const int64_t t0 = tz_a * g.nty * g.ntx, n = (tz_b - tz_a) * g.nty * g.ntx;
  uint32_t* off = (uint32_t*)((char*)ws + L.poff);
  k_tile_prefix<<<1, 1024, 0, st>>>((const TileMeta*)((char*)ws + L.meta), nullptr, t0, n, off,
                                    (unsigned long long*)n_entries);
  k_tile_pack<<<(unsigned)n, 128, 0, st>>>((const TileMeta*)((char*)ws + L.meta), (const uint16_t*)((char*)ws + L.oct),
                                           (const uint2*)((char*)ws + L.cent), t0, off, rec_out, (uint2*)ent_out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FASTRS_OK : cuda_fail(e, "pack tiles");
}

int fastrs_slab_unpack_tiles(void* ws, const int64_t* dims_ext, int64_t tz_a, int64_t tz_b, const uint32_t* rec_in,
                             const void* ent_in, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  Geom g;
  int rc = make_geom(dims_ext, 3, 1, g);
  if (rc) return rc;
  if (!ws || !rec_in || !ent_in || tz_a < 0 || tz_b > g.ntz || tz_a >= tz_b)
    return fail(FASTRS_EINVAL, "bad unpack arguments");
  const SlabLayout L = make_slab_layout(g);
  const int64_t t0 = tz_a * g.nty * g.ntx, n = (tz_b - tz_a) * g.nty * g.ntx;
  uint32_t* off = (uint32_t*)((char*)ws + L.poff);
  k_tile_prefix<<<1, 1024, 0, st>>>(nullptr, rec_in, t0, n, off, nullptr);
  k_tile_unpack<<<(unsigned)n, 128, 0, st>>>((TileMeta*)((char*)ws + L.meta), (uint16_t*)((char*)ws + L.oct),
                                             (uint2*)((char*)ws + L.cent), t0, off, rec_in, (const uint2*)ent_in);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FASTRS_OK : cuda_fail(e, "unpack tiles");
}

int fastrs_slab_dilate(const int32_t* labels, const uint32_t* d_ext, const int64_t* dims_ext, int64_t own_lo,
                       int64_t own_hi, int64_t Z, uint32_t dmax_global, int32_t max_label, uint32_t flags,
                       uint64_t* vol, uint64_t* n_shell, uint64_t* sum_lt, uint64_t* sum_shell_lt, uint32_t* max_lt2,
                       void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  Geom g;
  int rc = make_geom(dims_ext, 3, 1, g);
  if (rc) return rc;
  if (!ws || ((uintptr_t)ws & 255) != 0) return fail(FASTRS_EINVAL, "workspace NULL or not 256-byte aligned");
  const SlabLayout L = make_slab_layout(g);
  if (ws_bytes < L.total) return fail(FASTRS_ENOMEM, "workspace too small: %zu < %zu bytes", ws_bytes, L.total);
  if (!labels || !d_ext || !vol || !n_shell || !sum_lt || !sum_shell_lt || !max_lt2 || max_label < 1)
    return fail(FASTRS_EINVAL, "NULL pointer or max_label < 1");
  if ((rc = check_own(g, own_lo, own_hi))) return rc;
  WsHeader* hdr = (WsHeader*)((char*)ws + L.hdr);
  cudaError_t e = cudaMemsetAsync(hdr, 0, 256, st);  // (the tile data of fastrs_slab_prune stays)
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  rc = slab_dilate_impl(labels, d_ext, g, L, hdr, own_lo, own_hi, Z, dmax_global, max_label, flags, vol, n_shell,
                        sum_lt, sum_shell_lt, max_lt2, ws, st);
  if (rc) return rc;
  return finish_call(hdr, flags, st);
}

int fastrs_metrics_from_partials(const uint64_t* vol, const uint64_t* n_shell, const uint64_t* sum_lt,
                                 const uint64_t* sum_shell_lt, const uint32_t* max_lt2, int64_t n_labels, int ndim,
                                 int64_t nscale, uint32_t dmax_global, double* sphericity, double* roundness,
                                 const fastrs_object_stats* stats, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!vol || !n_shell || !sum_lt || !sum_shell_lt || !max_lt2 || n_labels < 1 || nscale < 1)
    return fail(FASTRS_EINVAL, "NULL pointer or empty sizes");
  if (ndim != 2 && ndim != 3) return fail(FASTRS_EINVAL, "ndim must be 2 or 3");
  if (!ws || ws_bytes < 256 || ((uintptr_t)ws & 255) != 0) return fail(FASTRS_ENOMEM, "workspace must be >= 256 aligned bytes");
  WsHeader* hdr = (WsHeader*)ws;
  cudaError_t e = cudaMemsetAsync(hdr, 0, 256, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  k_set_dmax<<<1, 1, 0, st>>>(hdr, dmax_global);
  Accum acc{};
  acc.vol = (unsigned long long*)vol;
  acc.nshell = (unsigned long long*)n_shell;
  acc.sum = (unsigned long long*)sum_lt;
  acc.sumshell = (unsigned long long*)sum_shell_lt;
  acc.maxlt2 = (uint32_t*)max_lt2;
  acc.M = n_labels;
  acc.max_label = (int32_t)n_labels;
  Outputs o{};
  o.sphericity = sphericity;
  o.roundness = roundness;
  if (stats) {
    o.volume = stats->volume;
    o.n_shell = stats->n_shell;
    o.max_lt2 = stats->max_lt2;
    o.mean_lt = stats->mean_lt;
    o.max_lt = stats->max_lt;
    o.shell_mean_lt = stats->shell_mean_lt;
    o.axis_a = stats->axis_a;
    o.axis_cb = stats->axis_cb;
  }
  Geom g{};
  g.ndim = ndim;
  g.nscale = nscale;
  launch_metrics(acc, g, o, hdr, st);
  return finish_call(hdr, 0, st);
}

}  // extern "C"
