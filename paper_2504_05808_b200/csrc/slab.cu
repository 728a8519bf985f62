// Multi-GPU z-slab driver inside libfastrs (north_star "a single large
// volume is split into z-slabs, with an NCCL all-to-all transpose for the EDT z-pass, a halo
// exchange of max-radius width for the dilation, and an allreduce of per-label partial sums").
//
// One process per GPU, one rank per z-slab.  NCCL is loaded at run time (dlopen of
// libnccl.so.2: the copy torch already mapped into the process, else the system one), so the
// library loads without it.  The communicator comes from fastrs_comm_init with a unique id the
// caller broadcasts (paper_2504_05808_b200/slab.py uses torch.distributed for that plumbing).
// Every computation runs in the same kernels as the single-GPU call, through the four slab
// phases of the C ABI (api.cu); this file plans and performs the exchanges between them:
//
//   0  labels of the slice below the slab (z-run flags of its first slice): 1-slice halo
//   A  K1 + K2 on the own slab -> packed words; allreduce(max) of max D_xy -> h
//   B  z pass, one of
//        N8 halo      : the h packed slices on each side (multi-hop plan when h exceeds a
//                       neighbour's slab), K3 on the h-extended slab
//        N1 transpose : all-to-all of the packed words from z-slabs to y-slabs ([Z][Y/P][X]
//                       per rank, no halo), K3 over whole z columns, all-to-all of D back
//      allreduce(max) of Dmax -> H = isqrt(Dmax - 1) rounded up to a tile layer
//   C  the H slices of D on each side; K4 on the H-extended slab, K5 (fused reductions) on the
//      own tiles -> exact integer partial sums; allreduce(sum) of the u64 words, allreduce(max)
//      of max LT^2
//   D  K6 closed forms -> every rank holds all labels' results
// Exactness: as slab.py (the z pass at an own element only looks sqrt(D_xy) <= h away; a kept
// ball reaching the own slab is centred within H slices; integer partials), so the result is
// bit-identical to fastrs_sphericity_roundness on the whole volume.
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "fastrs.h"

namespace fastrs {
namespace {

// ---- NCCL through dlopen ---------------------------------------------------------------
struct Nccl {
  bool tried = false, ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (n.tried) return n;
  n.tried = true;
  const char* env = getenv("FASTRS_NCCL_LIB");
  void* h = nullptr;
  if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // torch's copy, if mapped
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    n.why = "cannot load libnccl.so.2";
    return n;
  }
  auto sym = [&](auto& fn, const char* name) {
    fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
    if (!fn) n.why = std::string("libnccl lacks ") + name;
    return fn != nullptr;
  };
  n.ok = sym(n.GetUniqueId, "ncclGetUniqueId") && sym(n.CommInitRank, "ncclCommInitRank") &&
         sym(n.CommDestroy, "ncclCommDestroy") && sym(n.AllReduce, "ncclAllReduce") && sym(n.Send, "ncclSend") &&
         sym(n.Recv, "ncclRecv") && sym(n.GroupStart, "ncclGroupStart") && sym(n.GroupEnd, "ncclGroupEnd") &&
         sym(n.GetErrorString, "ncclGetErrorString");
  return n;
}

struct Comm {
  ncclComm_t c = nullptr;
  int rank = 0, nranks = 1, device = 0;
  cudaStream_t xs = nullptr;              // exchange stream (the z-halo overlaps the interior z pass)
  cudaEvent_t ev_a = nullptr, ev_x = nullptr;
};

int err(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  return set_error(code, buf);
}
int nccl_fail(ncclResult_t r, const char* where) {
  return err(FASTRS_ENCCL, "%s: %s", where, nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error");
}
int cuda_err(cudaError_t e, const char* where) { return err(FASTRS_ECUDA, "%s: %s", where, cudaGetErrorString(e)); }

#define NCCL_TRY(call, where)                 \
  do {                                        \
    ncclResult_t r_ = (call);                 \
    if (r_ != ncclSuccess) return nccl_fail(r_, where); \
  } while (0)
#define CUDA_TRY(call, where)                 \
  do {                                        \
    cudaError_t e_ = (call);                  \
    if (e_ != cudaSuccess) return cuda_err(e_, where); \
  } while (0)

// ---- plans (pure host code; exported for the CPU tests) ---------------------------------
constexpr int64_t kAlign = kTZ3;  // slab boundaries fall on K4/K5 tile layers

bool partition(int64_t Z, int P, std::vector<int64_t>& b) {
  b.assign(P + 1, 0);
  for (int i = 1; i < P; ++i) {
    // the rule of slab.py: round(Z * i / P / 8) * 8 (round half to even), kept monotone
    int64_t v = (int64_t)std::nearbyint((double)Z * i / P / (double)kAlign) * kAlign;
    v = v < b[i - 1] ? b[i - 1] : (v > Z ? Z : v);
    b[i] = v;
  }
  b[P] = Z;
  for (int i = 0; i < P; ++i)
    if (b[i + 1] <= b[i]) return false;
  return true;
}

struct Xfer {
  int src, dst, side;  // side 0: the receiver's lo halo, 1: its hi halo
  int64_t a, b;        // global slices [a, b)
};

// transfers that give every rank the w slices below (sides & 1) and above (sides & 2) its slab
// (several sources when w exceeds a neighbour's slab)
std::vector<Xfer> halo_plan(const std::vector<int64_t>& bd, int64_t w, int64_t Z, int sides = 3) {
  std::vector<Xfer> plan;
  const int P = (int)bd.size() - 1;
  for (int dst = 0; dst < P; ++dst) {
    const int64_t z0 = bd[dst], z1 = bd[dst + 1];
    const int64_t rng[2][2] = {{z0 - w > 0 ? z0 - w : 0, z0}, {z1, z1 + w < Z ? z1 + w : Z}};
    for (int side = 0; side < 2; ++side)
      for (int src = 0; src < P && ((sides >> side) & 1); ++src) {
        const int64_t lo = rng[side][0] > bd[src] ? rng[side][0] : bd[src];
        const int64_t hi = rng[side][1] < bd[src + 1] ? rng[side][1] : bd[src + 1];
        if (src != dst && lo < hi) plan.push_back({src, dst, side, lo, hi});
      }
  }
  return plan;
}

int64_t halo_edt(uint32_t dxy, int64_t Z) {  // smallest h with h^2 >= max D_xy (Z when no site)
  if (dxy >= kInf) return Z;
  if (dxy == 0) return 0;
  int64_t r = (int64_t)std::sqrt((double)(dxy - 1));
  while (r * r > (int64_t)dxy - 1) --r;
  while ((r + 1) * (r + 1) <= (int64_t)dxy - 1) ++r;
  return r + 1;
}
int64_t halo_lt(uint32_t dmax) {  // isqrt(Dmax - 1) rounded up to a tile layer
  if (dmax == 0) return 0;
  int64_t r = (int64_t)std::sqrt((double)(dmax - 1));
  while (r * r > (int64_t)dmax - 1) --r;
  while ((r + 1) * (r + 1) <= (int64_t)dmax - 1) ++r;
  return (r + kAlign - 1) / kAlign * kAlign;
}

// halo exchange of whole slices of `elem` 4-byte words: every rank sends the slices others need
// from its own slab `own` (global slices [z0, z1)) and receives into `ext`, whose slot 0 is
// global slice z0 - cap
int exchange(const Comm& cm, const std::vector<Xfer>& plan, const std::vector<int64_t>& bd, const void* own, void* ext,
             int64_t cap, int64_t YX, ncclDataType_t dt, cudaStream_t st, uint64_t* sent, uint64_t* recvd) {
  if (plan.empty()) return FASTRS_OK;
  Nccl& n = nccl();
  const int64_t z0 = bd[cm.rank];
  NCCL_TRY(n.GroupStart(), "ncclGroupStart");
  for (const Xfer& x : plan) {
    const size_t cnt = (size_t)((x.b - x.a) * YX);
    if (x.src == cm.rank) {
      NCCL_TRY(n.Send((const uint32_t*)own + (x.a - z0) * YX, cnt, dt, x.dst, cm.c, st), "ncclSend");
      *sent += cnt * 4;
    }
    if (x.dst == cm.rank) {
      NCCL_TRY(n.Recv((uint32_t*)ext + (x.a - (z0 - cap)) * YX, cnt, dt, x.src, cm.c, st), "ncclRecv");
      *recvd += cnt * 4;
    }
  }
  NCCL_TRY(n.GroupEnd(), "ncclGroupEnd");
  return FASTRS_OK;
}

// total kept centres announced by n tile records (FASTRS_TILE_RECORD_WORDS u32 each, count first)
__global__ void k_count_entries(const uint32_t* __restrict__ rec, int64_t n, uint64_t* __restrict__ out) {
  uint32_t c = 0;  // (<= 2048 per tile: no u32 overflow per thread or warp for < 2^21 tiles)
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) c += rec[i * FASTRS_TILE_RECORD_WORDS];
  const unsigned long long s = __reduce_add_sync(0xFFFFFFFFu, c);
  __shared__ unsigned long long w[8];
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += w[i];
    *out = t;
  }
}

__global__ void k_status_flags(const uint32_t* __restrict__ st, int n, uint32_t* __restrict__ flags) {
  uint32_t s = 0;
  for (int i = 0; i < n; ++i) s |= st[i];
  flags[0] = (s & kStBadLabel) ? 1u : 0u;
  flags[1] = (s & kStNoSite) ? 1u : 0u;
  flags[2] = (s & kStInternal) ? 1u : 0u;
  flags[3] = (s & kStShell) ? 1u : 0u;
}

inline size_t al256(size_t v) { return (v + 255) & ~size_t(255); }

struct CallLayout {
  size_t stat, flags, dxy, dmax, below, ext, dext, t0, t1, part, srec, sent, rrec, rent, cnt, phase, phase_bytes, total;
  int64_t send_tiles, recv_tiles;  // capacities of the kept-centre halo buffers (tiles)
};

int slab_phase_bytes(int64_t nz, int64_t Y, int64_t X, size_t* out) {
  const int64_t d[3] = {nz, Y, X};
  return fastrs_slab_workspace_bytes(d, out);
}

// workspace of one slab call: the exchange buffers, the partial sums and one phase workspace
// sized for the largest geometry a phase runs on
int call_layout(const std::vector<int64_t>& bd, int rank, int64_t Y, int64_t X, int32_t max_label, int64_t cap,
                bool transpose, bool dense, CallLayout& L) {
  const int P = (int)bd.size() - 1;
  const int64_t nz = bd[rank + 1] - bd[rank], Z = bd[P];
  const int64_t YX = Y * X, M = max_label;
  const int64_t ym = (Y * (rank + 1)) / P - (Y * rank) / P;
  size_t off = 0;
  auto take = [&](size_t b) {
    const size_t o = off;
    off += al256(b);
    return o;
  };
  L.stat = take(16 * 4);
  L.flags = take(4 * 4);
  L.dxy = take(4);
  L.dmax = take(3 * 4);  // one max D per z-pass launch (interior / two boundary ranges)
  L.below = take((size_t)YX * 4);
  L.ext = take((size_t)(nz + 2 * cap) * YX * 4);   // packed words (N8 halo) / own packed slab
  L.dext = take((size_t)(nz + 2 * cap) * YX * 4);  // D with its H halo
  const size_t tsz = transpose ? (size_t)((nz * YX > Z * ym * X) ? nz * YX : Z * ym * X) * 4 : 0;
  L.t0 = take(tsz);  // N1: send buffer, then D of the y-slab
  L.t1 = take(tsz);  // N1: receive buffers
  L.part = take((size_t)M * 8 * 6 + (size_t)M * 4);
  // kept-centre halo (N4): K4 records (FASTRS_TILE_RECORD_WORDS u32 per tile) and kept centres (<= 2048 per tile)
  const int64_t tpl = ((Y + kTZ3 - 1) / kTZ3) * ((X + 31) / 32), capl = (cap + kTZ3 - 1) / kTZ3;
  L.recv_tiles = dense ? 0 : 2 * capl * tpl;
  L.send_tiles = dense ? 0 : (2 * capl + (nz + kTZ3 - 1) / kTZ3) * tpl;
  L.srec = take((size_t)L.send_tiles * FASTRS_TILE_RECORD_WORDS * 4);
  L.sent = take((size_t)L.send_tiles * kTileVol * 8);
  L.rrec = take((size_t)L.recv_tiles * FASTRS_TILE_RECORD_WORDS * 4);
  L.rent = take((size_t)L.recv_tiles * kTileVol * 8);
  L.cnt = take((size_t)8 * P * 8);
  size_t pb = 0, v = 0;
  int rc = slab_phase_bytes(nz + 2 * cap > Z ? Z : nz + 2 * cap, Y, X, &pb);
  if (rc) return rc;
  if (transpose && ym > 0) {
    rc = slab_phase_bytes(Z, ym, X, &v);
    if (rc) return rc;
    pb = v > pb ? v : pb;
  }
  L.phase = take(pb);
  L.phase_bytes = pb;
  L.total = off;
  return FASTRS_OK;
}

}  // namespace
}  // namespace fastrs

using namespace fastrs;

extern "C" {

int fastrs_nccl_available(void) { return nccl().ok ? 1 : 0; }

int fastrs_nccl_unique_id(void* id_out) {
  if (!id_out) return err(FASTRS_EINVAL, "id_out is NULL");
  Nccl& n = nccl();
  if (!n.ok) return err(FASTRS_ENCCL, "%s", n.why.c_str());
  ncclUniqueId id;
  NCCL_TRY(n.GetUniqueId(&id), "ncclGetUniqueId");
  memcpy(id_out, &id, sizeof id);
  return FASTRS_OK;
}

int fastrs_comm_init(const void* id, int nranks, int rank, void** comm_out) {
  if (!id || !comm_out) return err(FASTRS_EINVAL, "NULL pointer");
  if (nranks < 1 || rank < 0 || rank >= nranks) return err(FASTRS_EINVAL, "rank %d of %d", rank, nranks);
  Nccl& n = nccl();
  if (!n.ok) return err(FASTRS_ENCCL, "%s", n.why.c_str());
  Comm* cm = new Comm();
  cm->rank = rank;
  cm->nranks = nranks;
  cudaGetDevice(&cm->device);
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  const ncclResult_t r = n.CommInitRank(&cm->c, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete cm;
    return nccl_fail(r, "ncclCommInitRank");
  }
  if (cudaStreamCreateWithFlags(&cm->xs, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&cm->ev_a, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&cm->ev_x, cudaEventDisableTiming) != cudaSuccess) {
    n.CommDestroy(cm->c);
    delete cm;
    return err(FASTRS_ECUDA, "exchange stream / events");
  }
  *comm_out = cm;
  return FASTRS_OK;
}

int fastrs_comm_destroy(void* comm) {
  if (!comm) return FASTRS_OK;
  Comm* cm = (Comm*)comm;
  ncclResult_t r = ncclSuccess;
  if (cm->c) r = nccl().CommDestroy(cm->c);
  if (cm->ev_a) cudaEventDestroy(cm->ev_a);
  if (cm->ev_x) cudaEventDestroy(cm->ev_x);
  if (cm->xs) cudaStreamDestroy(cm->xs);
  delete cm;
  return r == ncclSuccess ? FASTRS_OK : nccl_fail(r, "ncclCommDestroy");
}

int fastrs_slab_partition(int64_t Z, int nranks, int64_t* bounds) {
  if (!bounds || nranks < 1 || Z < 1) return err(FASTRS_EINVAL, "bad partition arguments");
  std::vector<int64_t> b;
  if (!partition(Z, nranks, b))
    return err(FASTRS_EINVAL, "cannot split Z=%lld into %d non-empty slabs aligned to %lld", (long long)Z, nranks,
               (long long)kAlign);
  for (int i = 0; i <= nranks; ++i) bounds[i] = b[i];
  return FASTRS_OK;
}

int fastrs_slab_halo_plan(const int64_t* bounds, int nranks, int64_t w, int64_t Z, int64_t* entries, int64_t cap,
                          int64_t* n_out) {
  if (!bounds || !n_out || nranks < 1 || w < 0) return err(FASTRS_EINVAL, "bad plan arguments");
  std::vector<int64_t> bd(bounds, bounds + nranks + 1);
  const std::vector<Xfer> plan = halo_plan(bd, w, Z);
  *n_out = (int64_t)plan.size();
  if (entries)
    for (size_t i = 0; i < plan.size() && (int64_t)i < cap; ++i) {
      entries[5 * i] = plan[i].src;
      entries[5 * i + 1] = plan[i].dst;
      entries[5 * i + 2] = plan[i].side;
      entries[5 * i + 3] = plan[i].a;
      entries[5 * i + 4] = plan[i].b;
    }
  return FASTRS_OK;
}

int fastrs_slab_call_workspace_bytes(const int64_t* dims_slab, int64_t z0, int64_t Z, int nranks, int rank,
                                     int32_t max_label, int64_t halo_cap, uint32_t flags, size_t* bytes) {
  if (!dims_slab || !bytes || max_label < 1 || halo_cap < 0) return err(FASTRS_EINVAL, "bad arguments");
  std::vector<int64_t> bd;
  if (!partition(Z, nranks, bd) || rank < 0 || rank >= nranks || bd[rank] != z0 ||
      bd[rank + 1] - bd[rank] != dims_slab[0])
    return err(FASTRS_EINVAL, "the slab [z0, z0 + nz) is not fastrs_slab_partition(Z, nranks)[rank]");
  CallLayout L;
  const int rc = call_layout(bd, rank, dims_slab[1], dims_slab[2], max_label, halo_cap,
                             (flags & FASTRS_SLAB_TRANSPOSE) != 0, (flags & FASTRS_SLAB_DENSE_HALO) != 0, L);
  if (rc) return rc;
  *bytes = L.total;
  return FASTRS_OK;
}

int fastrs_sphericity_roundness_slab(const int32_t* labels, const int64_t* dims_slab, int64_t z0, int64_t Z,
                                     int32_t max_label, uint32_t flags, int64_t halo_cap, double* sphericity,
                                     double* roundness, const fastrs_object_stats* stats, fastrs_slab_info* info,
                                     void* comm, void* ws, size_t ws_bytes, void* stream) {
  if (!labels || !dims_slab || !comm || !ws) return err(FASTRS_EINVAL, "NULL pointer");
  if (max_label < 1 || halo_cap < 0) return err(FASTRS_EINVAL, "max_label < 1 or halo_cap < 0");
  Comm& cm = *(Comm*)comm;
  cudaStream_t st = (cudaStream_t)stream;
  Nccl& n = nccl();
  if (!n.ok) return err(FASTRS_ENCCL, "%s", n.why.c_str());
  const int P = cm.nranks, rank = cm.rank;
  std::vector<int64_t> bd;
  if (!partition(Z, P, bd) || bd[rank] != z0 || bd[rank + 1] - z0 != dims_slab[0])
    return err(FASTRS_EINVAL, "the slab [z0, z0 + nz) is not fastrs_slab_partition(Z, nranks)[rank]");
  const int64_t nz = dims_slab[0], Y = dims_slab[1], X = dims_slab[2], YX = Y * X, z1 = z0 + nz;
  const bool transpose = (flags & FASTRS_SLAB_TRANSPOSE) != 0;
  CallLayout L;
  const bool dense = (flags & FASTRS_SLAB_DENSE_HALO) != 0;
  int rc = call_layout(bd, rank, Y, X, max_label, halo_cap, transpose, dense, L);
  if (rc) return rc;
  if (ws_bytes < L.total) return err(FASTRS_ENOMEM, "workspace too small: %zu < %zu bytes", ws_bytes, L.total);
  if (((uintptr_t)ws & 255) != 0) return err(FASTRS_EINVAL, "workspace must be 256-byte aligned");
  char* w = (char*)ws;
  uint32_t* stat = (uint32_t*)(w + L.stat);
  uint32_t* sflags = (uint32_t*)(w + L.flags);
  uint32_t* dxy = (uint32_t*)(w + L.dxy);
  uint32_t* dmx = (uint32_t*)(w + L.dmax);
  int32_t* below = (int32_t*)(w + L.below);
  uint32_t* ext = (uint32_t*)(w + L.ext);
  uint32_t* dext = (uint32_t*)(w + L.dext);
  uint64_t* part = (uint64_t*)(w + L.part);
  void* pw = w + L.phase;
  const size_t pwb = L.phase_bytes;
  const uint32_t pf = (flags & (FASTRS_BORDER_BACKGROUND | FASTRS_FORCE_FALLBACK | FASTRS_APPROX_LT)) | FASTRS_ASYNC;
  const int64_t M = max_label;
  uint64_t sent = 0, recvd = 0;
  int nstat = 0;
  auto keep_status = [&]() {  // the phases share one header: keep each phase's status word
    return cudaMemcpyAsync(stat + nstat++, pw, 4, cudaMemcpyDeviceToDevice, st);
  };
  CUDA_TRY(cudaMemsetAsync(stat, 0, 16 * 4, st), "cudaMemsetAsync");

  // 0: the label slice below the slab (global slice z0 - 1 lands in slot 0 of `below`)
  rc = exchange(cm, halo_plan(bd, 1, Z, 1), bd, labels, below, 1, YX, ncclInt32, st, &sent, &recvd);
  if (rc) return rc;
  // A: K1 + K2 -> packed words of the own slab at slot `cap` of ext
  rc = fastrs_slab_edt_xy(labels, z0 > 0 ? below : nullptr, dims_slab, max_label, pf, ext + halo_cap * YX, dxy, pw,
                          pwb, stream);
  if (rc) return rc;
  CUDA_TRY(keep_status(), "status copy");
  NCCL_TRY(n.AllReduce(dxy, dxy, 1, ncclUint32, ncclMax, cm.c, st), "allreduce max D_xy");
  uint32_t h_dxy = 0;
  CUDA_TRY(cudaMemcpyAsync(&h_dxy, dxy, 4, cudaMemcpyDeviceToHost, st), "D2H");
  CUDA_TRY(cudaStreamSynchronize(st), "sync");
  const int64_t h = halo_edt(h_dxy, Z);
  const bool use_t = transpose;  // N1 by request; N8 needs h <= halo_cap
  if (!use_t && h > halo_cap)
    return err(FASTRS_ENOMEM, "z-pass halo h = %lld slices exceeds halo_cap = %lld (use a larger halo_cap or "
               "FASTRS_SLAB_TRANSPOSE)", (long long)h, (long long)halo_cap);
  uint32_t* d_own = dext + halo_cap * YX;
  if (!use_t) {
    // B (N8): h packed slices per side on the exchange stream while K3 runs on the interior slices
    // (those >= h from both slab faces read no halo slice within their scan), then K3 on the two
    // boundary ranges.  (Interior CTAs may stage halo rows that are still arriving: only rows
    // within sqrt(D_xy) <= h of an element enter its minimum, and terms past that bound never
    // lower it.)
    const int64_t hlo = z0 - h > 0 ? h : z0, hhi = z1 + h < Z ? h : Z - z1;
    const int64_t de[3] = {hlo + nz + hhi, Y, X};
    const uint32_t* pe = ext + (halo_cap - hlo) * YX;
    CUDA_TRY(cudaEventRecord(cm.ev_a, st), "event");
    CUDA_TRY(cudaStreamWaitEvent(cm.xs, cm.ev_a, 0), "event wait");
    rc = exchange(cm, halo_plan(bd, h, Z), bd, ext + halo_cap * YX, ext, halo_cap, YX, ncclUint32, cm.xs, &sent, &recvd);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(cm.ev_x, cm.xs), "event");
    const int64_t i0 = hlo + (z0 > 0 ? h : 0), i1 = hlo + nz - (z1 < Z ? h : 0);  // interior (own-local + hlo)
    int nk = 0;
    if (i1 > i0) {
      rc = fastrs_slab_edt_z(pe, de, i0, i1, z0 - hlo, Z, pf, d_own + (i0 - hlo) * YX, dmx + nk++, pw, pwb, stream);
      if (rc) return rc;
      CUDA_TRY(keep_status(), "status copy");
    }
    CUDA_TRY(cudaStreamWaitEvent(st, cm.ev_x, 0), "event wait");
    const int64_t rng[2][2] = {{hlo, i1 > i0 ? i0 : hlo + nz}, {i1 > i0 ? i1 : hlo + nz, hlo + nz}};
    for (const auto& r : rng)
      if (r[1] > r[0]) {
        rc = fastrs_slab_edt_z(pe, de, r[0], r[1], z0 - hlo, Z, pf, d_own + (r[0] - hlo) * YX, dmx + nk++, pw, pwb,
                               stream);
        if (rc) return rc;
        CUDA_TRY(keep_status(), "status copy");
      }
    for (; nk < 3; ++nk) CUDA_TRY(cudaMemsetAsync(dmx + nk, 0, 4, st), "memset");
  } else {
    // B (N1): z-slabs -> y-slabs, K3 over whole columns, back
    uint32_t* t0 = (uint32_t*)(w + L.t0);
    uint32_t* t1 = (uint32_t*)(w + L.t1);
    const uint32_t* own = ext + halo_cap * YX;
    auto ylo = [&](int s) { return (Y * s) / P; };
    const int64_t y0m = ylo(rank), ym = ylo(rank + 1) - y0m;
    for (int s = 0; s < P; ++s) {  // pack: block s = [nz][Y_s][X]
      const int64_t ys = ylo(s + 1) - ylo(s);
      if (ys > 0)
        CUDA_TRY(cudaMemcpy2DAsync(t0 + nz * ylo(s) * X, ys * X * 4, own + ylo(s) * X, YX * 4, ys * X * 4, nz,
                                   cudaMemcpyDeviceToDevice, st), "pack");
    }
    NCCL_TRY(n.GroupStart(), "ncclGroupStart");
    for (int s = 0; s < P; ++s) {  // block s -> rank s; from rank r its [nz_r][ym][X] at z offset bd[r]
      const int64_t ys = ylo(s + 1) - ylo(s);
      const size_t cs = (size_t)(nz * ys * X), cr = (size_t)((bd[s + 1] - bd[s]) * ym * X);
      if (s == rank) {
        if (cs) CUDA_TRY(cudaMemcpyAsync(t1 + z0 * ym * X, t0 + nz * ylo(s) * X, cs * 4, cudaMemcpyDeviceToDevice, st),
                         "self copy");
        continue;
      }
      if (cs) {
        NCCL_TRY(n.Send(t0 + nz * ylo(s) * X, cs, ncclUint32, s, cm.c, st), "ncclSend");
        sent += cs * 4;
      }
      if (cr) {
        NCCL_TRY(n.Recv(t1 + bd[s] * ym * X, cr, ncclUint32, s, cm.c, st), "ncclRecv");
        recvd += cr * 4;
      }
    }
    NCCL_TRY(n.GroupEnd(), "ncclGroupEnd");
    if (ym > 0) {
      const int64_t dy[3] = {Z, ym, X};
      rc = fastrs_slab_edt_z(t1, dy, 0, Z, 0, Z, pf, t0, dmx, pw, pwb, stream);  // D of the y-slab -> t0
      if (rc) return rc;
      CUDA_TRY(keep_status(), "status copy");
    } else {
      CUDA_TRY(cudaMemsetAsync(dmx, 0, 4, st), "memset");
    }
    CUDA_TRY(cudaMemsetAsync(dmx + 1, 0, 8, st), "memset");
    NCCL_TRY(n.GroupStart(), "ncclGroupStart");
    for (int s = 0; s < P; ++s) {  // back: rank r gets [nz_r][ym][X] of D; from s a [nz][Y_s][X] block
      const int64_t ys = ylo(s + 1) - ylo(s);
      const size_t cs = (size_t)((bd[s + 1] - bd[s]) * ym * X), cr = (size_t)(nz * ys * X);
      if (s == rank) {
        if (cr) CUDA_TRY(cudaMemcpyAsync(t1 + nz * ylo(s) * X, t0 + z0 * ym * X, cr * 4, cudaMemcpyDeviceToDevice, st),
                         "self copy");
        continue;
      }
      if (cs) {
        NCCL_TRY(n.Send(t0 + bd[s] * ym * X, cs, ncclUint32, s, cm.c, st), "ncclSend");
        sent += cs * 4;
      }
      if (cr) {
        NCCL_TRY(n.Recv(t1 + nz * ylo(s) * X, cr, ncclUint32, s, cm.c, st), "ncclRecv");
        recvd += cr * 4;
      }
    }
    NCCL_TRY(n.GroupEnd(), "ncclGroupEnd");
    for (int s = 0; s < P; ++s) {  // unpack into D of the own z-slab
      const int64_t ys = ylo(s + 1) - ylo(s);
      if (ys > 0)
        CUDA_TRY(cudaMemcpy2DAsync(d_own + ylo(s) * X, YX * 4, t1 + nz * ylo(s) * X, ys * X * 4, ys * X * 4, nz,
                                   cudaMemcpyDeviceToDevice, st), "unpack");
    }
  }
  NCCL_TRY(n.AllReduce(dmx, dmx, 3, ncclUint32, ncclMax, cm.c, st), "allreduce max D");
  uint32_t hd[3] = {0, 0, 0};
  CUDA_TRY(cudaMemcpyAsync(hd, dmx, 12, cudaMemcpyDeviceToHost, st), "D2H");
  CUDA_TRY(cudaStreamSynchronize(st), "sync");
  const uint32_t h_dmax = hd[0] > hd[1] ? (hd[0] > hd[2] ? hd[0] : hd[2]) : (hd[1] > hd[2] ? hd[1] : hd[2]);
  const int64_t H = halo_lt(h_dmax);
  if (H > halo_cap)
    return err(FASTRS_ENOMEM, "dilation halo H = %lld slices exceeds halo_cap = %lld", (long long)H,
               (long long)halo_cap);
  // C: the dilation halo.  The extended slab covers the global slices [z0 - Hlo, z1 + Hhi).
  const int64_t Hlo = z0 - H > 0 ? H : z0, Hhi = z1 + H < Z ? H : Z - z1;
  const int64_t dc[3] = {Hlo + nz + Hhi, Y, X};
  uint64_t* vol = part;
  uint64_t* nsh = part + M;
  uint64_t* sum = part + 2 * M;
  uint64_t* sums = part + 4 * M;
  uint32_t* mx = (uint32_t*)(part + 6 * M);
  uint32_t* dwin = dext + (halo_cap - Hlo) * YX;
  if (dense) {
    // dense (FASTRS_SLAB_DENSE_HALO): H slices of D per side, K4 on the whole extended slab
    rc = exchange(cm, halo_plan(bd, H, Z), bd, d_own, dext, halo_cap, YX, ncclUint32, st, &sent, &recvd);
    if (rc) return rc;
    rc = fastrs_slab_reduce(labels, dwin, dc, Hlo, Hlo + nz, Z, h_dmax, max_label, pf, vol, nsh, sum, sums, mx, pw, pwb,
                            stream);
    if (rc) return rc;
    CUDA_TRY(keep_status(), "status copy");
  } else {
    // kept-centre halo (N4, default): 3 slices of D per side (K4's stencil), K4 on the own tile
    // layers, then the K4 outputs (records + kept centres) of the tile layers within H slices of
    // each neighbour's slab instead of its D; K5 on the own tiles
    rc = exchange(cm, halo_plan(bd, 3, Z), bd, d_own, dext, halo_cap, YX, ncclUint32, st, &sent, &recvd);
    if (rc) return rc;
    rc = fastrs_slab_prune(dwin, dc, Hlo, Hlo + nz, pf, pw, pwb, stream);
    if (rc) return rc;
    CUDA_TRY(keep_status(), "status copy");
    const std::vector<Xfer> plan = halo_plan(bd, H, Z);
    const int64_t tpl = ((Y + kTZ3 - 1) / kTZ3) * ((X + 31) / 32);
    auto win0 = [&](int r) {  // global slice of rank r's extended-slab slot 0
      return bd[r] - (bd[r] - H > 0 ? H : bd[r]);
    };
    uint32_t* srec = (uint32_t*)(w + L.srec);
    uint2* sent_e = (uint2*)(w + L.sent);
    uint32_t* rrec = (uint32_t*)(w + L.rrec);
    uint2* rent_e = (uint2*)(w + L.rent);
    uint64_t* cnt = (uint64_t*)(w + L.cnt);  // [0, 4P): entries per send transfer, [4P, 8P): per receive
    struct Part {
      int peer;
      int64_t la, lb, tile_off;  // own-window tile layers [la, lb), offset in the record / entry buffers
    };
    std::vector<Part> sends, recvs;
    int64_t soff = 0, roff = 0;
    for (const Xfer& x : plan) {
      if (x.src == rank) {
        const int64_t la = (x.a - win0(rank)) / kTZ3, lb = (x.b - win0(rank) + kTZ3 - 1) / kTZ3;
        sends.push_back({x.dst, la, lb, soff});
        soff += (lb - la) * tpl;
      }
      if (x.dst == rank) {
        const int64_t la = (x.a - win0(rank)) / kTZ3, lb = (x.b - win0(rank) + kTZ3 - 1) / kTZ3;
        recvs.push_back({x.src, la, lb, roff});
        roff += (lb - la) * tpl;
      }
    }
    if (soff > L.send_tiles || roff > L.recv_tiles || (int)(sends.size() + recvs.size()) > 4 * P)
      return err(FASTRS_ENOMEM, "kept-centre halo buffers too small (halo H = %lld)", (long long)H);
    for (size_t k = 0; k < sends.size(); ++k) {
      rc = fastrs_slab_pack_tiles(pw, dc, sends[k].la, sends[k].lb, srec + sends[k].tile_off * FASTRS_TILE_RECORD_WORDS,
                                  sent_e + sends[k].tile_off * kTileVol, cnt + k, stream);
      if (rc) return rc;
    }
    NCCL_TRY(n.GroupStart(), "ncclGroupStart");  // round 1: the fixed-size tile records
    for (const Part& q : sends) {
      const size_t c = (size_t)((q.lb - q.la) * tpl * FASTRS_TILE_RECORD_WORDS);
      NCCL_TRY(n.Send(srec + q.tile_off * FASTRS_TILE_RECORD_WORDS, c, ncclUint32, q.peer, cm.c, st), "ncclSend");
      sent += c * 4;
    }
    for (const Part& q : recvs) {
      const size_t c = (size_t)((q.lb - q.la) * tpl * FASTRS_TILE_RECORD_WORDS);
      NCCL_TRY(n.Recv(rrec + q.tile_off * FASTRS_TILE_RECORD_WORDS, c, ncclUint32, q.peer, cm.c, st), "ncclRecv");
      recvd += c * 4;
    }
    NCCL_TRY(n.GroupEnd(), "ncclGroupEnd");
    for (size_t k = 0; k < recvs.size(); ++k)  // entries announced by the received records
      k_count_entries<<<1, 256, 0, st>>>(rrec + recvs[k].tile_off * FASTRS_TILE_RECORD_WORDS, (recvs[k].lb - recvs[k].la) * tpl,
                                         cnt + 4 * P + k);
    std::vector<uint64_t> hc(8 * P, 0);
    CUDA_TRY(cudaMemcpyAsync(hc.data(), cnt, 8 * P * sizeof(uint64_t), cudaMemcpyDeviceToHost, st), "D2H");
    CUDA_TRY(cudaStreamSynchronize(st), "sync");
    NCCL_TRY(n.GroupStart(), "ncclGroupStart");  // round 2: the kept centres (uint2 = 2 u32)
    for (size_t k = 0; k < sends.size(); ++k)
      if (hc[k]) {
        NCCL_TRY(n.Send(sent_e + sends[k].tile_off * kTileVol, (size_t)hc[k] * 2, ncclUint32, sends[k].peer, cm.c, st),
                 "ncclSend");
        sent += hc[k] * 8;
      }
    for (size_t k = 0; k < recvs.size(); ++k)
      if (hc[4 * P + k]) {
        NCCL_TRY(n.Recv(rent_e + recvs[k].tile_off * kTileVol, (size_t)hc[4 * P + k] * 2, ncclUint32, recvs[k].peer,
                        cm.c, st),
                 "ncclRecv");
        recvd += hc[4 * P + k] * 8;
      }
    NCCL_TRY(n.GroupEnd(), "ncclGroupEnd");
    for (const Part& q : recvs) {
      rc = fastrs_slab_unpack_tiles(pw, dc, q.la, q.lb, rrec + q.tile_off * FASTRS_TILE_RECORD_WORDS, rent_e + q.tile_off * kTileVol, stream);
      if (rc) return rc;
    }
    rc = fastrs_slab_dilate(labels, dwin, dc, Hlo, Hlo + nz, Z, h_dmax, max_label, pf, vol, nsh, sum, sums, mx, pw, pwb,
                            stream);
    if (rc) return rc;
    CUDA_TRY(keep_status(), "status copy");
  }
  NCCL_TRY(n.GroupStart(), "ncclGroupStart");
  NCCL_TRY(n.AllReduce(part, part, (size_t)(6 * M), ncclUint64, ncclSum, cm.c, st), "allreduce partial sums");
  NCCL_TRY(n.AllReduce(mx, mx, (size_t)M, ncclUint32, ncclMax, cm.c, st), "allreduce max LT^2");
  NCCL_TRY(n.GroupEnd(), "ncclGroupEnd");
  // D: closed forms (every rank holds the results of all labels)
  rc = fastrs_metrics_from_partials(vol, nsh, sum, sums, mx, M, 3, Z * YX, h_dmax, sphericity, roundness, stats, pw,
                                    pwb, stream);
  if (rc) return rc;
  CUDA_TRY(keep_status(), "status copy");
  k_status_flags<<<1, 1, 0, st>>>(stat, nstat, sflags);
  NCCL_TRY(n.AllReduce(sflags, sflags, 4, ncclUint32, ncclSum, cm.c, st), "allreduce status");
  uint32_t hf[4];
  CUDA_TRY(cudaMemcpyAsync(hf, sflags, 16, cudaMemcpyDeviceToHost, st), "D2H");
  CUDA_TRY(cudaStreamSynchronize(st), "sync");
  if (info) {
    info->mode = use_t ? 1 : 0;
    info->h = use_t ? 0 : h;
    info->H = H;
    info->dmax = h_dmax;
    info->dxy_max = h_dxy;
    info->bytes_sent = sent;
    info->bytes_received = recvd;
  }
  if (hf[0]) return err(FASTRS_EINVAL, "a label is < 0 or > max_label");
  if (hf[1]) return err(FASTRS_ENOSITE, "an object element has no site");
  if (hf[2] || hf[3]) return err(FASTRS_EINTERNAL, "device invariant violated");
  return FASTRS_OK;
}

}  // extern "C"
