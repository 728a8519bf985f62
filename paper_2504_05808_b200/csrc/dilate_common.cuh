// Shared by the dilation kernels (lt.cu fallback, dilate.cu default): row epilogue.
#pragma once
#include "common.cuh"

namespace fastrs {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr uint32_t kFxLut = 65536;  // entries of the fixed-point sqrt table
constexpr uint32_t kU16Max = 65535u;

// Shell + per-label reductions + optional LT writes for one 32-wide row held in a warp
// (lane = x), given each lane's LT^2 `c`, label L and squared distance d (L = 0 outside the
// grid).  Returns 1 if the invariant LT^2 >= D failed.
// FAST: reductions only, with the fixed-point table (no LT outputs): the per-element option
// tests fold away.
template <bool FAST = false>
static __device__ __forceinline__ uint32_t row_epilogue_v(uint32_t c, int32_t L, uint32_t d, int lane, int64_t gi,
                                                   int64_t b, const Accum& acc, int do_reduce, double scale,
                                                   uint32_t* __restrict__ lt2_out, float* __restrict__ lt_out,
                                                   const unsigned long long* __restrict__ fxlut = nullptr) {
  uint32_t bad = 0;
  bool shell = false;
  unsigned long long fx = 0;
  if (L != 0) {
    if (c < d) bad = 1;
    shell = d == 1;
    // fixed-point sqrt(LT^2) * 2^s: from the per-call table when LT^2 < 65536 (bit-identical:
    // the table holds the same correctly rounded values)
    if ((FAST || fxlut) && c < kFxLut) {
      fx = __ldg(fxlut + c);
    } else {
      fx = (unsigned long long)__double2ull_rn(sqrt((double)c) * scale);
    }
    if (!FAST && lt2_out) lt2_out[gi] = c;
    if (!FAST && lt_out) lt_out[gi] = (float)sqrt((double)c);
  }
  if (FAST || do_reduce) {
    if ((uint32_t)L > (uint32_t)acc.max_label) L = 0;  // also catches L < 0
    uint32_t act = __ballot_sync(kFull, L != 0);
    while (act) {
      const int leader = __ffs(act) - 1;
      const int32_t key = __shfl_sync(kFull, L, leader);
      const uint32_t grp = __ballot_sync(kFull, L == key);
      const bool in = (grp >> lane) & 1u;
      const unsigned long long t1 = in ? fx : 0ull, t2 = (in && shell) ? fx : 0ull;
      const uint32_t h1 = __reduce_add_sync(kFull, (uint32_t)(t1 >> 24));
      const uint32_t l1 = __reduce_add_sync(kFull, (uint32_t)(t1 & 0xFFFFFFull));
      const uint32_t h2 = __reduce_add_sync(kFull, (uint32_t)(t2 >> 24));
      const uint32_t l2 = __reduce_add_sync(kFull, (uint32_t)(t2 & 0xFFFFFFull));
      const uint32_t mx = __reduce_max_sync(kFull, in ? c : 0u);
      const uint32_t nsh = __popc(__ballot_sync(kFull, in && shell));
      if (lane == leader) {
        const int64_t id = b * acc.max_label + (key - 1);
        atomicAdd(acc.vol + id, (unsigned long long)__popc(grp));
        if (nsh) atomicAdd(acc.nshell + id, (unsigned long long)nsh);
        atomicAdd(acc.sum + id, ((unsigned long long)h1 << 24) + l1);
        if (nsh) atomicAdd(acc.sumshell + id, ((unsigned long long)h2 << 24) + l2);
        atomicMax(acc.maxlt2 + id, mx);
      }
      act &= ~grp;
    }
  }
  return bad;
}

cudaError_t dilate_cover_setup();


}  // namespace fastrs
