// Shared by the dilation kernels (lt.cu fallback, dilate.cu default): row epilogue.
#pragma once
#include "common.cuh"

namespace fastrs {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr uint32_t kU16Max = 65535u;

// fixed-point LT term of the sums: round(sqrt(c) * 2^32) (correctly rounded sqrt in double, the
// same value the per-device table holds for c < kFxLut)
static __device__ __forceinline__ unsigned long long fx_term(uint32_t c, const unsigned long long* __restrict__ fxlut) {
  return c < kFxLut ? __ldg(fxlut + c) : (unsigned long long)__double2ull_rn(sqrt((double)c) * kFxScale);
}

// Warp-aggregated accumulation: every lane holds a (label L, count, shell count, value) record
// (L <= 0: none); records of the same label are summed in the warp and the group's first lane
// adds them to the per-label accumulators: vol += cnt, n_shell += scnt, sum += cnt * fx(v),
// sum_shell += scnt * fx(v), max_lt2 = max(max_lt2, v).  The u64 sums of up to 32 records are
// formed from 24-bit pieces and split into the hi / lo accumulator words; the pieces cannot
// overflow while every record term cnt * fx(v) < 2^51 (the fused paint: v < 2^16 so fx < 2^40,
// cnt <= 2048; the per-element epilogue: cnt = 1, fx < 2^47).
static __device__ __forceinline__ void accumulate_records(int32_t L, uint32_t cnt, uint32_t scnt, uint32_t v,
                                                          int lane, int64_t b, const Accum& acc,
                                                          const unsigned long long* __restrict__ fxlut) {
  if ((uint32_t)L > (uint32_t)acc.max_label) L = 0;  // also catches L < 0
  uint32_t act = __ballot_sync(kFull, L != 0);
  if (!act) return;
  const unsigned long long fx = L != 0 ? fx_term(v, fxlut) : 0ull;
  while (act) {
    const int leader = __ffs(act) - 1;
    const int32_t key = __shfl_sync(kFull, L, leader);
    const uint32_t grp = __ballot_sync(kFull, L == key);
    const bool in = (grp >> lane) & 1u;
    const unsigned long long t1 = in ? fx * cnt : 0ull, t2 = in ? fx * scnt : 0ull;
    const uint32_t h1 = __reduce_add_sync(kFull, (uint32_t)(t1 >> 24));
    const uint32_t l1 = __reduce_add_sync(kFull, (uint32_t)(t1 & 0xFFFFFFull));
    const uint32_t h2 = __reduce_add_sync(kFull, (uint32_t)(t2 >> 24));
    const uint32_t l2 = __reduce_add_sync(kFull, (uint32_t)(t2 & 0xFFFFFFull));
    const uint32_t nv = __reduce_add_sync(kFull, in ? cnt : 0u);
    const uint32_t ns = __reduce_add_sync(kFull, in ? scnt : 0u);
    const uint32_t mx = __reduce_max_sync(kFull, in ? v : 0u);
    if (lane == leader) {
      const int64_t id = b * acc.max_label + (key - 1);
      const unsigned long long T1 = ((unsigned long long)h1 << 24) + l1, T2 = ((unsigned long long)h2 << 24) + l2;
      atomicAdd(acc.vol + id, (unsigned long long)nv);
      atomicAdd(acc.sum + id, T1 >> 32);
      atomicAdd(acc.sum + acc.M + id, T1 & 0xFFFFFFFFull);
      if (ns) {
        atomicAdd(acc.nshell + id, (unsigned long long)ns);
        atomicAdd(acc.sumshell + id, T2 >> 32);
        atomicAdd(acc.sumshell + acc.M + id, T2 & 0xFFFFFFFFull);
      }
      atomicMax(acc.maxlt2 + id, mx);
    }
    act &= ~grp;
  }
}

// Shell + per-label reductions + optional LT writes for one 32-wide row held in a warp
// (lane = x), given each lane's LT^2 `c`, label L and squared distance d (L = 0 outside the
// grid).  Returns 1 if the invariant LT^2 >= D failed.
static __device__ __forceinline__ uint32_t row_epilogue_v(uint32_t c, int32_t L, uint32_t d, int lane, int64_t gi,
                                                          int64_t b, const Accum& acc, int do_reduce,
                                                          uint32_t* __restrict__ lt2_out, float* __restrict__ lt_out,
                                                          const unsigned long long* __restrict__ fxlut) {
  uint32_t bad = 0;
  bool shell = false;
  if (L != 0) {
    if (c < d) bad = 1;
    shell = d == 1;
    if (lt2_out) lt2_out[gi] = c;
    if (lt_out) lt_out[gi] = (float)sqrt((double)c);
  }
  if (do_reduce) accumulate_records(L, 1u, shell ? 1u : 0u, c, lane, b, acc, fxlut);
  return bad;
}

cudaError_t dilate_cover_setup();


}  // namespace fastrs
