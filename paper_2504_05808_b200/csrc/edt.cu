// Exact label-aware squared EDT as three separable passes.
//
// D(p) = min over sites s of |p - s|^2, sites = elements with another label (plus the
// virtual border layer with FASTRS_BORDER_BACKGROUND): the substrate of local thickness
// (§4, "exact squared-distance computation via separable per-axis
// passes").  The passes reduce the global label-aware problem to per-RUN problems: along
// each axis an element only interacts with the same-label run it lies in, because every
// element beyond a run end is dominated by the run end's neighbour, which is itself a site
// at distance 0 in the partial field.
//
//   K1 edt_x : warp per row.  Two warp sweeps with ballot/ffs find run starts and ends;
//              g = (distance to the nearest run end's neighbour)^2.  Fused: label
//              validation (a1) and the y/z run-start flags packed into bits 31/30 (S2), so
//              later passes never re-read labels.
//   K2/K3    : column passes along y / z.  A CTA stages a [256 + 2*32][32] column tile of
//              packed words in shared memory (coalesced 128-byte rows) and each thread runs
//              the exact windowed scan  best = min(best, g(p +- dq) + dq^2)  until dq^2 >=
//              best or a run end (a site at distance dq) is met; reads outside the staged
//              window fall back to global (L2).  The final pass emits D, Dmax, n_fg and
//              flags elements with no site (ENOSITE).
#include "common.cuh"

namespace fastrs {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

template <int U>
__global__ void __launch_bounds__(256) k_edt_x(const int32_t* __restrict__ lab,
                                               const int32_t* __restrict__ below, uint32_t* __restrict__ out,
                                               int64_t nrows, int X, int64_t Y, int64_t Z,
                                               int32_t max_label, int border, int is3d,
                                               WsHeader* __restrict__ hdr) {
  extern __shared__ uint16_t s_end[];
  const int warps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * warps + warp;
  if (row >= nrows) return;
  uint16_t* ends = s_end + (size_t)warp * X;
  const int64_t y = row % Y;
  const int64_t z = (row / Y) % Z;
  const int32_t* L = lab + row * X;
  const int32_t* Ly = y > 0 ? L - X : nullptr;
  // z-1 neighbour: the previous slice, or (slab path) the caller's slice just below the slab
  const int32_t* Lz = is3d ? (z > 0 ? L - X * Y : (below ? below + y * X : nullptr)) : nullptr;
  uint32_t* O = out + row * X;
  const int nchunk = (X + 31) >> 5;

  // sweep 1 (right to left): end of the run containing x
  int carry_end = X - 1;
  int32_t right_next = 0;
#pragma unroll U
  for (int c = nchunk - 1; c >= 0; --c) {
    const int x = (c << 5) + lane;
    const int32_t v = x < X ? __ldg(L + x) : 0;
    int32_t r = __shfl_down_sync(kFull, v, 1);
    if (lane == 31) r = right_next;
    const bool is_end = x < X && (x == X - 1 || v != r);
    const uint32_t m = __ballot_sync(kFull, is_end);
    const uint32_t ge = m & (kFull << lane);
    const int e = ge ? (c << 5) + __ffs(ge) - 1 : carry_end;
    if (x < X) ends[x] = (uint16_t)e;
    if (m) carry_end = (c << 5) + __ffs(m) - 1;
    right_next = __shfl_sync(kFull, v, 0);
  }

  // sweep 2 (left to right): start of the run, distances, flags
  int carry_start = 0;
  int32_t left_prev = 0;
  uint32_t bad = 0;
#pragma unroll U
  for (int c = 0; c < nchunk; ++c) {
    const int x = (c << 5) + lane;
    const int32_t v = x < X ? __ldg(L + x) : 0;
    int32_t l = __shfl_up_sync(kFull, v, 1);
    if (lane == 0) l = left_prev;
    const bool is_start = x < X && (x == 0 || v != l);
    const uint32_t m = __ballot_sync(kFull, is_start);
    const uint32_t le = m & (kFull >> (31 - lane));
    const int s = le ? (c << 5) + 31 - __clz(le) : carry_start;
    if (m) carry_start = (c << 5) + 31 - __clz(m);
    left_prev = __shfl_sync(kFull, v, 31);
    if (x < X) {
      uint32_t g = 0;
      if (v != 0) {
        if (v < 0 || v > max_label) bad = 1;
        const int e = ends[x];
        const uint32_t dl = (s > 0 || border) ? (uint32_t)(x - s + 1) : kFull;
        const uint32_t dr = (e < X - 1 || border) ? (uint32_t)(e + 1 - x) : kFull;
        const uint32_t d = min(dl, dr);
        g = d == kFull ? kInf : d * d;
      }
      uint32_t bits = 0;
      if (!Ly || __ldg(Ly + x) != v) bits |= kBitY;
      if (!Lz || __ldg(Lz + x) != v) bits |= kBitZ;
      O[x] = g | bits;
    }
  }
  if (__any_sync(kFull, bad) && lane == 0) atomicOr(&hdr->status, kStBadLabel);
}

constexpr int kColS = 256;  // positions per CTA
constexpr int kColH = 48;   // staged halo on each side
constexpr int kColRows = kColS + 2 * kColH;
constexpr int kColWarps = 8;
constexpr int kScanU = 4;  // rows per iteration of the hoisted scan loops (C4 y/z ms: 1: 7.33/6.19, 2: 6.45/5.55, 4: 6.20/5.50, 6: 6.27/5.61, 8: 6.34/5.80)

// Slow path of the column scan for an element whose window leaves the staged rows: the same
// exact scan, reading beyond the window from global memory (L2).
__device__ __noinline__ uint32_t scan_global(const uint32_t* __restrict__ in, int64_t base, int64_t astride, int64_t p,
                                             int64_t L, int64_t lo, int64_t hi, const uint32_t* tile, int lane,
                                             uint32_t v, uint32_t chbit, int border, int64_t gofs, int64_t Lg) {
  uint32_t best = v & kMask;
  {
    uint32_t dq = 1, dq2 = 1;
    int64_t q = p + 1;
    while (dq2 < best) {
      if (q >= L) {  // end of the staged axis: the grid end (slab path: h^2 >= D guarantees it)
        if (border && gofs + q >= Lg) best = min(best, dq2);
        break;
      }
      const uint32_t w = q < hi ? tile[(q - lo) * 32 + lane] : __ldg(in + base + q * astride);
      if (w & chbit) {
        best = min(best, dq2);
        break;
      }
      best = min(best, (w & kMask) + dq2);
      dq2 += 2 * dq + 1;
      ++dq;
      ++q;
    }
  }
  {
    uint32_t dq = 1, dq2 = 1, chk = v & chbit;
    int64_t q = p - 1;
    while (dq2 < best) {
      if (chk) {
        if (gofs + q >= 0 || border) best = min(best, dq2);
        break;
      }
      const uint32_t w = q >= lo ? tile[(q - lo) * 32 + lane] : __ldg(in + base + q * astride);
      best = min(best, (w & kMask) + dq2);
      chk = w & chbit;
      dq2 += 2 * dq + 1;
      ++dq;
      --q;
    }
  }
  return best;
}

template <bool FINAL>
__global__ void __launch_bounds__(256) k_edt_col(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                 int64_t L, int64_t astride, int X, int nxb, int nseg,
                                                 int64_t n_inner, int64_t inner_mult, int64_t outer_mult,
                                                 uint32_t chbit, int border, int64_t p_lo, int64_t p_hi,
                                                 int64_t gofs, int64_t Lg, WsHeader* __restrict__ hdr) {
  __shared__ uint32_t tile[kColRows * 32];
  int64_t bid = blockIdx.x;
  const int xb = (int)(bid % nxb);
  bid /= nxb;
  const int seg = (int)(bid % nseg);
  const int64_t outer = bid / nseg;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t base = (outer / n_inner) * outer_mult + (outer % n_inner) * inner_mult + (int64_t)xb * 32 + lane;
  const bool xin = xb * 32 + lane < X;
  const int64_t s0 = p_lo + (int64_t)seg * kColS;
  const int64_t lo = s0 - kColH > 0 ? s0 - kColH : 0;
  const int64_t hi = s0 + kColS + kColH < L ? s0 + kColS + kColH : L;
  for (int64_t r = lo + warp; r < hi; r += kColWarps)
    tile[(r - lo) * 32 + lane] = xin ? __ldg(in + base + r * astride) : 0u;
  __syncthreads();

  uint32_t dmax = 0, nfg = 0, nosite = 0;
  const int64_t pend = s0 + kColS < p_hi ? s0 + kColS : p_hi;
  for (int64_t p = s0 + warp; p < pend; p += kColWarps) {
    const uint32_t v = tile[(p - lo) * 32 + lane];
    const uint32_t g = v & kMask;
    uint32_t res = FINAL ? 0u : v;
    if (xin && g != 0) {
      uint32_t best = g;
      // Fast path: pure shared-memory scan in 32-bit indices.  up side: rows p+1, p+2, ... until a
      // run end (the element there is a site) or dq^2 >= best; leaving the staged rows before
      // that hands the element to the slow path below.
      const int i = (int)(p - lo), nt = (int)(hi - lo);
      bool slow = false;
      // dq^2 < best <= g bounds the scan: when isqrt(g-1) rows exist on a side, that side's loop
      // needs no window-end check (the common case)
      const int reach = (int)sqrtf((float)(g - 1)) + 1;  // >= isqrt(g - 1)
      {
        uint32_t dq2 = 1, inc = 3;
        const uint32_t* w_ptr = tile + (i + 1) * 32 + lane;
        if (reach + kScanU - 1 <= nt - 1 - i) {
          // kScanU rows per iteration (the staged rows suffice): a row's term is an exact
          // candidate even when an earlier one made dq^2 >= best
          while (dq2 < best) {
            uint32_t w[kScanU];
#pragma unroll
            for (int u = 0; u < kScanU; ++u) w[u] = w_ptr[32 * u];
            bool stop = false;
#pragma unroll
            for (int u = 0; u < kScanU; ++u) {
              if (w[u] & chbit) {
                best = min(best, dq2);
                stop = true;
                break;
              }
              best = min(best, (w[u] & kMask) + dq2);
              dq2 += inc;
              inc += 2;
            }
            if (stop) break;
            w_ptr += 32 * kScanU;
          }
        } else {
          const uint32_t* w_end = tile + nt * 32 + lane;
          while (dq2 < best) {
            if (w_ptr >= w_end) {
              if (hi < L) slow = true;  // more rows exist beyond the staged window
              else if (border && gofs + L >= Lg) best = min(best, dq2);  // the grid end
              break;
            }
            const uint32_t w = *w_ptr;
            if (w & chbit) {
              best = min(best, dq2);
              break;
            }
            best = min(best, (w & kMask) + dq2);
            dq2 += inc;
            inc += 2;
            w_ptr += 32;
          }
        }
      }
      // down side: rows p-1, p-2, ...; element p-dq lies outside the run iff p-dq+1 starts it
      {
        uint32_t dq2 = 1, inc = 3, chk = v & chbit;
        const uint32_t* w_ptr = tile + (i - 1) * 32 + lane;
        if (reach + kScanU - 1 <= i) {
          while (dq2 < best) {
            if (chk) {  // the element at p-dq is inside the staged window: a real site
              best = min(best, dq2);
              break;
            }
            uint32_t w[kScanU];
#pragma unroll
            for (int u = 0; u < kScanU; ++u) w[u] = w_ptr[-32 * u];
            bool stop = false;
#pragma unroll
            for (int u = 0; u < kScanU; ++u) {
              best = min(best, (w[u] & kMask) + dq2);
              dq2 += inc;
              inc += 2;
              chk = w[u] & chbit;
              if (u + 1 < kScanU && chk) {  // p-dq (now) lies below the run start: a site
                best = min(best, dq2);
                stop = true;
                break;
              }
            }
            if (stop) break;
            w_ptr -= 32 * kScanU;
          }
        } else {
          int r = i - 1;
          while (dq2 < best) {
            if (chk) {
              if (gofs + lo + r >= 0 || border) best = min(best, dq2);
              break;
            }
            if (r < 0) {  // lo > 0 here (element 0 of the axis always starts a run)
              slow = true;
              break;
            }
            const uint32_t w = tile[r * 32 + lane];
            best = min(best, (w & kMask) + dq2);
            chk = w & chbit;
            dq2 += inc;
            inc += 2;
            --r;
          }
        }
      }
      if (slow) best = scan_global(in, base, astride, p, L, lo, hi, tile, lane, v, chbit, border, gofs, Lg);
      dmax = max(dmax, best);
      if (FINAL) {
        res = best;
        nfg += 1;
        nosite |= best >= kInf;
      } else {
        res = best | (v & (kBitY | kBitZ));
      }
    }
    if (xin) out[base + (p - p_lo) * astride] = res;
  }
  if (!FINAL) {  // the max partial distance bounds the next pass's window (slab z halo)
    dmax = __reduce_max_sync(kFull, dmax);
    if (lane == 0 && dmax) atomicMax(&hdr->dxymax, dmax);
  } else {
    dmax = __reduce_max_sync(kFull, dmax);
    nfg = __reduce_add_sync(kFull, nfg);
    nosite = __any_sync(kFull, nosite);
    if (lane == 0) {
      if (dmax) atomicMax(&hdr->dmax, dmax);
      if (nfg) atomicAdd(&hdr->n_fg, (unsigned long long)nfg);
      if (nosite) atomicOr(&hdr->status, kStNoSite);
    }
  }
}

}  // namespace

void launch_edt_x(const int32_t* labels, const int32_t* labels_below, uint32_t* out, const Geom& g,
                  int32_t max_label, bool border, WsHeader* hdr, cudaStream_t st) {
  const int64_t nrows = g.B * g.Z * g.Y;
  int warps = (int)(49152 / (2 * g.X));
  warps = warps < 1 ? 1 : (warps > 8 ? 8 : warps);
  const size_t smem = (size_t)warps * g.X * sizeof(uint16_t);
  const int64_t blocks = (nrows + warps - 1) / warps;
  // sweep unroll 2: measured on C4 4.13 ms vs 4.46 (4), 4.35 (8), 4.26 (16)
  k_edt_x<2><<<(unsigned)blocks, warps * 32, smem, st>>>(labels, labels_below, out, nrows, (int)g.X, g.Y, g.Z, max_label,
                                                         border ? 1 : 0, g.ndim == 3 ? 1 : 0, hdr);
}

// axis 1 = y, axis 2 = z.
void launch_edt_col(const uint32_t* in, uint32_t* out, const Geom& g, int axis, bool final_pass, bool border,
                    WsHeader* hdr, cudaStream_t st, int64_t p_lo, int64_t p_hi, int64_t gofs, int64_t Lg) {
  int64_t L, astride, n_outer, n_inner, inner_mult, outer_mult;
  uint32_t chbit;
  if (axis == 1) {
    L = g.Y;
    astride = g.X;
    n_outer = g.B * g.Z;
    n_inner = 1;
    inner_mult = 0;
    outer_mult = g.Y * g.X;
    chbit = kBitY;
  } else {
    L = g.Z;
    astride = g.Y * g.X;
    n_outer = g.B * g.Y;
    n_inner = g.Y;
    inner_mult = g.X;
    outer_mult = g.Z * g.Y * g.X;
    chbit = kBitZ;
  }
  if (p_hi < 0) p_hi = L;
  if (Lg < 0) Lg = L;
  const int nxb = (int)((g.X + 31) / 32);
  const int nseg = (int)((p_hi - p_lo + kColS - 1) / kColS);
  if (nseg <= 0) return;
  const int64_t blocks = (int64_t)nxb * nseg * n_outer;
  if (final_pass)
    k_edt_col<true><<<(unsigned)blocks, kColWarps * 32, 0, st>>>(in, out, L, astride, (int)g.X, nxb, nseg, n_inner,
                                                                  inner_mult, outer_mult, chbit, border ? 1 : 0, p_lo, p_hi, gofs, Lg, hdr);
  else
    k_edt_col<false><<<(unsigned)blocks, kColWarps * 32, 0, st>>>(in, out, L, astride, (int)g.X, nxb, nseg, n_inner,
                                                                   inner_mult, outer_mult, chbit, border ? 1 : 0, p_lo, p_hi, gofs, Lg, hdr);
}

}  // namespace fastrs
