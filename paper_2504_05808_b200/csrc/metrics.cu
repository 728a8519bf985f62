// K6: per-object closed forms, one thread per (batch item, label).
//   a = mean LT, V/A = count, R_max = sqrt(max LT^2)
//   (PAPER.md:142), r_bar = mean shell LT; sphericity by Eqs. 1,6-8 (3D) or
//   Eqs. 2,9-11 (2D); roundness = r_bar / R_max.
#include <math.h>

#include "common.cuh"
#include "fastrs.h"
#include "formulas.cuh"

namespace fastrs {
namespace {

__global__ void k_metrics(Accum acc, Outputs o, int ndim, WsHeader* __restrict__ hdr) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) hdr->scale_log2 = 32;
  if (i >= acc.M) return;
  const unsigned long long V = acc.vol[i];
  const unsigned long long nsh = acc.nshell[i];
  const uint32_t m2 = acc.maxlt2[i];
  double sph = nan(""), rnd = nan(""), mean = nan(""), rmax = nan(""), smean = nan(""), cb = nan("");
  if (V > 0) {
    // sums = hi * 2^32 + lo in units of 2^-32 (common.cuh "Accum")
    const unsigned long long sh = acc.sum[i], sl = acc.sum[acc.M + i];
    const unsigned long long ssh = acc.sumshell[i], ssl = acc.sumshell[acc.M + i];
    const double inv = 1.0 / kFxScale;
    mean = ((double)sh + (double)sl * inv) / (double)V;
    rmax = sqrt((double)m2);
    const double sshell = (double)ssh + (double)ssl * inv;  // sum of shell LT radii
    smean = nsh ? sshell / (double)nsh : nan("");
    if (ndim == 3) {
      sph = sphericity_3d((double)V, mean);
      cb = c_axis_3d((double)V, mean);
    } else {
      sph = sphericity_2d((double)V, mean);
      cb = b_axis_2d((double)V, mean);
    }
    // roundness r_bar / R_max evaluated in the fixed-point system the shell terms were
    // summed in: every shell term is <= fx(R_max) (monotone rounding), so the invariant
    // r_bar <= R_max is checked exactly in (128-bit) integers, and R = 1 exactly
    // when every shell element carries the maximum.
    const unsigned long long fxmax = __double2ull_rn(rmax * kFxScale);
    const unsigned __int128 ss = ((unsigned __int128)ssh << 32) + (unsigned __int128)ssl;
    const unsigned __int128 bound = (unsigned __int128)nsh * fxmax;
    if (nsh == 0 || ss > bound) atomicOr(&hdr->status, kStShell);
    rnd = (ss == bound) ? 1.0 : (sshell / (double)nsh) / rmax;
  }
  if (o.sphericity) o.sphericity[i] = sph;
  if (o.roundness) o.roundness[i] = rnd;
  if (o.volume) o.volume[i] = (int64_t)V;
  if (o.n_shell) o.n_shell[i] = (int64_t)nsh;
  if (o.max_lt2) o.max_lt2[i] = m2;
  if (o.mean_lt) o.mean_lt[i] = mean;
  if (o.max_lt) o.max_lt[i] = rmax;
  if (o.shell_mean_lt) o.shell_mean_lt[i] = smean;
  if (o.axis_a) o.axis_a[i] = mean;
  if (o.axis_cb) o.axis_cb[i] = cb;
}

}  // namespace

void launch_metrics(const Accum& acc, const Geom& g, const Outputs& o, WsHeader* hdr, cudaStream_t st) {
  const int64_t blocks = (acc.M + 255) / 256;
  k_metrics<<<(unsigned)(blocks > 0 ? blocks : 1), 256, 0, st>>>(acc, o, g.ndim, hdr);
}

}  // namespace fastrs

extern "C" {
double fastrs_spheroid_area(double a, double c) { return fastrs::spheroid_area(a, c); }
double fastrs_ramanujan_perimeter(double a, double b) { return fastrs::ramanujan_perimeter(a, b); }
double fastrs_sphericity_3d(double V, double mean_lt) { return fastrs::sphericity_3d(V, mean_lt); }
double fastrs_sphericity_2d(double A, double mean_lt) { return fastrs::sphericity_2d(A, mean_lt); }
}
