// Lower end of the Chebyshev interval: lambda_min(S) >= -alpha lambda_max(Z)
// for S = X_k - alpha Z_k with X_k PSD.  The iteration kernel derives the
// bound from the Gershgorin radius of Z (its adjoint gather), which for the
// Max-Cut instances is ~2.6x the spectral value (config 2: Gershgorin lo =
// -12.6, lambda_min(S) = -4.87, tools/gpu_lo_check.py): a damped interval
// that wide slows the filter on every column near the cut.  This kernel
// estimates lambda_max(Z_k) with a short Lanczos run (one CTA per instance,
// vectors in shared memory) and stores it, with a margin of 2% of the
// estimated spectral width, in State::zlam; the iteration kernel then uses
// max(Gershgorin, -alpha zlam).  The eigensolver accepts Ritz pairs on their
// residuals only, so a misestimate costs filter efficiency, never accuracy
// (and eigenvalues slightly below the interval are amplified by only
// cosh(m sqrt(2 delta))).  Replaces nothing in the reference: ARPACK
// (symmat.py:189-199) needs no spectral interval.
#pragma once
#include "common.cuh"

namespace pdsdp {

#ifndef PDSDP_ZL_STEPS
#define PDSDP_ZL_STEPS 48      // Lanczos steps per estimate
#endif
#define PDSDP_ZL_THREADS 512
#define PDSDP_ZL_NMAX 8192     // vectors q, q_prev, w in shared memory

__device__ __forceinline__ double zl_block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += red[i];   // fixed order: identical in every thread
  return s;
}

// number of eigenvalues of the tridiagonal (a, b) below x (Sturm sequence)
__device__ int zl_sturm(const double* a, const double* b, int k, double x) {
  int cnt = 0;
  double d = 1.0;
  for (int i = 0; i < k; ++i) {
    const double bb = (i > 0) ? b[i - 1] * b[i - 1] : 0.0;
    d = (a[i] - x) - ((i > 0) ? bb / d : 0.0);
    if (d == 0.0) d = -1e-300;
    if (d < 0.0) ++cnt;
  }
  return cnt;
}

// list[2 i] = instance, list[2 i + 1] = y parity of the Z buffer to use
__global__ void __launch_bounds__(PDSDP_ZL_THREADS, 1)
zlanczos_kernel(const Inst* __restrict__ insts, const int* __restrict__ list) {
  extern __shared__ __align__(16) double zsm[];
  __shared__ double red[32];
  __shared__ double ta[PDSDP_ZL_STEPS], tb[PDSDP_ZL_STEPS];
  const Inst& d = insts[list[2 * blockIdx.x]];
  State* st = d.st;
  const int n = d.n, tid = threadIdx.x, nt = blockDim.x;
  if (d.nd > 0 || n > PDSDP_ZL_NMAX || n < 2) {   // dense rank-one rows: keep Gershgorin
    if (tid == 0) st->zlam_ok = 0.0;
    return;
  }
  const double* __restrict__ zv = (list[2 * blockIdx.x + 1] & 1) ? d.zbuf1 : d.zbuf0;
  double* q = zsm;
  double* qp = zsm + n;
  double* w = zsm + 2 * n;
  double s2 = 0.0;
  for (int i = tid; i < n; i += nt) {
    const double v = hash_uniform(0x1A2C05ull, (uint64_t)i, 7ull) - 0.5;
    q[i] = v;
    qp[i] = 0.0;
    s2 = fma(v, v, s2);
  }
  const double nrm = sqrt(zl_block_sum(s2, red));
  for (int i = tid; i < n; i += nt) q[i] /= nrm;
  __syncthreads();
  int k = 0;
  double beta = 0.0;
  for (int j = 0; j < PDSDP_ZL_STEPS; ++j) {
    double aq = 0.0;
    for (int i = tid; i < n; i += nt) {
      double acc = 0.0;
      for (int e = d.zptr[i]; e < d.zptr[i + 1]; ++e) acc = fma(zv[e], q[d.zcol[e]], acc);
      w[i] = acc;
      aq = fma(acc, q[i], aq);
    }
    const double a = zl_block_sum(aq, red);
    double b2 = 0.0;
    for (int i = tid; i < n; i += nt) {
      const double v = w[i] - a * q[i] - beta * qp[i];
      w[i] = v;
      b2 = fma(v, v, b2);
    }
    const double bn = sqrt(zl_block_sum(b2, red));
    if (tid == 0) { ta[j] = a; tb[j] = bn; }
    k = j + 1;
    if (!(bn > 1e-12 * fabs(a) + 1e-300)) break;   // invariant subspace
    for (int i = tid; i < n; i += nt) { qp[i] = q[i]; q[i] = w[i] / bn; }
    beta = bn;
    __syncthreads();
  }
  __syncthreads();
  if (tid == 0) {
    // extreme eigenvalues of T_k by bisection in its Gershgorin interval
    double lo = 1e300, hi = -1e300;
    for (int i = 0; i < k; ++i) {
      const double r = ((i > 0) ? fabs(tb[i - 1]) : 0.0) + ((i + 1 < k) ? fabs(tb[i]) : 0.0);
      lo = fmin(lo, ta[i] - r);
      hi = fmax(hi, ta[i] + r);
    }
    double x0 = lo, x1 = hi;          // largest: count(x) == k - 1 <-> x below it
    for (int it = 0; it < 100 && x1 - x0 > 1e-13 * fmax(fabs(x0), fabs(x1)); ++it) {
      const double xm = 0.5 * (x0 + x1);
      if (zl_sturm(ta, tb, k, xm) >= k) x1 = xm; else x0 = xm;
    }
    const double tmax = x1;
    double y0 = lo, y1 = hi;          // smallest: count(x) == 0 <-> x below it
    for (int it = 0; it < 100 && y1 - y0 > 1e-13 * fmax(fabs(y0), fabs(y1)); ++it) {
      const double xm = 0.5 * (y0 + y1);
      if (zl_sturm(ta, tb, k, xm) >= 1) y1 = xm; else y0 = xm;
    }
    const double tmin = y0;
    const bool ok = isfinite(tmax) && isfinite(tmin) && k >= 2;
    st->zlam = tmax + 0.02 * (tmax - tmin);
    st->zlam_ok = ok ? 1.0 : 0.0;
  }
}

}  // namespace pdsdp
