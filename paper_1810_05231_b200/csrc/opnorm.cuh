// Operator-norm power iteration on M^T M (reference problem.py:157-185) and
// the op-level linear maps M(X), M^T(y) over packed positions
// (reference problem.py:140-154).  Vectors live in "T-space": the packed
// positions touched by at least one constraint row (every other packed entry
// of M^T y is zero, so the iteration never leaves that subspace after the
// first product).  All reductions are two-level with a fixed order.
#pragma once
#include "common.cuh"

namespace pdsdp {

#define SEG_LEN 2048

struct OpnormDev {
  int mp, nT, nseg, pad;
  const int* seg_lo;    // [nseg] first entry of the segment
  const int* seg_hi;    // [nseg]
  const int* row_seg;   // [mp+1] segments of each row
  const int* mcol;      // [nnz] T-index of each entry
  const double* mval;   // [nnz] packed value
  const int* tptr;      // [nT+1] rows touching each T position
  const int* trow;
  const double* tval;
  double* x;            // [nT]
  double* y;            // [mp]
  double* seg_part;     // [nseg]
  double* norm_part;    // [NORM_BLOCKS]
  double* scal;         // [4]: |y|, |x|
  double* s_hist;       // [chunk]
};

#define NORM_BLOCKS 148

__global__ void seg_dot_kernel(OpnormDev o) {
  const int sgi = blockIdx.x;
  double s = 0.0;
  for (int e = o.seg_lo[sgi] + threadIdx.x; e < o.seg_hi[sgi]; e += blockDim.x) s = fma(o.mval[e], o.x[o.mcol[e]], s);
  s = warp_sum(s);
  __shared__ double w[32];
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += w[i];
    o.seg_part[sgi] = t;
  }
}

__global__ void seg_final_kernel(OpnormDev o) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < o.mp; i += gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int sgi = o.row_seg[i]; sgi < o.row_seg[i + 1]; ++sgi) t += o.seg_part[sgi];
    o.y[i] = t;
  }
}

__global__ void adjT_kernel(OpnormDev o) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < o.nT; t += gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int e = o.tptr[t]; e < o.tptr[t + 1]; ++e) a = fma(o.tval[e], o.y[o.trow[e]], a);
    o.x[t] = a;
  }
}

// sum of squares of v[0..len) -> part[blockIdx.x]
__global__ void sumsq_kernel(const double* __restrict__ v, int len, double* part) {
  double s = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) s = fma(v[i], v[i], s);
  s = warp_sum(s);
  __shared__ double w[32];
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += w[i];
    part[blockIdx.x] = t;
  }
}

// dst = sqrt(sum part); optionally also store into hist[idx]
__global__ void norm_final_kernel(const double* part, int np, double* dst, double* hist, int idx) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < np; ++i) t += part[i];
    const double s = sqrt(t);
    *dst = s;
    if (hist) hist[idx] = s;
  }
}

__global__ void inv_scale_kernel(double* v, int len, const double* nrm) {
  const double s = *nrm;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) v[i] = v[i] / s;
}

}  // namespace pdsdp
