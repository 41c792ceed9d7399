// Operator-norm power iteration on M^T M (reference problem.py:157-185) and
// the op-level linear maps M(X), M^T(y) over packed positions
// (reference problem.py:140-154).  Vectors live in "T-space": the packed
// positions touched by at least one constraint row (every other packed entry
// of M^T y is zero, so the iteration never leaves that subspace after the
// first product).  All reductions are two-level with a fixed order.
#pragma once
#include <cooperative_groups.h>
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
  double* norm_part;    // [2 * NORM_BLOCKS]
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

// `iters` power iterations x <- M^T M x / |M^T M x| in ONE cooperative launch
// (grid-wide barriers between the phases instead of eight launches per
// iteration); hist[it] = |M x| of iteration it.  The work decomposition is
// independent of the grid size (segment blocks of 256 threads as in
// seg_dot_kernel, NORM_BLOCKS virtual blocks for the norms, final sums in
// index order), so the estimates do not depend on the launch shape.
__global__ void __launch_bounds__(256) opnorm_power_kernel(OpnormDev o, int iters, double* __restrict__ hist) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double w[32];
  __shared__ double bc;
  const int tid = threadIdx.x;
  const int gtid = blockIdx.x * blockDim.x + tid, gsize = gridDim.x * blockDim.x;
  auto block_total = [&](double s) {      // fixed order: warp tree, then the warps in index order (thread 0)
    s = warp_sum(s);
    __syncthreads();
    if ((tid & 31) == 0) w[tid >> 5] = s;
    __syncthreads();
    double t = 0.0;
    if (tid == 0) for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += w[i];
    return t;
  };
  auto sumsq_parts = [&](const double* v, int len, double* part) {
    for (int vb = blockIdx.x; vb < NORM_BLOCKS; vb += gridDim.x) {
      double s = 0.0;
      for (int i = vb * 256 + tid; i < len; i += NORM_BLOCKS * 256) s = fma(v[i], v[i], s);
      const double t = block_total(s);
      if (tid == 0) part[vb] = t;
    }
  };
  for (int it = 0; it < iters; ++it) {
    // y = M x: segment partials, then the rows
    for (int sgi = blockIdx.x; sgi < o.nseg; sgi += gridDim.x) {
      double s = 0.0;
      for (int e = o.seg_lo[sgi] + tid; e < o.seg_hi[sgi]; e += 256) s = fma(o.mval[e], o.x[o.mcol[e]], s);
      const double t = block_total(s);
      if (tid == 0) o.seg_part[sgi] = t;
    }
    grid.sync();
    for (int i = gtid; i < o.mp; i += gsize) {
      double t = 0.0;
      for (int sgi = o.row_seg[i]; sgi < o.row_seg[i + 1]; ++sgi) t += o.seg_part[sgi];
      o.y[i] = t;
    }
    grid.sync();
    // |y|^2 partials and x = M^T y
    sumsq_parts(o.y, o.mp, o.norm_part);
    for (int t = gtid; t < o.nT; t += gsize) {
      double a = 0.0;
      for (int e = o.tptr[t]; e < o.tptr[t + 1]; ++e) a = fma(o.tval[e], o.y[o.trow[e]], a);
      o.x[t] = a;
    }
    grid.sync();
    if (blockIdx.x == 0 && tid == 0) {
      double t = 0.0;
      for (int i = 0; i < NORM_BLOCKS; ++i) t += o.norm_part[i];
      const double s = sqrt(t);
      o.scal[0] = s;
      hist[it] = s;
    }
    sumsq_parts(o.x, o.nT, o.norm_part + NORM_BLOCKS);
    grid.sync();
    if (tid == 0) {
      double t = 0.0;
      for (int i = 0; i < NORM_BLOCKS; ++i) t += o.norm_part[NORM_BLOCKS + i];
      bc = sqrt(t);
    }
    __syncthreads();
    const double nx = bc;
    if (blockIdx.x == 0 && tid == 0) o.scal[1] = nx;
    for (int t = gtid; t < o.nT; t += gsize) o.x[t] = o.x[t] / nx;
    grid.sync();
  }
}

}  // namespace pdsdp
