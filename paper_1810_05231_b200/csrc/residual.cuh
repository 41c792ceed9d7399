// Whole-GPU kernels around the cluster iteration:
//   residual_kernel   verification mode only (pdsdp_set_verify_residual): the
//                     dense part ||dX/alpha||_F^2 of the primal residual
//                     (reference pdhg.py:198-208) evaluated entry by entry on
//                     FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64), next to
//                     the factored form the iteration kernel uses:
//                     dX/alpha = [V | F] diag(lamN, -lamF)/alpha [V | F]^T is a
//                     rank-(r + rF) SYRK evaluated tile by tile over the upper
//                     triangle and reduced to one scalar; nothing n x n is stored.
//   objective_kernel  tr(C X) over the C/constraint support (reference pdhg.py:
//                     ProgressInfo objective, lowrank.py:159,168,191)
//   pack_kernel       X -> packed upper triangle with sqrt(2) off-diagonals
//                     (reference symmat.py:66-86) for the boundary download
//   init_kernel       reset of an instance (X0 = 0, y0 = 0, Z = C)
#pragma once
#include "common.cuh"

namespace pdsdp {

#define RES_TILE 64
#define RES_THREADS 128
#define RES_KMAX (2 * PDSDP_BMAX)

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__device__ __forceinline__ void tile_of(int t, int nt, int& I, int& J) {
  int i = 0;
  while (t >= nt - i) { t -= nt - i; ++i; }
  I = i;
  J = i + t;
}

// grid: (max tiles, active instances); block RES_THREADS (4 warps)
__global__ void __launch_bounds__(RES_THREADS)
residual_kernel(const Inst* __restrict__ insts, const Ctl* __restrict__ ctls, const int* __restrict__ active,
                int step) {
  extern __shared__ __align__(16) double rsm[];
  const int inst_id = active[blockIdx.y];
  const Inst d = insts[inst_id];
  if (*(volatile int*)d.stopf) return;
  const State* st = d.st;
  const int n = d.n, ld = d.ld;
  const int nt = (n + RES_TILE - 1) / RES_TILE;
  const int ntile = nt * (nt + 1) / 2;
  if ((int)blockIdx.x >= ntile) return;
  int I, J;
  tile_of(blockIdx.x, nt, I, J);
  const int rN = st->r_cur, rF = st->rF_used;
  const int K = rN + rF;
  const int Kp = (K + 3) & ~3;
  const int lda = Kp + 1;
  double* GI = rsm;
  double* GJ = rsm + RES_TILE * lda;
  const double ia = 1.0 / d.alpha;
  for (int e = threadIdx.x; e < RES_TILE * Kp; e += blockDim.x) {
    const int row = e / Kp, l = e % Kp;
    const int gi = I * RES_TILE + row, gj = J * RES_TILE + row;
    double a = 0.0, bb = 0.0;
    if (l < rN) {
      if (st->lamN[l] != 0.0) {
        if (gi < n) a = d.V[(size_t)gi * ld + l] * (st->lamN[l] * ia);
        if (gj < n) bb = d.V[(size_t)gj * ld + l];
      }
    } else if (l < K) {
      const int q = l - rN;
      if (st->lamF[q] != 0.0) {
        if (gi < n) a = -d.F[(size_t)gi * ld + q] * (st->lamF[q] * ia);
        if (gj < n) bb = d.F[(size_t)gj * ld + q];
      }
    }
    GI[row * lda + l] = a;
    GJ[row * lda + l] = bb;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  double acc[2][8][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) { acc[a][b][0] = 0.0; acc[a][b][1] = 0.0; }
  for (int k0 = 0; k0 < Kp; k0 += 4) {
    double af[2], bf[8];
#pragma unroll
    for (int a = 0; a < 2; ++a) af[a] = GI[(warp * 16 + a * 8 + g) * lda + k0 + tq];
#pragma unroll
    for (int b = 0; b < 8; ++b) bf[b] = GJ[(b * 8 + g) * lda + k0 + tq];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
  }
  double sum = 0.0;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = I * RES_TILE + warp * 16 + a * 8 + g;
        const int j = J * RES_TILE + b * 8 + tq * 2 + h;
        if (i < n && j < n && (I < J || i <= j)) {
          const double v = acc[a][b][h];
          sum = fma((i == j) ? 1.0 : 2.0, v * v, sum);
        }
      }
  sum = warp_sum(sum);
  __shared__ double wsum[RES_THREADS / 32];
  __shared__ unsigned int ticket;
  if (lane == 0) wsum[warp] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < RES_THREADS / 32; ++w) t += wsum[w];
    d.rpart[blockIdx.x] = t;
    __threadfence();
    ticket = atomicAdd(d.rcount, 1u);
  }
  __syncthreads();
  if (ticket != (unsigned)(ntile - 1)) return;
  // last block: deterministic final reduction of the tile partials
  __threadfence();
  double t = 0.0;
  for (int i = threadIdx.x; i < ntile; i += blockDim.x) t += ((volatile double*)d.rpart)[i];
  t = warp_sum(t);
  if (lane == 0) wsum[warp] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double dense = 0.0;
    for (int w = 0; w < (int)(RES_THREADS / 32); ++w) dense += wsum[w];
    d.out[step * PDSDP_OUT_LEN + O_DENSE_EXACT] = dense;
    *d.rcount = 0u;
  }
}

// tr(C X) for X = U diag(lam) U^T, U = V (which == 0, lamN, r_cur) or F
// (which == 1, lamF, rF_used).  One block per instance-slice, last block sums.
__global__ void objective_kernel(const Inst* __restrict__ insts, const int* __restrict__ active, int which,
                                 double* __restrict__ partial, unsigned int* counter, double* result) {
  const Inst d = insts[active[blockIdx.y]];
  const State* st = d.st;
  const int ld = d.ld;
  const double* U = which ? d.F : d.V;
  const double* lam = which ? st->lamF : st->lamN;
  const int r = which ? st->rF_used : st->r_cur;
  double s = 0.0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < d.nz; e += gridDim.x * blockDim.x) {
    const double c = d.cval[e];
    if (c == 0.0) continue;
    const double* Ui = U + (size_t)d.zrow[e] * ld;
    const double* Uj = U + (size_t)d.zcol[e] * ld;
    double xv = 0.0;
    for (int l = 0; l < r; ++l) if (lam[l] != 0.0) xv = fma(Ui[l] * lam[l], Uj[l], xv);
    s = fma(c, xv, s);
  }
  s = warp_sum(s);
  __shared__ double ws[32];
  __shared__ unsigned int tk;
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  const int slot = blockIdx.y * gridDim.x + blockIdx.x;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
    partial[slot] = t;
    __threadfence();
    tk = atomicAdd(counter + blockIdx.y, 1u);
  }
  __syncthreads();
  if (tk != gridDim.x - 1) return;
  __threadfence();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (unsigned i = 0; i < gridDim.x; ++i) t += ((volatile double*)partial)[blockIdx.y * gridDim.x + i];
    result[blockIdx.y] = t;
    counter[blockIdx.y] = 0u;
  }
}

// packed[pos] for the upper triangle, row-major (reference packed_index).
__global__ void pack_kernel(const Inst* __restrict__ insts, int inst, int which, double* __restrict__ out) {
  const Inst d = insts[inst];
  const State* st = d.st;
  const int n = d.n, ld = d.ld;
  const double* U = which ? d.F : d.V;
  const double* lam = which ? st->lamF : st->lamN;
  const int r = which ? st->rF_used : st->r_cur;
  const long long P = (long long)n * (n + 1) / 2;
  for (long long pos = blockIdx.x * (long long)blockDim.x + threadIdx.x; pos < P;
       pos += (long long)gridDim.x * blockDim.x) {
    // row i: start(i) = i*n - i(i-1)/2 ; invert by float estimate + fix-up
    double disc = (2.0 * n + 1.0) * (2.0 * n + 1.0) - 8.0 * (double)pos;
    long long i = (long long)floor(((2.0 * n + 1.0) - sqrt(fmax(disc, 0.0))) * 0.5);
    if (i < 0) i = 0;
    if (i > n - 1) i = n - 1;
    while (i > 0 && i * n - i * (i - 1) / 2 > pos) --i;
    while (i + 1 < n && (i + 1) * n - (i + 1) * i / 2 <= pos) ++i;
    const long long j = pos - (i * n - i * (i - 1) / 2) + i;
    const double* Ui = U + (size_t)i * ld;
    const double* Uj = U + (size_t)j * ld;
    double xv = 0.0;
    for (int l = 0; l < r; ++l) if (lam[l] != 0.0) xv = fma(Ui[l] * lam[l], Uj[l], xv);
    out[pos] = (i == j) ? xv : xv * 1.4142135623730951;
  }
}

// reset: y = 0, Z = C, state cleared; gersh(C) via max over rows
__global__ void init_kernel(const Inst* __restrict__ insts, int inst, double seed) {
  const Inst d = insts[inst];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < d.nz; e += gridDim.x * blockDim.x) { d.zbuf0[e] = d.cval[e]; d.zbuf1[e] = d.cval[e]; }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d.mp; i += gridDim.x * blockDim.x) {
    d.ybuf0[i] = 0.0; d.ybuf1[i] = 0.0; d.dy[i] = 0.0;
  }
  double g = 0.0;
  for (int rho = blockIdx.x * blockDim.x + threadIdx.x; rho < d.n; rho += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int e = d.zptr[rho]; e < d.zptr[rho + 1]; ++e) s += fabs(d.cval[e]);
    g = fmax(g, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) g = fmax(g, __shfl_xor_sync(0xffffffffu, g, o));
  if ((threadIdx.x & 31) == 0 && g > 0.0)
    atomicMax((unsigned long long*)&d.st->lo_par[0], (unsigned long long)__double_as_longlong(g));  // non-negative doubles order as integers
}

}  // namespace pdsdp
