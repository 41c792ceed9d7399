// Dense-iterate path of the hot loop: the same iteration as iterate.cuh with
// X_k held as a dense n x n matrix in HBM and the PSD projection done by a
// FULL eigendecomposition on the device.  It is what the reference falls back
// to whenever its Krylov path does not apply --
//   truncated_eigen: dense eigh when n <= 32 or 2k > n or ARPACK fails
//                    (pkg/src/pdsdp/symmat.py:158-161,181-185,200-207),
//   proj_psd:        full eigh of the exact solver (symmat.py:223-226,
//                    pdhg.py:166-174, 221-288)
// -- and what this library switches an instance to when the projection
// argument has more positive eigenvalues than an in-shared-memory eigen block
// (PDSDP_BMAX) holds.  Every step is a whole-GPU, HBM-bound kernel:
//
//   dense_arg_*        S = X_k - alpha (C + M^T y_k)           lowrank.py:97-98
//   jacobi_round       full eigendecomposition of S (one-sided Jacobi)
//   eig_finalize/sort  eigenvalues, unit eigenvectors, descending order
//   recon              X+ = sum_{i<r, lam_i>0} lam_i u_i u_i^T  symmat.py:212-220
//   dense_dual         y+ = u - alpha proj_box(u/alpha)         pdhg.py:185-195
//   dense_adjoint      Z_k+1 = C + M^T y+, support correction   problem.py:147-154
//   dense_presid       ||dX/alpha - M^T dy||_F, finiteness      pdhg.py:198-218
//
// Eigensolver: Hestenes one-sided Jacobi on W = S + c I with c twice the
// Gershgorin radius, so W is SPD with condition <= 3.  Rotating ROWS p, q of
// the (symmetric, row-major) W from the left by the plane rotation that makes
// them orthogonal converges to W' = Lambda' Q^T: row j is (lam_j + c) q_j^T.
// No separate eigenvector matrix is accumulated: the rows themselves are the
// scaled eigenvectors and lam_j = ||row_j|| - c.  Each round of the round-robin
// ordering holds n/2 disjoint pairs -> one CTA per pair, both rows staged in
// shared memory (read once, written once per rotation: HBM/L2 streaming).
// Deterministic: fixed reduction trees, the only atomic is an integer counter.
#pragma once
#include "common.cuh"
#include "small_dense.cuh"

namespace pdsdp {

#define DENSE_THREADS 256
#define DENSE_PART_MAX 8192      // per-block partial slots (x 4 quantities)
#define DENSE_SCAL 64

// scalar slots (device doubles)
enum { DS_SHIFT = 0, DS_NSEL, DS_LAMK, DS_ED2, DS_DYSD, DS_FIN, DS_CORR, DS_DENSE, DS_QN, DS_QD = DS_QN + PDSDP_NDMAX,
       DS_XFIN = DS_QD + PDSDP_NDMAX, DS_ROT };

struct DenseDev {
  int n;
  double* X[2];        // X_k / X_k+1 (cur = index of X_k)
  double* W;           // projection argument, then scaled eigenvectors (rows)
  double* lam;         // [n] eigenvalues (unsorted, row order)
  double* lams;        // [n] sorted descending
  int* idx;            // [n] row of the i-th largest eigenvalue
  double* rowsum;      // [n]
  double* part;        // [4][DENSE_PART_MAX] per-block partials
  double* scal;        // [DENSE_SCAL]
  unsigned int* rot;   // rotations applied in the current sweep
  unsigned long long* maxoff;   // blocked Jacobi: largest relative off-diagonal Gram entry of the sweep
};

__device__ __forceinline__ double block_sum_256(double v, double* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sh[k];
  return t;
}

// W = X - sum_q coef_q u_q u_q^T  (dense rank-one constraint rows; coef_q =
// alpha sig_q y_k[row_q]); one block row per matrix row.
__global__ void dense_arg_kernel(int n, const double* __restrict__ X, double* __restrict__ W, double alpha,
                                 int nd, const double* __restrict__ du, const double* __restrict__ yk, Inst d) {
  const int i = blockIdx.y;
  double cf[PDSDP_NDMAX];
  for (int q = 0; q < PDSDP_NDMAX; ++q) cf[q] = (q < nd) ? alpha * d.dsig[q] * yk[d.drow[q]] * du[(size_t)q * n + i] : 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    double v = X ? X[(size_t)i * n + j] : 0.0;
    for (int q = 0; q < nd; ++q) v = fma(-cf[q], du[(size_t)q * n + j], v);
    W[(size_t)i * n + j] = v;
  }
}

// W[i, j] -= alpha Z[i, j] over the slots of the symmetric CSR (both triangles present)
__global__ void dense_arg_sparse_kernel(int n, int nz, const int* __restrict__ zrow, const int* __restrict__ zcol,
                                        const double* __restrict__ zv, double* __restrict__ W, double alpha) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nz; e += gridDim.x * blockDim.x)
    W[(size_t)zrow[e] * n + zcol[e]] -= alpha * zv[e];
}

// rowsum[i] = sum_j |W[i, j]|   (one warp per row)
__global__ void dense_rowabs_kernel(int n, const double* __restrict__ W, double* __restrict__ rowsum) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= n) return;
  double s = 0.0;
  for (int j = lane; j < n; j += 32) s += fabs(W[(size_t)row * n + j]);
  s = warp_sum(s);
  if (lane == 0) rowsum[row] = s;
}

// shift c = 2 max_i rowsum_i (1 when the matrix is zero); W += c I.  One block.
__global__ void dense_shift_kernel(int n, double* __restrict__ W, const double* __restrict__ rowsum,
                                   double* __restrict__ scal) {
  __shared__ double sh[32];
  double g = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) g = fmax(g, rowsum[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) g = fmax(g, __shfl_xor_sync(0xffffffffu, g, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = g;
  __syncthreads();
  double m = 0.0;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) m = fmax(m, sh[k]);
  double c = 2.0 * m;
  if (!(c > 0.0)) c = 1.0;
  if (!isfinite(c)) c = 0.0;      // non-finite input: eigenvalues come out non-finite, reported as such
  if (threadIdx.x == 0) scal[DS_SHIFT] = c;
  for (int i = threadIdx.x; i < n; i += blockDim.x) W[(size_t)i * n + i] += c;
}

// round-robin pairing of nn = n + (n & 1) indices, round t in [0, nn - 1)
__device__ __forceinline__ void rr_pair(int j, int t, int nn, int& p, int& q) {
  const int R = nn - 1, t0 = j, t1 = nn - 1 - j;
  p = (t0 == 0) ? 0 : 1 + (t0 - 1 + t) % R;
  q = 1 + (t1 - 1 + t) % R;
  if (p > q) { const int s = p; p = q; q = s; }
}

// One round of the one-sided Jacobi sweep: CTA j rotates rows (p, q) of W.
// Dynamic shared memory: 2 n doubles.
__global__ void __launch_bounds__(DENSE_THREADS)
jacobi_round_kernel(int n, double* __restrict__ W, int t, double tol, unsigned int* __restrict__ rot) {
  extern __shared__ __align__(16) double jsm[];
  __shared__ double sh[3][DENSE_THREADS / 32];
  const int nn = n + (n & 1);
  int p, q;
  rr_pair(blockIdx.x, t, nn, p, q);
  if (q >= n) return;                       // the padding index of an odd n
  double* rp = jsm;
  double* rq = jsm + n;
  double* gp = W + (size_t)p * n;
  double* gq = W + (size_t)q * n;
  double a = 0.0, b = 0.0, d = 0.0;
  for (int k = threadIdx.x; k < n; k += DENSE_THREADS) {
    const double x = gp[k], y = gq[k];
    rp[k] = x; rq[k] = y;
    a = fma(x, x, a); b = fma(y, y, b); d = fma(x, y, d);
  }
  a = warp_sum(a); b = warp_sum(b); d = warp_sum(d);
  if ((threadIdx.x & 31) == 0) { sh[0][threadIdx.x >> 5] = a; sh[1][threadIdx.x >> 5] = b; sh[2][threadIdx.x >> 5] = d; }
  __syncthreads();
  a = b = d = 0.0;
  for (int k = 0; k < DENSE_THREADS / 32; ++k) { a += sh[0][k]; b += sh[1][k]; d += sh[2][k]; }
  if (!(fabs(d) > tol * sqrt(a * b))) return;      // already orthogonal (or non-finite: leave it)
  // rotation making the rows orthogonal: tan(2 phi) = 2 d / (a - b)
  const double zeta = (b - a) / (2.0 * d);
  const double tt = ((zeta >= 0.0) ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  const double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
  for (int k = threadIdx.x; k < n; k += DENSE_THREADS) {
    const double x = rp[k], y = rq[k];
    gp[k] = c * x - s * y;
    gq[k] = s * x + c * y;
  }
  if (threadIdx.x == 0) atomicAdd(rot, 1u);
}

// The same round with both rows moved by TMA bulk copies (cp.async.bulk,
// SASS UBLKCP): one thread issues the two row loads against an mbarrier, so a
// CTA has its whole 16 n bytes in flight at once instead of one 8-byte load
// per thread; the rotated rows go back with bulk stores from shared memory.
// Needs 16-byte aligned rows: n even.  Dynamic shared memory: 2 n doubles.
__device__ __forceinline__ unsigned dp_smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(DENSE_THREADS)
jacobi_round_tma_kernel(int n, double* __restrict__ W, int t, double tol, unsigned int* __restrict__ rot) {
  extern __shared__ __align__(16) double jsm[];
  __shared__ double sh[3][DENSE_THREADS / 32];
  __shared__ __align__(8) unsigned long long mbar;
  const int nn = n + (n & 1);
  int p, q;
  rr_pair(blockIdx.x, t, nn, p, q);
  if (q >= n) return;
  double* rp = jsm;
  double* rq = jsm + n;
  double* gp = W + (size_t)p * n;
  double* gq = W + (size_t)q * n;
  const unsigned bytes = (unsigned)n * 8u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(dp_smem_u32(&mbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(dp_smem_u32(&mbar)), "r"(2u * bytes) : "memory");
    for (unsigned off = 0; off < bytes; off += 65536u) {
      const unsigned piece = min(65536u, bytes - off);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dp_smem_u32(rp) + off), "l"(reinterpret_cast<const char*>(gp) + off), "r"(piece),
                     "r"(dp_smem_u32(&mbar)) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dp_smem_u32(rq) + off), "l"(reinterpret_cast<const char*>(gq) + off), "r"(piece),
                     "r"(dp_smem_u32(&mbar)) : "memory");
    }
  }
  __syncthreads();       // the barrier is initialised before anyone waits on it
  asm volatile("{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra WAIT_%=;\n\t}"
               ::"r"(dp_smem_u32(&mbar)) : "memory");
  double a = 0.0, b = 0.0, d = 0.0;
  for (int k = threadIdx.x; k < n; k += DENSE_THREADS) {
    const double x = rp[k], y = rq[k];
    a = fma(x, x, a); b = fma(y, y, b); d = fma(x, y, d);
  }
  a = warp_sum(a); b = warp_sum(b); d = warp_sum(d);
  if ((threadIdx.x & 31) == 0) { sh[0][threadIdx.x >> 5] = a; sh[1][threadIdx.x >> 5] = b; sh[2][threadIdx.x >> 5] = d; }
  __syncthreads();
  a = b = d = 0.0;
  for (int k = 0; k < DENSE_THREADS / 32; ++k) { a += sh[0][k]; b += sh[1][k]; d += sh[2][k]; }
  if (!(fabs(d) > tol * sqrt(a * b))) return;
  const double zeta = (b - a) / (2.0 * d);
  const double tt = ((zeta >= 0.0) ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  const double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
  for (int k = threadIdx.x; k < n; k += DENSE_THREADS) {
    const double x = rp[k], y = rq[k];
    rp[k] = c * x - s * y;
    rq[k] = s * x + c * y;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic-proxy writes visible to the bulk stores
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(rot, 1u);
    for (unsigned off = 0; off < bytes; off += 65536u) {
      const unsigned piece = min(65536u, bytes - off);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   ::"l"(reinterpret_cast<char*>(gp) + off), "r"(dp_smem_u32(rp) + off), "r"(piece) : "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   ::"l"(reinterpret_cast<char*>(gq) + off), "r"(dp_smem_u32(rq) + off), "r"(piece) : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");     // shared memory is released when the CTA exits
  }
}

// Blocked one-sided Jacobi round (n >= PDSDP_BJ_NMIN, or PDSDP_DENSE_BLOCK_NMIN in the environment): the rows are grouped in
// blocks of BJ_BS; a CTA takes one block pair (I, J) of the round-robin
// ordering, forms the 2 BS x 2 BS Gram matrix G = W_IJ W_IJ^T by streaming
// the 2 BS rows once through shared memory (64-column tiles), diagonalises G
// in shared memory (jacobi_eig4: G = Q Lam Q^T) and replaces the rows by
// Q^T W_IJ in a second streaming pass, which makes all 2 BS rows mutually
// orthogonal at once.  Per sweep every row block meets every other one:
// (n / BS) passes over the matrix instead of n with the scalar rotations --
// 16x less memory traffic -- and ~n / (2 BS) CTAs per round (one wave at
// n ~ 4700).  The Gram route is safe here because W = S + c I has condition
// <= 3.  maxoff receives the largest |g_ij| / sqrt(g_ii g_jj) seen (as the
// bits of a non-negative double): the host stops when a sweep stays below tol.
#define BJ_BS 16
#define BJ_B2 (2 * BJ_BS)
#define BJ_TC 64
#define BJ_LDS (BJ_B2 + 1)
#define BJ_THREADS 256
// jacobi_eig4's table buffer: pair decode [np (np + 1) / 2] at 0, pair index lists behind BMAX (BMAX / 2 + 1) / 2 + 8
#define BJ_TAB_INTS (PDSDP_BMAX * (PDSDP_BMAX / 2 + 1) / 2 + 8 + 2 * (PDSDP_BMAX / 2 + 1) + 16)
// measured per dense iteration (tools/gpu_dense_time.py, 11-13 sweeps either way): n = 2048 0.42 s
// blocked vs 0.30 s scalar rotations, n = 4096 1.78 vs 2.21 s -- the in-CTA 32 x 32 eigensolve and
// the single-buffered tile passes cost more than the saved traffic until the matrix leaves L2
#ifndef PDSDP_BJ_NMIN
#define PDSDP_BJ_NMIN 4096
#endif
inline size_t block_jacobi_smem_bytes() {
  return (size_t)(BJ_B2 * (BJ_TC + 1) + 4 * BJ_B2 * BJ_LDS + 4 * PDSDP_BMAX) * sizeof(double) +
         (size_t)(BJ_TAB_INTS + 8) * sizeof(int) + 64;
}
__global__ void __launch_bounds__(BJ_THREADS)
block_jacobi_round_kernel(int n, double* __restrict__ W, int t, int nbk, double tol,
                          unsigned long long* __restrict__ maxoff) {
  double* sm = reinterpret_cast<double*>(pdsdp_dsm);
  double* tile = sm;                                  // [B2][TC + 1]
  double* A = tile + BJ_B2 * (BJ_TC + 1);
  double* A2 = A + BJ_B2 * BJ_LDS;
  double* Q = A2 + BJ_B2 * BJ_LDS;
  double* Q2 = Q + BJ_B2 * BJ_LDS;
  double* cs = Q2 + BJ_B2 * BJ_LDS;                   // 4 * BMAX
  int* tab = reinterpret_cast<int*>(cs + 4 * PDSDP_BMAX);
  int* sflag = tab + BJ_TAB_INTS;
  __shared__ double redmax[BJ_THREADS / 32];
  const int tid = threadIdx.x;
  int I, J;
  rr_pair(blockIdx.x, t, nbk + (nbk & 1), I, J);
  if (J >= nbk) return;                                // the phantom block of an odd count
  auto grow = [&](int l) { return (l < BJ_BS) ? I * BJ_BS + l : J * BJ_BS + (l - BJ_BS); };
  auto load_tile = [&](int c0) {
    for (int e = tid; e < BJ_B2 * BJ_TC; e += BJ_THREADS) {
      const int l = e / BJ_TC, c = e % BJ_TC;
      const int gr = grow(l);
      tile[l * (BJ_TC + 1) + c] = (gr < n && c0 + c < n) ? W[(size_t)gr * n + c0 + c] : 0.0;
    }
  };
  // ---- Gram matrix: thread (ta, tb) owns the 2 x 2 block (2 ta .. , 2 tb ..) ----
  const int ta = tid >> 4, tb = tid & 15;
  double g00 = 0.0, g01 = 0.0, g10 = 0.0, g11 = 0.0;
  for (int c0 = 0; c0 < n; c0 += BJ_TC) {
    load_tile(c0);
    __syncthreads();
    const double* ra0 = tile + (2 * ta) * (BJ_TC + 1);
    const double* ra1 = ra0 + (BJ_TC + 1);
    const double* rb0 = tile + (2 * tb) * (BJ_TC + 1);
    const double* rb1 = rb0 + (BJ_TC + 1);
#pragma unroll 8
    for (int k = 0; k < BJ_TC; ++k) {
      const double a0 = ra0[k], a1 = ra1[k], b0 = rb0[k], b1 = rb1[k];
      g00 = fma(a0, b0, g00); g01 = fma(a0, b1, g01);
      g10 = fma(a1, b0, g10); g11 = fma(a1, b1, g11);
    }
    __syncthreads();
  }
  A[(2 * ta) * BJ_LDS + 2 * tb] = g00; A[(2 * ta) * BJ_LDS + 2 * tb + 1] = g01;
  A[(2 * ta + 1) * BJ_LDS + 2 * tb] = g10; A[(2 * ta + 1) * BJ_LDS + 2 * tb + 1] = g11;
  __syncthreads();
  // ---- largest relative off-diagonal entry; nothing to do below tol ----
  double rel = 0.0;
  for (int e = tid; e < BJ_B2 * BJ_B2; e += BJ_THREADS) {
    const int i = e / BJ_B2, j = e % BJ_B2;
    if (i != j) {
      const double dd = A[i * BJ_LDS + i] * A[j * BJ_LDS + j];
      if (dd > 0.0) rel = fmax(rel, fabs(A[i * BJ_LDS + j]) * rsqrt(dd));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) rel = fmax(rel, __shfl_xor_sync(0xffffffffu, rel, o));
  if ((tid & 31) == 0) redmax[tid >> 5] = rel;
  __syncthreads();
  rel = 0.0;
  for (int w = 0; w < BJ_THREADS / 32; ++w) rel = fmax(rel, redmax[w]);
  if (tid == 0 && rel == rel) atomicMax(maxoff, (unsigned long long)__double_as_longlong(rel));
  if (!(rel > tol)) return;
  // ---- G = Q Lam Q^T ----
  double *Aj, *Qj;
  jacobi_eig4(A, A2, Q, Q2, BJ_B2, BJ_LDS, cs, tab, sflag, BJ_B2, &Aj, &Qj);
  // ---- rows <- Q^T rows: thread (ti, cg) owns row ti, columns cg, cg + 8, ... of a tile ----
  const int ti = tid >> 3, cg = tid & 7;
  const int gr = grow(ti);
  for (int c0 = 0; c0 < n; c0 += BJ_TC) {
    load_tile(c0);
    __syncthreads();
    double out[BJ_TC / 8];
#pragma unroll
    for (int u = 0; u < BJ_TC / 8; ++u) out[u] = 0.0;
    for (int k = 0; k < BJ_B2; ++k) {
      const double q = Qj[k * BJ_LDS + ti];
      const double* row = tile + k * (BJ_TC + 1) + cg;
#pragma unroll
      for (int u = 0; u < BJ_TC / 8; ++u) out[u] = fma(q, row[8 * u], out[u]);
    }
    if (gr < n)
#pragma unroll
      for (int u = 0; u < BJ_TC / 8; ++u)
        if (c0 + cg + 8 * u < n) W[(size_t)gr * n + c0 + cg + 8 * u] = out[u];
    __syncthreads();
  }
}

// lam[j] = ||row_j|| - c ; row_j <- row_j / ||row_j||   (one block per row)
__global__ void eig_finalize_kernel(int n, double* __restrict__ W, const double* __restrict__ scal,
                                    double* __restrict__ lam) {
  __shared__ double sh[32];
  const int j = blockIdx.x;
  double* row = W + (size_t)j * n;
  double a = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) a = fma(row[k], row[k], a);
  a = block_sum_256(a, sh);
  const double nrm = sqrt(a);
  const double inv = (nrm > 0.0) ? 1.0 / nrm : 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) row[k] *= inv;
  if (threadIdx.x == 0) lam[j] = nrm - scal[DS_SHIFT];
}

// descending rank by counting (ties by index): idx[rank] = j, lams[rank] = lam[j]
__global__ void eig_sort_kernel(int n, const double* __restrict__ lam, int* __restrict__ idx,
                                double* __restrict__ lams) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double lj = lam[j];
  int rank = 0;
  bool bad = !isfinite(lj);
  for (int i = 0; i < n; ++i) {
    const double li = lam[i];
    if (!isfinite(li)) bad = true;
    if (li > lj || (li == lj && i < j)) ++rank;
  }
  if (bad) rank = j;
  idx[rank] = j;
  lams[rank] = lj;
}

// kept pairs: the positive ones among the first r (a prefix of the sorted
// order); lambda_k, k = min(r + 1, n)  (symmat.py:240-245)
__global__ void eig_select_kernel(int n, int r, const double* __restrict__ lams, double* __restrict__ scal) {
  if (threadIdx.x || blockIdx.x) return;
  int ns = 0;
  double fin = 1.0;
  for (int i = 0; i < r && i < n; ++i) {
    if (lams[i] > 0.0) ++ns;
    if (!isfinite(lams[i])) fin = 0.0;
  }
  scal[DS_NSEL] = ns;
  const int k = (r + 1 < n) ? r + 1 : n;
  scal[DS_LAMK] = lams[k - 1];
  scal[DS_XFIN] = fin;
}

// Xn = sum_{t < nsel} lams[t] q_t q_t^T with q_t = vector idx[t] of Q, element
// i of vector v at Q[v * sv + i * si].  64 x 64 output tiles (upper triangle of
// tiles, mirrored), 16 x 16 threads x (4 x 4) outputs, 16 vectors per stage.
// With idx == nullptr the vectors are 0 .. nsel-1 and nsel comes from nsel_arg.
#define RECON_TILE 64
#define RECON_KS 16
__global__ void __launch_bounds__(256)
recon_kernel(int n, const double* __restrict__ Q, long long sv, long long si, const int* __restrict__ idx,
             const double* __restrict__ lams, const double* __restrict__ scal, int nsel_arg,
             double* __restrict__ Xn) {
  __shared__ double As[RECON_KS][RECON_TILE + 1];
  __shared__ double Bs[RECON_KS][RECON_TILE + 1];
  const int nt = (n + RECON_TILE - 1) / RECON_TILE;
  int I = 0, t = blockIdx.x;
  while (t >= nt - I) { t -= nt - I; ++I; }
  const int J = I + t;
  const int nsel = scal ? (int)scal[DS_NSEL] : nsel_arg;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int k0 = 0; k0 < nsel; k0 += RECON_KS) {
    for (int e = threadIdx.x; e < RECON_KS * RECON_TILE; e += 256) {
      const int kk = e / RECON_TILE, c = e % RECON_TILE;
      const int tsel = k0 + kk;
      double av = 0.0, bv = 0.0;
      if (tsel < nsel) {
        const long long v = idx ? idx[tsel] : tsel;
        const double l = lams[tsel];
        const int gi = I * RECON_TILE + c, gj = J * RECON_TILE + c;
        if (gi < n) av = Q[v * sv + gi * si] * l;
        if (gj < n) bv = Q[v * sv + gj * si];
      }
      As[kk][c] = av;
      Bs[kk][c] = bv;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < RECON_KS; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { a[u] = As[kk][ty * 4 + u]; b[u] = Bs[kk][tx * 4 + u]; }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int gi = I * RECON_TILE + ty * 4 + u, gj = J * RECON_TILE + tx * 4 + v;
      if (gi < n && gj < n) {
        if (I < J) { Xn[(size_t)gi * n + gj] = acc[u][v]; Xn[(size_t)gj * n + gi] = acc[u][v]; }
        else if (gi <= gj) {
          // diagonal tile: symmetrise exactly (symmat.py:219 forms (P + P^T) / 2)
          Xn[(size_t)gi * n + gj] = acc[u][v];
          if (gi != gj) Xn[(size_t)gj * n + gi] = acc[u][v];
        }
      }
    }
}

// out[0] = sum of v[0 .. len) in a fixed order (one block)
__global__ void reduce_sum_kernel(const double* __restrict__ v, int len, double* __restrict__ out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < len; i += blockDim.x) s += v[i];
  s = block_sum_256(s, sh);
  if (threadIdx.x == 0) out[0] = s;
}

// Quadratic forms of the dense rank-one rows, row by row:
//   tmp[(2 q) n + i]     = u_q[i] (Xn u_q)[i],   tmp[(2 q + 1) n + i] = u_q[i] (Xo u_q)[i]
// (summed over i by reduce_sum_kernel: u_q^T X u_q)
__global__ void dense_quad_kernel(int n, const double* __restrict__ Xn, const double* __restrict__ Xo, int nd,
                                  const double* __restrict__ du, double* __restrict__ tmp) {
  __shared__ double sh[32];
  const int i = blockIdx.x;
  for (int q = 0; q < nd; ++q) {
    const double* u = du + (size_t)q * n;
    double sn = 0.0, so = 0.0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      sn = fma(Xn[(size_t)i * n + j], u[j], sn);
      so = fma(Xo[(size_t)i * n + j], u[j], so);
    }
    sn = block_sum_256(sn, sh);
    so = block_sum_256(so, sh);
    if (threadIdx.x == 0) {
      tmp[(size_t)(2 * q) * n + i] = u[i] * sn;
      tmp[(size_t)(2 * q + 1) * n + i] = u[i] * so;
    }
  }
}

// Dual step (pdhg.py:185-195): one thread per constraint row.
//   u = y + alpha <A_i, 2 Xn - Xo>;  y+ = u - alpha b_i  (equalities)
//                                    y+ = u - alpha min(u / alpha, h_i)  (inequalities)
// per-row outputs: rowt[i] = (dy_i/alpha - <A_i, dX>)^2, rowt[mp + i] = dy_i <A_i, dX>,
// rowt[2 mp + i] = 1 if y+_i is not finite.
__global__ void dense_dual_kernel(Inst d, const double* __restrict__ Xn, const double* __restrict__ Xo,
                                  const double* __restrict__ yk, double* __restrict__ yn,
                                  const double* __restrict__ scal, double* __restrict__ rowt) {
  const int n = d.n, mp = d.mp;
  const double alpha = d.alpha;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < mp; i += gridDim.x * blockDim.x) {
    double s2 = 0.0, sd = 0.0;
    for (int e = d.aptr[i]; e < d.aptr[i + 1]; ++e) {
      const size_t o = (size_t)d.ai[e] * n + d.aj[e];
      const double xn = Xn[o], xo = Xo[o], g = d.ag[e];
      s2 = fma(g, 2.0 * xn - xo, s2);
      sd = fma(g, xn - xo, sd);
    }
    for (int q = 0; q < d.nd; ++q)
      if (i == d.drow[q]) {
        const double qn = scal[DS_QN + q], qo = scal[DS_QD + q];
        s2 = d.dsig[q] * (2.0 * qn - qo);
        sd = d.dsig[q] * (qn - qo);
      }
    const double u = yk[i] + alpha * s2;
    const double pr = (i < d.m) ? d.bv[i] : fmin(u / alpha, d.hv[i - d.m]);
    const double ynew = u - alpha * pr;
    const double dyi = ynew - yk[i];
    yn[i] = ynew;
    d.dy[i] = dyi;
    const double t = dyi / alpha - sd;
    rowt[i] = t * t;
    rowt[mp + i] = dyi * sd;
    rowt[2 * mp + i] = isfinite(ynew) ? 0.0 : 1.0;
  }
}

// Adjoint gather (problem.py:147-154) over the slots M^T y touches: Z_k+1 =
// C + M^T y+ into zvn, and the sparse-support part of the primal residual:
// with t0 = dX_ij/alpha - (dense-row part of M^T dy)_ij (what dense_presid
// squares for every entry) and a = (sparse M^T dy)_ij,
//   corr += w ((t0 - a)^2 - t0^2),  w = 1 (diagonal) or 2 (both triangles).
// Fixed grid: partial sums per block -> part[block].
__global__ void dense_adjoint_kernel(Inst d, const double* __restrict__ Xn, const double* __restrict__ Xo,
                                     const double* __restrict__ yn, double* __restrict__ zvn,
                                     double* __restrict__ part) {
  __shared__ double sh[32];
  const int n = d.n;
  const double ia = 1.0 / d.alpha;
  const int nk = d.dptr[n];
  double dlt[PDSDP_NDMAX];
  for (int q = 0; q < PDSDP_NDMAX; ++q) dlt[q] = (q < d.nd) ? d.dsig[q] * d.dy[d.drow[q]] : 0.0;
  double corr = 0.0;
  for (int kk = blockIdx.x * blockDim.x + threadIdx.x; kk < nk; kk += gridDim.x * blockDim.x) {
    const int e = d.dslot[kk];
    double z = d.cval[e], a = 0.0;
    for (int t = d.tptr[e]; t < d.tptr[e + 1]; ++t) {
      const int row = d.trow[t];
      const double cf = d.tcoef[t];
      z = fma(yn[row], cf, z);
      a = fma(d.dy[row], cf, a);
    }
    zvn[e] = z;
    const int i = d.zrow[e], j = d.zcol[e];
    if (j >= i) {
      const size_t o = (size_t)i * n + j;
      double t0 = (Xn[o] - Xo[o]) * ia;
      for (int q = 0; q < d.nd; ++q) t0 = fma(-dlt[q] * d.du[(size_t)q * n + i], d.du[(size_t)q * n + j], t0);
      const double t1 = t0 - a;
      corr = fma((i == j) ? 1.0 : 2.0, t1 * t1 - t0 * t0, corr);
    }
  }
  corr = block_sum_256(corr, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = corr;
}

// Dense part of the primal residual, row by row: rowt[i] = sum_j (dX_ij/alpha -
// sum_q dlt_q u_qi u_qj)^2, rowt[n + i] = 1 if row i of Xn holds a non-finite entry.
__global__ void dense_presid_kernel(Inst d, const double* __restrict__ Xn, const double* __restrict__ Xo,
                                    double* __restrict__ rowt) {
  __shared__ double sh[32];
  const int n = d.n, i = blockIdx.x;
  const double ia = 1.0 / d.alpha;
  double cf[PDSDP_NDMAX];
  for (int q = 0; q < PDSDP_NDMAX; ++q)
    cf[q] = (q < d.nd) ? d.dsig[q] * d.dy[d.drow[q]] * d.du[(size_t)q * n + i] : 0.0;
  double s = 0.0, bad = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double xn = Xn[(size_t)i * n + j];
    double t0 = (xn - Xo[(size_t)i * n + j]) * ia;
    for (int q = 0; q < d.nd; ++q) t0 = fma(-cf[q], d.du[(size_t)q * n + j], t0);
    s = fma(t0, t0, s);
    if (!isfinite(xn)) bad = 1.0;
  }
  s = block_sum_256(s, sh);
  bad = block_sum_256(bad, sh);
  if (threadIdx.x == 0) { rowt[i] = s; rowt[n + i] = (bad > 0.0) ? 1.0 : 0.0; }
}

// tr(C X) over the C pattern (both triangles of the symmetric CSR), fixed grid
__global__ void dense_objective_kernel(int n, int nz, const int* __restrict__ zrow, const int* __restrict__ zcol,
                                       const double* __restrict__ cval, const double* __restrict__ X,
                                       double* __restrict__ part) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nz; e += gridDim.x * blockDim.x) {
    const double c = cval[e];
    if (c != 0.0) s = fma(c, X[(size_t)zrow[e] * n + zcol[e]], s);
  }
  s = block_sum_256(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// packed upper triangle (row-major, sqrt 2 off-diagonals; symmat.py:66-86) of a dense X
__global__ void dense_pack_kernel(int n, const double* __restrict__ X, double* __restrict__ out) {
  const int i = blockIdx.y;
  const long long start = (long long)i * n - (long long)i * (i - 1) / 2;
  for (int j = i + blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double v = 0.5 * (X[(size_t)i * n + j] + X[(size_t)j * n + i]);
    out[start + (j - i)] = (i == j) ? v : v * 1.4142135623730951;
  }
}

}  // namespace pdsdp
