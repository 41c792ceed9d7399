// Block-local dense kernels on b x b FP64 matrices in shared memory
// (b <= PDSDP_BMAX).  Every CTA of a cluster runs these redundantly on
// bit-identical inputs, so every CTA holds bit-identical results and no
// broadcast barrier is needed.  All routines are deterministic.
//
// They replace the small dense work ARPACK does inside dsaupd/dseupd
// (reference symmat.py:189-199): Gram Cholesky (orthonormalisation),
// the Rayleigh-Ritz eigensolve and the descending sort of symmat.py:208.
#pragma once
#include "common.cuh"

// Jacobi rotation thresholds relative to ||A||_F: pairs whose Ritz values are
// used (kept pairs and the certificate) and guard pairs (warm start only)
#ifndef PDSDP_JAC_TOL_IMP
#define PDSDP_JAC_TOL_IMP 1e-14
#endif
#ifndef PDSDP_JAC_TOL_GUARD
#define PDSDP_JAC_TOL_GUARD 1e-8
#endif

namespace pdsdp {

// In-place Cholesky G = L L^T (lower) of an SPD matrix scaled to unit
// diagonal first: G' = D G D, D = diag(G)^-1/2.  On exit G holds L' (lower,
// upper triangle zeroed) and dsc[i] = D_ii.  Returns false on breakdown.
__device__ bool chol_scaled(double* G, int b, int lds, double* dsc, int* sflag) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) *sflag = 1;
  for (int i = tid; i < b; i += nt) {
    double g = G[i * lds + i];
    dsc[i] = (g > 0.0 && isfinite(g)) ? rsqrt(g) : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < b * b; e += nt) {
    int i = e / b, j = e % b;
    G[i * lds + j] = (j <= i) ? G[i * lds + j] * dsc[i] * dsc[j] : 0.0;
  }
  __syncthreads();
  for (int j = 0; j < b; ++j) {
    double d = G[j * lds + j];
    if (!(d > 1e-28)) {  // breakdown (also catches NaN)
      if (tid == 0) *sflag = 0;
      __syncthreads();
      return false;
    }
    d = sqrt(d);
    __syncthreads();
    for (int i = j + 1 + tid; i < b; i += nt) G[i * lds + j] /= d;
    if (tid == 0) G[j * lds + j] = d;
    __syncthreads();
    const int rem = b - j - 1;
    for (int e = tid; e < rem * rem; e += nt) {
      int i = j + 1 + e / rem, k = j + 1 + e % rem;
      if (k <= i) G[i * lds + k] -= G[i * lds + j] * G[k * lds + j];
    }
    __syncthreads();
  }
  return true;
}

// X = L^{-1} (lower triangular inverse), one column per thread.
__device__ void tri_inv_lower(const double* L, double* X, int b, int lds) {
  for (int c = threadIdx.x; c < b; c += blockDim.x) {
    for (int i = 0; i < c; ++i) X[i * lds + c] = 0.0;
    for (int i = c; i < b; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = c; k < i; ++k) s -= L[i * lds + k] * X[k * lds + c];
      X[i * lds + c] = s / L[i * lds + i];
    }
  }
  __syncthreads();
}

// Cyclic parallel two-sided Jacobi: A (b x b symmetric) -> diag, Q columns =
// eigenvectors.  Round-robin pairing, b/2 disjoint rotations per round.
// Rotations below 2.2e-16 ||A||_F are skipped (they cannot move an
// eigenvalue by more than rounding); pairs with both indices >= nimp (trailing
// guard columns) are only reduced to 1e-8 ||A||_F.  sflag[0] returns sweeps.
__device__ void jacobi_eig(double* A, double* Q, int b, int lds, double* cs, int* pq, int* sflag, int nimp) {
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ double fro_part[32];
  double f = 0.0;
  for (int e = tid; e < b * b; e += nt) {
    const int i = e / b, j = e % b;
    Q[i * lds + j] = (i == j) ? 1.0 : 0.0;
    const double v = A[i * lds + j];
    f = fma(v, v, f);
  }
  f = warp_sum(f);
  if ((tid & 31) == 0) fro_part[tid >> 5] = f;
  __syncthreads();
  double fro = 0.0;
  for (int w = 0; w < (int)(nt >> 5); ++w) fro += fro_part[w];
  fro = sqrt(fro);
  const double thr_imp = PDSDP_JAC_TOL_IMP * fro, thr_guard = PDSDP_JAC_TOL_GUARD * fro;
  if (tid == 0) sflag[0] = 0;
  if (b == 1) { __syncthreads(); return; }
  const int bb = b + (b & 1);
  const int np = bb / 2;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (tid == 0) sflag[1] = 0;
    __syncthreads();
    for (int round = 0; round < bb - 1; ++round) {
      for (int j = tid; j < np; j += nt) {
        int t0 = j, t1 = bb - 1 - j;
        int p = (t0 == 0) ? 0 : 1 + (t0 - 1 + round) % (bb - 1);
        int q = 1 + (t1 - 1 + round) % (bb - 1);
        if (p > q) { int tmp = p; p = q; q = tmp; }
        double c = 1.0, s = 0.0;
        if (q < b) {
          const double apq = A[p * lds + q];
          const double thr = (p < nimp) ? thr_imp : thr_guard;
          if (fabs(apq) > thr) {
            const double tau = (A[q * lds + q] - A[p * lds + p]) / (2.0 * apq);
            double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            if (!isfinite(tau)) t = 0.0;
            c = rsqrt(1.0 + t * t);
            s = t * c;
            if (t != 0.0) sflag[1] = 1;
          }
        }
        cs[2 * j] = c; cs[2 * j + 1] = s;
        pq[2 * j] = p; pq[2 * j + 1] = q;
      }
      __syncthreads();
      // rows p, q  <-  J^T A
      for (int e = tid; e < np * b; e += nt) {
        int j = e / b, col = e % b;
        int p = pq[2 * j], q = pq[2 * j + 1];
        double s = cs[2 * j + 1];
        if (q >= b || s == 0.0) continue;
        double c = cs[2 * j];
        double ap = A[p * lds + col], aq = A[q * lds + col];
        A[p * lds + col] = c * ap - s * aq;
        A[q * lds + col] = s * ap + c * aq;
      }
      __syncthreads();
      // columns p, q  <-  A J ;  Q <- Q J
      for (int e = tid; e < np * b; e += nt) {
        int j = e / b, row = e % b;
        int p = pq[2 * j], q = pq[2 * j + 1];
        double s = cs[2 * j + 1];
        if (q >= b || s == 0.0) continue;
        double c = cs[2 * j];
        double ap = A[row * lds + p], aq = A[row * lds + q];
        double np_ = c * ap - s * aq, nq_ = s * ap + c * aq;
        if (row == p) nq_ = 0.0;
        if (row == q) np_ = 0.0;
        A[row * lds + p] = np_;
        A[row * lds + q] = nq_;
        double qp = Q[row * lds + p], qq = Q[row * lds + q];
        Q[row * lds + p] = c * qp - s * qq;
        Q[row * lds + q] = s * qp + c * qq;
      }
      __syncthreads();
    }
    if (tid == 0) sflag[0] = sweep + 1;
    int f = sflag[1];
    __syncthreads();
    if (!f) break;
  }
}

// Descending order of the diagonal of A: perm[rank] = index (ties by index).
__device__ void sort_desc(const double* A, int b, int lds, double* theta, int* perm) {
  // every caller passes shared-memory workspaces: LDS/STS, not generic loads
  A = as_shared(A);
  theta = as_shared(theta);
  perm = as_shared(perm);
  for (int i = threadIdx.x; i < b; i += blockDim.x) {
    double ti = A[i * lds + i];
    int rank = 0;
    bool bad = !isfinite(ti);
    for (int j = 0; j < b; ++j) {
      double tj = A[j * lds + j];
      if (!isfinite(tj)) bad = true;
      if (tj > ti || (tj == ti && j < i)) ++rank;
    }
    if (bad) rank = i;
    perm[rank] = i;
    theta[rank] = ti;
  }
  __syncthreads();
}

// C = A * B   (a x k) * (k x c), all shared memory, leading dims given.
__device__ void sm_gemm(const double* A, int lda, const double* B, int ldb, double* C, int ldc,
                        int a, int k, int c) {
  // every caller passes shared-memory workspaces: LDS/STS, not generic loads
  A = as_shared(A);
  B = as_shared(B);
  C = as_shared(C);
  for (int e = threadIdx.x; e < a * c; e += blockDim.x) {
    int i = e / c, j = e % c;
    double s = 0.0;
    for (int t = 0; t < k; ++t) s += A[i * lda + t] * B[t * ldb + j];
    C[i * ldc + j] = s;
  }
  __syncthreads();
}


// ---------------------------------------------------------------------------
// Single-warp variants (warp 0 only; the rest of the block waits at a
// __syncthreads): the b x b problems are tiny, so block-wide barriers
// (hundreds per pass) cost far more than the arithmetic.

// In-place scaled Cholesky (see chol_scaled); returns false on breakdown.
__device__ bool chol_scaled_warp(double* G, int b, int lds, double* dsc) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < b; i += 32) {
    const double g = G[i * lds + i];
    dsc[i] = (g > 0.0 && isfinite(g)) ? rsqrt(g) : 0.0;
  }
  __syncwarp();
  for (int e = lane; e < b * b; e += 32) {
    const int i = e / b, j = e % b;
    G[i * lds + j] = (j <= i) ? G[i * lds + j] * dsc[i] * dsc[j] : 0.0;
  }
  __syncwarp();
  for (int j = 0; j < b; ++j) {
    double d = G[j * lds + j];
    if (!(d > 1e-28)) return false;
    d = sqrt(d);
    __syncwarp();
    for (int i = j + 1 + lane; i < b; i += 32) G[i * lds + j] /= d;
    if (lane == 0) G[j * lds + j] = d;
    __syncwarp();
    const int rem = b - j - 1;
    for (int e = lane; e < rem * rem; e += 32) {
      const int i = j + 1 + e / rem, k = j + 1 + e % rem;
      if (k <= i) G[i * lds + k] -= G[i * lds + j] * G[k * lds + j];
    }
    __syncwarp();
  }
  return true;
}

// Cyclic two-sided Jacobi in one warp; rotations below 2.2e-16 ||A||_F are
// skipped (they cannot move an eigenvalue by more than rounding).  Returns
// the number of sweeps.
__device__ int jacobi_eig_warp(double* A, double* Q, int b, int lds, double* cs, int* pq) {
  const int lane = threadIdx.x & 31;
  double f = 0.0;
  for (int e = lane; e < b * b; e += 32) {
    const int i = e / b, j = e % b;
    Q[i * lds + j] = (i == j) ? 1.0 : 0.0;
    const double v = A[i * lds + j];
    f = fma(v, v, f);
  }
  f = warp_sum(f);
  const double thr = 2.2e-16 * sqrt(f);
  __syncwarp();
  if (b == 1) return 0;
  const int bb = b + (b & 1), np = bb / 2;
  int sweeps = 0;
  for (int sweep = 0; sweep < 30; ++sweep) {
    bool any = false;
    for (int round = 0; round < bb - 1; ++round) {
      for (int j = lane; j < np; j += 32) {
        const int t0 = j, t1 = bb - 1 - j;
        int p = (t0 == 0) ? 0 : 1 + (t0 - 1 + round) % (bb - 1);
        int q = 1 + (t1 - 1 + round) % (bb - 1);
        if (p > q) { const int tmp = p; p = q; q = tmp; }
        double c = 1.0, sn = 0.0;
        if (q < b) {
          const double apq = A[p * lds + q];
          if (fabs(apq) > thr) {
            const double tau = (A[q * lds + q] - A[p * lds + p]) / (2.0 * apq);
            double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            if (!isfinite(tau)) t = 0.0;
            c = rsqrt(1.0 + t * t);
            sn = t * c;
            if (t != 0.0) any = true;
          }
        }
        cs[2 * j] = c; cs[2 * j + 1] = sn;
        pq[2 * j] = p; pq[2 * j + 1] = q;
      }
      __syncwarp();
      for (int e = lane; e < np * b; e += 32) {
        const int j = e / b, col = e % b;
        const double sn = cs[2 * j + 1];
        const int p = pq[2 * j], q = pq[2 * j + 1];
        if (q >= b || sn == 0.0) continue;
        const double c = cs[2 * j];
        const double ap = A[p * lds + col], aq = A[q * lds + col];
        A[p * lds + col] = c * ap - sn * aq;
        A[q * lds + col] = sn * ap + c * aq;
      }
      __syncwarp();
      for (int e = lane; e < np * b; e += 32) {
        const int j = e / b, row = e % b;
        const double sn = cs[2 * j + 1];
        const int p = pq[2 * j], q = pq[2 * j + 1];
        if (q >= b || sn == 0.0) continue;
        const double c = cs[2 * j];
        const double ap = A[row * lds + p], aq = A[row * lds + q];
        double np_ = c * ap - sn * aq, nq_ = sn * ap + c * aq;
        if (row == p) nq_ = 0.0;
        if (row == q) np_ = 0.0;
        A[row * lds + p] = np_;
        A[row * lds + q] = nq_;
        const double qp = Q[row * lds + p], qq = Q[row * lds + q];
        Q[row * lds + p] = c * qp - sn * qq;
        Q[row * lds + q] = sn * qp + c * qq;
      }
      __syncwarp();
    }
    ++sweeps;
    if (!__any_sync(0xffffffffu, any)) break;
  }
  return sweeps;
}


// ---------------------------------------------------------------------------
// One-barrier-per-step variants (all threads of the CTA).

// Scaled Cholesky with a single __syncthreads per column: step j updates the
// trailing columns from the (final) column j without normalising it; the
// normalisation happens once at the end.  Same contract as chol_scaled.
__device__ bool chol_scaled_1s(double* G, int b, int lds, double* dsc) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < b; i += nt) {
    const double g = G[i * lds + i];
    dsc[i] = (g > 0.0 && isfinite(g)) ? rsqrt(g) : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < b * b; e += nt) {
    const int i = e / b, j = e % b;
    G[i * lds + j] = (j <= i) ? G[i * lds + j] * dsc[i] * dsc[j] : 0.0;
  }
  __syncthreads();
  for (int j = 0; j < b; ++j) {
    const double djj = G[j * lds + j];
    if (!(djj > 1e-28)) { __syncthreads(); return false; }
    const double inv = 1.0 / djj;
    const int rem = b - j - 1;
    for (int e = tid; e < rem * rem; e += nt) {
      const int i = j + 1 + e / rem, k = j + 1 + e % rem;
      if (k <= i) G[i * lds + k] -= G[i * lds + j] * G[k * lds + j] * inv;
    }
    __syncthreads();
  }
  for (int e = tid; e < b * b; e += nt) {
    const int i = e / b, j = e % b;
    if (j <= i) {
      const double sj = sqrt(G[j * lds + j]);
      if (i != j) G[i * lds + j] = G[i * lds + j] / sj;
    }
  }
  __syncthreads();
  for (int j = tid; j < b; j += nt) G[j * lds + j] = sqrt(G[j * lds + j]);
  __syncthreads();
  return true;
}

// X = L^{-1} (lower) by row elimination, one barrier per row.
__device__ void tri_inv_lower_1s(const double* L, double* X, int b, int lds) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < b * b; e += nt) X[(e / b) * lds + (e % b)] = (e / b == e % b) ? 1.0 : 0.0;
  __syncthreads();
  for (int kk = 0; kk < b - 1; ++kk) {
    const double lkk = L[kk * lds + kk];
    const int rows = b - kk - 1, cols = kk + 1;
    for (int e = tid; e < rows * cols; e += nt) {
      const int i = kk + 1 + e / cols, c = e % cols;
      X[i * lds + c] -= L[i * lds + kk] * (X[kk * lds + c] / lkk);
    }
    __syncthreads();
  }
  for (int e = tid; e < b * b; e += nt) {
    const int i = e / b, c = e % b;
    X[i * lds + c] = (c <= i) ? X[i * lds + c] / L[i * lds + i] : 0.0;
  }
  __syncthreads();
}

__device__ __forceinline__ int jac_partner(int i, int t, int bb) {
  if (i == 0) return 1 + (bb - 2 + t) % (bb - 1);
  const int u = 1 + (((i - 1 - t) % (bb - 1)) + (bb - 1)) % (bb - 1);
  const int v = bb - 1 - u;
  return (v == 0) ? 0 : 1 + (v - 1 + t) % (bb - 1);
}

__device__ __forceinline__ void jac_rot(double app, double aqq, double apq, double thr, double& c, double& s) {
  c = 1.0; s = 0.0;
  if (fabs(apq) > thr) {
    const double tau = (aqq - app) / (2.0 * apq);
    double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
    if (!isfinite(tau)) t = 0.0;
    c = rsqrt(1.0 + t * t);
    s = t * c;
  }
}

// Cyclic two-sided Jacobi with one __syncthreads per round: every thread
// forms its elements of J^T A J and Q J in one pass (ping-pong buffers), and
// the threads owning the entries of next round's pairs form next round's
// rotations directly.  Same thresholds as jacobi_eig.  On return *Aout / *Qout
// point at the buffers holding the diagonalised matrix and the eigenvectors;
// sflag[0] = sweeps.
__device__ void jacobi_eig_1s(double* A, double* A2, double* Q, double* Q2, int b, int lds, double* csn,
                              int* sflag, int nimp, double** Aout, double** Qout) {
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ double fro_part[32];
  double f = 0.0;
  for (int e = tid; e < b * b; e += nt) {
    const int i = e / b, j = e % b;
    Q[i * lds + j] = (i == j) ? 1.0 : 0.0;
    const double v = A[i * lds + j];
    f = fma(v, v, f);
  }
  f = warp_sum(f);
  if ((tid & 31) == 0) fro_part[tid >> 5] = f;
  __syncthreads();
  double fro = 0.0;
  for (int w = 0; w < (int)(nt >> 5); ++w) fro += fro_part[w];
  fro = sqrt(fro);
  const double thr_imp = PDSDP_JAC_TOL_IMP * fro, thr_guard = PDSDP_JAC_TOL_GUARD * fro;
  *Aout = A; *Qout = Q;
  if (tid == 0) sflag[0] = 0;
  if (b == 1) { __syncthreads(); return; }
  const int bb = b + (b & 1);
  // rotation tables indexed by the smaller index p of a pair: csn[2][2*BMAX]
  double* cur = csn;
  double* nxt = csn + 2 * PDSDP_BMAX;
  // rotations of round 0
  int any = 0;
  for (int p = tid; p < b; p += nt) {
    const int q = jac_partner(p, 0, bb);
    double c = 1.0, sn = 0.0;
    if (p < q && q < b) jac_rot(A[p * lds + p], A[q * lds + q], A[p * lds + q], (p < nimp) ? thr_imp : thr_guard, c, sn);
    if (sn != 0.0) any = 1;
    cur[2 * p] = c; cur[2 * p + 1] = sn;
  }
  any = __syncthreads_or(any);
  double *Ac = A, *An = A2, *Qc = Q, *Qn = Q2;
  int sweeps = 0, sweep_any = any;
  for (int it = 0; it < 40 * (bb - 1); ++it) {
    const int t = it % (bb - 1);
    const int t1 = (t + 1) % (bb - 1);
    int nany = 0;
    for (int e = tid; e < 2 * b * b; e += nt) {
      const bool isQ = e >= b * b;
      const int ee = isQ ? e - b * b : e;
      const int i = ee / b, j = ee % b;
      // column coefficients (J[.][j])
      const int pj = jac_partner(j, t, bb);
      double cj0 = 1.0, cj1 = 0.0;       // J[j][j], J[pj][j]
      if (pj < b) {
        const int pp = min(j, pj);
        const double c = cur[2 * pp], sn = cur[2 * pp + 1];
        cj0 = c;
        cj1 = (j == pp) ? -sn : sn;
      }
      if (isQ) {
        const double v = cj0 * Qc[i * lds + j] + ((pj < b) ? cj1 * Qc[i * lds + pj] : 0.0);
        Qn[i * lds + j] = v;
        continue;
      }
      const int pi = jac_partner(i, t, bb);
      double ri0 = 1.0, ri1 = 0.0;       // J[i][i], J[pi][i]
      if (pi < b) {
        const int pp = min(i, pi);
        const double c = cur[2 * pp], sn = cur[2 * pp + 1];
        ri0 = c;
        ri1 = (i == pp) ? -sn : sn;
      }
      auto elem = [&](int ii, int jj) {
        const int pii = jac_partner(ii, t, bb), pjj = jac_partner(jj, t, bb);
        double a0 = 1.0, a1 = 0.0, b0 = 1.0, b1 = 0.0;
        if (pii < b) { const int pp = min(ii, pii); a0 = cur[2 * pp]; a1 = (ii == pp) ? -cur[2 * pp + 1] : cur[2 * pp + 1]; }
        if (pjj < b) { const int pp = min(jj, pjj); b0 = cur[2 * pp]; b1 = (jj == pp) ? -cur[2 * pp + 1] : cur[2 * pp + 1]; }
        double v = a0 * (b0 * Ac[ii * lds + jj] + ((pjj < b) ? b1 * Ac[ii * lds + pjj] : 0.0));
        if (pii < b) v += a1 * (b0 * Ac[pii * lds + jj] + ((pjj < b) ? b1 * Ac[pii * lds + pjj] : 0.0));
        if (pii == jj && pii < b) {
          const int pp = min(ii, pii);
          if (cur[2 * pp + 1] != 0.0) v = 0.0;       // the rotated pair is annihilated
        }
        return v;
      };
      (void)ri0; (void)ri1;
      const double v = elem(i, j);
      An[i * lds + j] = v;
      // owner of next round's pair (p', q') with p' = i < q' = j forms its rotation
      const int q1 = jac_partner(i, t1, bb);
      if (j == q1 && i < j) {
        const double app = elem(i, i), aqq = elem(j, j);
        double c, sn;
        jac_rot(app, aqq, v, (i < nimp) ? thr_imp : thr_guard, c, sn);
        nxt[2 * i] = c; nxt[2 * i + 1] = sn;
        if (sn != 0.0) nany = 1;
      }
    }
    // indices whose next partner is the dummy (odd b) or >= b: no rotation
    for (int p = tid; p < b; p += nt) {
      const int q = jac_partner(p, t1, bb);
      if (q >= b && p < q) { nxt[2 * p] = 1.0; nxt[2 * p + 1] = 0.0; }
    }
    nany = __syncthreads_or(nany);
    { double* tmp = Ac; Ac = An; An = tmp; tmp = Qc; Qc = Qn; Qn = tmp; tmp = cur; cur = nxt; nxt = tmp; }
    if (t == bb - 2) {                  // a full sweep finished
      ++sweeps;
      if (!sweep_any) break;
      sweep_any = nany;                 // rotations already decided for the next sweep's round 0
    } else {
      sweep_any |= nany;
    }
  }
  *Aout = Ac; *Qout = Qc;
  if (tid == 0) sflag[0] = sweeps;
  __syncthreads();
}


// Fast, deterministic FP64 reciprocal / reciprocal square root: hardware
// approximation + Newton steps (full double accuracy to within a few ulp).
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-x, r, 2.0);
  r = r * fma(-x, r, 2.0);
  return r;
}
__device__ __forceinline__ double fast_rsqrt(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-0.5 * x * r, r, 1.5);
  r = r * fma(-0.5 * x * r, r, 1.5);
  return r;
}

// Same contract and arithmetic as chol_scaled_1s, with a fixed thread map:
// thread (i, p) owns row i and the columns k = j+1+p, j+1+p+P, ... of each
// step j (P = blockDim / b parts per row): no per-element index division and
// one barrier per step.
__device__ bool chol_scaled_rows(double* G, int b, int lds, double* dsc) {
  // every caller passes shared-memory workspaces: LDS/STS, not generic loads
  G = as_shared(G);
  dsc = as_shared(dsc);
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < b; i += nt) {
    const double g = G[i * lds + i];
    dsc[i] = (g > 0.0 && isfinite(g)) ? rsqrt(g) : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < b * b; e += nt) {
    const int i = e / b, j = e % b;
    G[i * lds + j] = (j <= i) ? G[i * lds + j] * dsc[i] * dsc[j] : 0.0;
  }
  __syncthreads();
  const int P = max(1, nt / b);
  const int ri = tid / P, pp = tid - ri * P;
  for (int j = 0; j < b; ++j) {
    const double djj = G[j * lds + j];
    if (!(djj > 1e-28)) { __syncthreads(); return false; }
    if (ri < b && ri > j) {
      const double gij = G[ri * lds + j] * fast_rcp(djj);
      double* Gi = G + ri * lds;
      for (int k = j + 1 + pp; k <= ri; k += P) Gi[k] = fma(-gij, G[k * lds + j], Gi[k]);
    }
    __syncthreads();
  }
  for (int e = tid; e < b * b; e += nt) {
    const int i = e / b, j = e % b;
    if (j < i) G[i * lds + j] = G[i * lds + j] / sqrt(G[j * lds + j]);
  }
  __syncthreads();
  for (int j = tid; j < b; j += nt) G[j * lds + j] = sqrt(G[j * lds + j]);
  __syncthreads();
  return true;
}

// X = L^{-1} (lower) as tri_inv_lower_1s, with the fixed (row, part) thread map.
__device__ void tri_inv_lower_rows(const double* L, double* X, int b, int lds) {
  // every caller passes shared-memory workspaces: LDS/STS, not generic loads
  L = as_shared(L);
  X = as_shared(X);
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < b * b; e += nt) X[(e / b) * lds + (e % b)] = (e / b == e % b) ? 1.0 : 0.0;
  __syncthreads();
  const int P = max(1, nt / b);
  const int ri = tid / P, pp = tid - ri * P;
  for (int kk = 0; kk < b - 1; ++kk) {
    if (ri < b && ri > kk) {
      const double f = L[ri * lds + kk] * fast_rcp(L[kk * lds + kk]);
      double* Xi = X + ri * lds;
      const double* Xk = X + kk * lds;
      for (int c = pp; c <= kk; c += P) Xi[c] = fma(-f, Xk[c], Xi[c]);
    }
    __syncthreads();
  }
  for (int e = tid; e < b * b; e += nt) {
    const int i = e / b, c = e % b;
    X[i * lds + c] = (c <= i) ? X[i * lds + c] / L[i * lds + i] : 0.0;
  }
  __syncthreads();
}

// Two-barrier-per-round cyclic Jacobi: (1) one thread per pair forms the
// rotation from a precomputed pairing table, (2) every thread forms its
// elements of J^T A J and Q J in one pass into ping-pong buffers.  The
// rotation only needs to be an exact orthogonal matrix (c^2 + s^2 = 1 to
// rounding); residual off-diagonals are removed by later sweeps.
// Thresholds as jacobi_eig.  tab: >= (bb-1) * bb ints of scratch.
__device__ void jacobi_eig2(double* A, double* A2, double* Q, double* Q2, int b, int lds, double* cs,
                            int* tab, int* sflag, int nimp, double** Aout, double** Qout) {
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ double fro_part[32];
  double f = 0.0;
  for (int e = tid; e < b * b; e += nt) {
    const int i = e / b, j = e % b;
    Q[i * lds + j] = (i == j) ? 1.0 : 0.0;
    const double v = A[i * lds + j];
    f = fma(v, v, f);
  }
  f = warp_sum(f);
  if ((tid & 31) == 0) fro_part[tid >> 5] = f;
  const int bb = b + (b & 1), np = bb / 2, R = bb - 1;
  // pairing table: tab[t * bb + i] = partner of i in round t (>= b: none)
  for (int e = tid; e < R * bb; e += nt) {
    const int t = e / bb, j = e % bb;
    if (j < np) {
      const int t0 = j, t1 = bb - 1 - j;
      const int p = (t0 == 0) ? 0 : 1 + (t0 - 1 + t) % R;
      const int q = 1 + (t1 - 1 + t) % R;
      tab[t * bb + p] = q;
      tab[t * bb + q] = p;
    }
  }
  __syncthreads();
  double fro = 0.0;
  for (int w = 0; w < (int)(nt >> 5); ++w) fro += fro_part[w];
  fro = sqrt(fro);
  const double thr_imp = PDSDP_JAC_TOL_IMP * fro, thr_guard = PDSDP_JAC_TOL_GUARD * fro;
  double *Ac = A, *An = A2, *Qc = Q, *Qn = Q2;
  int sweeps = 0;
  if (b > 1) {
    for (int sweep = 0; sweep < 40; ++sweep) {
      int any = 0;
      for (int t = 0; t < R; ++t) {
        const int* pt = tab + t * bb;
        // (1) rotations, indexed by the smaller index of each pair
        for (int p = tid; p < b; p += nt) {
          const int q = pt[p];
          if (p < q) {
            double c = 1.0, sn = 0.0;
            if (q < b) {
              const double apq = Ac[p * lds + q];
              if (fabs(apq) > ((p < nimp) ? thr_imp : thr_guard)) {
                const double tau = (Ac[q * lds + q] - Ac[p * lds + p]) * fast_rcp(2.0 * apq);
                const double at = fabs(tau);
                double tt;
                if (at < 1e150) {
                  const double u = fma(tau, tau, 1.0);
                  tt = fast_rcp(at + u * fast_rsqrt(u));
                } else {
                  tt = 0.5 * fast_rcp(at);
                }
                tt = (tau >= 0.0) ? tt : -tt;
                if (!isfinite(tau)) tt = 0.0;
                c = fast_rsqrt(fma(tt, tt, 1.0));
                sn = tt * c;
                if (sn != 0.0) any = 1;
              }
            }
            cs[2 * p] = c;
            cs[2 * p + 1] = sn;
          }
        }
        __syncthreads();
        // (2) A' = J^T A J and Q' = Q J, element-wise
        for (int e = tid; e < 2 * b * b; e += nt) {
          const bool isQ = e >= b * b;
          const int ee = isQ ? e - b * b : e;
          const int i = ee / b, j = ee % b;
          const int pj = pt[j];
          double b0 = 1.0, b1 = 0.0;
          if (pj < b) {
            const int pp = min(j, pj);
            b0 = cs[2 * pp];
            b1 = (j == pp) ? -cs[2 * pp + 1] : cs[2 * pp + 1];
          }
          if (isQ) {
            double v = b0 * Qc[i * lds + j];
            if (pj < b) v = fma(b1, Qc[i * lds + pj], v);
            Qn[i * lds + j] = v;
            continue;
          }
          const int pi = pt[i];
          double a0 = 1.0, a1 = 0.0;
          if (pi < b) {
            const int pp = min(i, pi);
            a0 = cs[2 * pp];
            a1 = (i == pp) ? -cs[2 * pp + 1] : cs[2 * pp + 1];
          }
          double v = b0 * Ac[i * lds + j];
          if (pj < b) v = fma(b1, Ac[i * lds + pj], v);
          v *= a0;
          if (pi < b) {
            double w = b0 * Ac[pi * lds + j];
            if (pj < b) w = fma(b1, Ac[pi * lds + pj], w);
            v = fma(a1, w, v);
            if (pi == j && cs[2 * min(i, pi) + 1] != 0.0) v = 0.0;   // annihilated pair
          }
          An[i * lds + j] = v;
        }
        __syncthreads();
        { double* tp = Ac; Ac = An; An = tp; tp = Qc; Qc = Qn; Qn = tp; }
      }
      ++sweeps;
      if (!__syncthreads_or(any)) break;
    }
  }
  *Aout = Ac; *Qout = Qc;
  if (tid == 0) sflag[0] = sweeps;
  __syncthreads();
}


// Second-order finish of a nearly diagonal A, in place of further Jacobi
// sweeps: with every off-diagonal entry small against its diagonal gap,
//   U = I + K,  K_ij = a_ij / (a_jj - a_ii)  (i != j),  columns normalised,
//   Q <- Q U,   A <- diag(a_jj + sum_i a_ij K_ij),
// leaves eigenvector errors O(a_ij^2 / gap) (first-order perturbation theory;
// U is orthonormal to O(K^2)).  Applied only when that is below a tenth of
// the pair's rotation threshold, so the result meets the same tolerance as
// the sweeps it replaces; otherwise returns false and changes nothing.  Three
// barriers instead of b - 1 rounds of two.  An / Qn receive the new A / Q.
#ifndef PDSDP_JAC_PERTURB
#define PDSDP_JAC_PERTURB 1
#endif
__device__ bool jacobi_perturb_finish(const double* Ac, const double* Qc, double* An, double* Qn, int b, int lds,
                                      int nimp, double thr_imp, double thr_guard, double* cs) {
  const int tid = threadIdx.x, nt = blockDim.x;
  int bad = 0;
  for (int e = tid; e < b * b; e += nt) {
    const int i = e / b, j = e - (e / b) * b;
    double k = 0.0;
    if (i != j) {
      const int lo_ = min(i, j), hi_ = max(i, j);
      const double a = Ac[lo_ * lds + hi_];
      const double gap = Ac[j * lds + j] - Ac[i * lds + i];
      const double thr = (lo_ < nimp) ? thr_imp : thr_guard;
      if (fabs(a) <= 1e-3 * fabs(gap)) {
        k = a / gap;
        if (fabs(a) > thr && !(a * a <= 0.1 * thr * fabs(gap))) bad = 1;
      } else if (fabs(a) > thr) {
        bad = 1;
      }
    }
    An[i * lds + j] = k;
  }
  if (__syncthreads_or(bad)) return false;
  double* nrm = cs;
  double* lam = cs + PDSDP_BMAX;
  if (tid < b) {
    const int j = tid;
    double s2 = 1.0, l = Ac[j * lds + j];
    for (int i = 0; i < b; ++i) {
      if (i == j) continue;
      const double k = An[i * lds + j];
      s2 = fma(k, k, s2);
      l = fma(k, Ac[min(i, j) * lds + max(i, j)], l);
    }
    nrm[j] = 1.0 / sqrt(s2);
    lam[j] = l;
  }
  __syncthreads();
  for (int e = tid; e < b * b; e += nt) {
    const int i = e / b, j = e - (e / b) * b;
    double acc = Qc[i * lds + j];
    for (int l = 0; l < b; ++l)
      if (l != j) acc = fma(Qc[i * lds + l], An[l * lds + j], acc);
    Qn[i * lds + j] = acc * nrm[j];
  }
  __syncthreads();
  for (int e = tid; e < b * b; e += nt) {
    const int i = e / b, j = e - (e / b) * b;
    An[i * lds + j] = (i == j) ? lam[i] : 0.0;
  }
  __syncthreads();
  return true;
}

// Parallel-order cyclic Jacobi for the b x b (b <= 64) projected matrix,
// block-wide.  Same contract and rotations as jacobi_eig2, restructured for
// latency: per round, thread p (< b) writes the row coefficients (a0, a1) of
// index p -- an unpaired index is its own partner with (1, 0) -- so the
// element update  A' = J^T A J,  Q' = Q J  is branch-free; thread (i, j0)
// owns row i and columns j0, j0+8, ... (no index division); a sweep starts
// only if some off-diagonal entry is above its threshold (no trailing no-op
// sweep).
__device__ void jacobi_eig3(double* A, double* A2, double* Q, double* Q2, int b, int lds, double* cs,
                            int* tab, int* sflag, int nimp, double** Aout, double** Qout) {
  // every caller passes shared-memory workspaces: LDS/STS, not generic loads
  A = as_shared(A);
  A2 = as_shared(A2);
  Q = as_shared(Q);
  Q2 = as_shared(Q2);
  cs = as_shared(cs);
  tab = as_shared(tab);
  sflag = as_shared(sflag);
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ double fro_part[32];
  double f = 0.0;
  for (int e = tid; e < b * b; e += nt) {
    const int i = e / b, j = e % b;
    Q[i * lds + j] = (i == j) ? 1.0 : 0.0;
    const double v = A[i * lds + j];
    f = fma(v, v, f);
  }
  f = warp_sum(f);
  if ((tid & 31) == 0) fro_part[tid >> 5] = f;
  const int bb = b + (b & 1), np = bb / 2, R = bb - 1;
  for (int e = tid; e < R * bb; e += nt) {
    const int t = e / bb, j = e % bb;
    if (j < np) {
      const int t0 = j, t1 = bb - 1 - j;
      const int p = (t0 == 0) ? 0 : 1 + (t0 - 1 + t) % R;
      const int q = 1 + (t1 - 1 + t) % R;
      tab[t * bb + p] = (q < b) ? q : p;
      tab[t * bb + q] = (p < b) ? p : q;
    }
  }
  __syncthreads();
  double fro = 0.0;
  for (int w = 0; w < (int)(nt >> 5); ++w) fro += fro_part[w];
  fro = sqrt(fro);
  const double thr_imp = PDSDP_JAC_TOL_IMP * fro, thr_guard = PDSDP_JAC_TOL_GUARD * fro;
  double* c0a = cs;                 // a0 per index
  double* c1a = cs + PDSDP_BMAX;    // a1 per index (signed)
  double *Ac = A, *An = A2, *Qc = Q, *Qn = Q2;
  const int ri = tid >> 3, cj = tid & 7;    // first row and first column of this thread
  const int rstep = nt >> 3;
  int sweeps = 0;
  if (b > 1) {
    for (int sweep = 0; sweep < 40; ++sweep) {
      // any off-diagonal entry above its threshold?
      int need = 0;
      for (int i = ri; i < b; i += rstep)
        for (int j = cj; j < b; j += 8)
          if (j > i && fabs(Ac[i * lds + j]) > ((i < nimp) ? thr_imp : thr_guard)) need = 1;
      if (!__syncthreads_or(need)) break;
      if (PDSDP_JAC_PERTURB && jacobi_perturb_finish(Ac, Qc, An, Qn, b, lds, nimp, thr_imp, thr_guard, cs)) {
        double* tp = Ac; Ac = An; An = tp; tp = Qc; Qc = Qn; Qn = tp;
        ++sweeps;
        break;
      }
      for (int t = 0; t < R; ++t) {
        Ac = as_shared(Ac); An = as_shared(An); Qc = as_shared(Qc); Qn = as_shared(Qn);
        const int* pt = tab + t * bb;
        int rot = 0;                    // a non-identity rotation in this round
        // (1) rotation of the pair (p, q), p < q, stored per index
        if (tid < b) {
          const int p = tid, q = pt[p];
          double c = 1.0, sn = 0.0;
          if (q != p) {
            const int lo_ = min(p, q), hi_ = max(p, q);
            const double apq = Ac[lo_ * lds + hi_];
            if (fabs(apq) > ((lo_ < nimp) ? thr_imp : thr_guard)) {
              const double tau = (Ac[hi_ * lds + hi_] - Ac[lo_ * lds + lo_]) * fast_rcp(2.0 * apq);
              const double at = fabs(tau);
              double tt;
              if (at < 1e150) {
                const double u = fma(tau, tau, 1.0);
                tt = fast_rcp(at + u * fast_rsqrt(u));
              } else {
                tt = 0.5 * fast_rcp(at);
              }
              tt = (tau >= 0.0) ? tt : -tt;
              if (!isfinite(tau)) tt = 0.0;
              c = fast_rsqrt(fma(tt, tt, 1.0));
              sn = tt * c;
            }
            // column lo_ -> c*col_lo - s*col_hi ; column hi_ -> s*col_lo + c*col_hi
            c0a[p] = c;
            c1a[p] = (p == lo_) ? -sn : sn;
            rot |= (sn != 0.0);
          } else {
            c0a[p] = 1.0;
            c1a[p] = 0.0;
          }
        }
        // a round of identity rotations leaves A and Q bit-for-bit unchanged: skip it
        if (!__syncthreads_or(rot)) continue;
        // (2) A' = J^T A J and Q' = Q J
        for (int i = ri; i < b; i += rstep) {
          const int pi = pt[i];
          const double a0 = c0a[i], a1 = c1a[i];
          const double* Ar = Ac + i * lds;
          const double* Apr = Ac + pi * lds;
          const double* Qr = Qc + i * lds;
          for (int j = cj; j < b; j += 8) {
            const int pj = pt[j];
            const double b0 = c0a[j], b1 = c1a[j];
            double v = fma(b1, Ar[pj], b0 * Ar[j]);
            const double w = fma(b1, Apr[pj], b0 * Apr[j]);
            v = fma(a1, w, a0 * v);
            if (pj == i && pj != j && b1 != 0.0) v = 0.0;      // annihilated pair
            An[i * lds + j] = v;
            Qn[i * lds + j] = fma(b1, Qr[pj], b0 * Qr[j]);
          }
        }
        __syncthreads();
        { double* tp = Ac; Ac = An; An = tp; tp = Qc; Qc = Qn; Qn = tp; }
      }
      ++sweeps;
    }
  }
  *Aout = Ac; *Qout = Qc;
  if (tid == 0) sflag[0] = sweeps;
  __syncthreads();
}

// Cyclic parallel Jacobi with (pair, pair) block updates.  Same round-robin
// order, rotations and thresholds as jacobi_eig3, but each work item updates
// a whole 2x2 block of A (rows of pair a, columns of pair b; a <= b, the
// mirror block written too) from four loads, and each Q item one row of a
// column pair: a quarter of the shared-memory traffic of the per-element
// form and no per-element partner lookups.  Per round: thread k < np forms
// the rotation of pair k; one barrier; block updates; one barrier.
// scratch: cs >= 4 * PDSDP_BMAX doubles; tab >= PDSDP_BMAX * (PDSDP_BMAX + 2) / 8 + 2 * PDSDP_BMAX ints.
__device__ void jacobi_eig4(double* A, double* A2, double* Q, double* Q2, int b, int lds, double* cs,
                            int* tab, int* sflag, int nimp, double** Aout, double** Qout) {
  // every caller passes shared-memory workspaces: LDS/STS, not generic loads
  A = as_shared(A);
  A2 = as_shared(A2);
  Q = as_shared(Q);
  Q2 = as_shared(Q2);
  cs = as_shared(cs);
  tab = as_shared(tab);
  sflag = as_shared(sflag);
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ double fro_part[32];
  double f = 0.0;
  for (int e = tid; e < b * b; e += nt) {
    const int i = e / b, j = e % b;
    Q[i * lds + j] = (i == j) ? 1.0 : 0.0;
    const double v = A[i * lds + j];
    f = fma(v, v, f);
  }
  f = warp_sum(f);
  if ((tid & 31) == 0) fro_part[tid >> 5] = f;
  const int bb = b + (b & 1), np = bb / 2, R = bb - 1;
  const int nA = np * (np + 1) / 2, nQ = b * np;
  // upper-triangular (a, b) decode of block items
  int* tri = tab;                       // [nA]
  int* plo = tab + PDSDP_BMAX * (PDSDP_BMAX / 2 + 1) / 2 + 8;   // [np] pair lower index
  int* phi = plo + PDSDP_BMAX / 2 + 1;  // [np] pair upper index (-1: none)
  double* pc = cs;                      // [np] cosine
  double* ps = cs + PDSDP_BMAX;         // [np] sine
  for (int a = tid; a < np; a += nt) {
    int base = a * np - a * (a - 1) / 2;
    for (int c = a; c < np; ++c) tri[base + (c - a)] = (a << 8) | c;
  }
  __syncthreads();
  double fro = 0.0;
  for (int w = 0; w < (int)(nt >> 5); ++w) fro += fro_part[w];
  fro = sqrt(fro);
  const double thr_imp = PDSDP_JAC_TOL_IMP * fro, thr_guard = PDSDP_JAC_TOL_GUARD * fro;
  double *Ac = A, *An = A2, *Qc = Q, *Qn = Q2;
  const int ri = tid >> 3, cj = tid & 7, rstep = nt >> 3;
  int sweeps = 0;
  if (b > 1) {
    for (int sweep = 0; sweep < 40; ++sweep) {
      int need = 0;
      for (int i = ri; i < b; i += rstep)
        for (int j = cj; j < b; j += 8)
          if (j > i && fabs(Ac[i * lds + j]) > ((i < nimp) ? thr_imp : thr_guard)) need = 1;
      if (!__syncthreads_or(need)) break;
      if (PDSDP_JAC_PERTURB && jacobi_perturb_finish(Ac, Qc, An, Qn, b, lds, nimp, thr_imp, thr_guard, cs)) {
        double* tp = Ac; Ac = An; An = tp; tp = Qc; Qc = Qn; Qn = tp;
        ++sweeps;
        break;
      }
      for (int t = 0; t < R; ++t) {
        Ac = as_shared(Ac); An = as_shared(An); Qc = as_shared(Qc); Qn = as_shared(Qn);
        // (1) rotation of pair k (round-robin order of jacobi_eig3)
        int rot = 0;                    // a non-identity rotation in this round
        for (int k = tid; k < np; k += nt) {
          const int p = (k == 0) ? 0 : 1 + (k - 1 + t) % R;
          const int q = 1 + (bb - 2 - k + t) % R;
          const int lo_ = min(p, q), hi_ = max(p, q);
          double c = 1.0, sn = 0.0;
          if (hi_ < b) {
            const double apq = Ac[lo_ * lds + hi_];
            if (fabs(apq) > ((lo_ < nimp) ? thr_imp : thr_guard)) {
              const double tau = (Ac[hi_ * lds + hi_] - Ac[lo_ * lds + lo_]) * fast_rcp(2.0 * apq);
              const double at = fabs(tau);
              double tt;
              if (at < 1e150) {
                const double u = fma(tau, tau, 1.0);
                tt = fast_rcp(at + u * fast_rsqrt(u));
              } else {
                tt = 0.5 * fast_rcp(at);
              }
              tt = (tau >= 0.0) ? tt : -tt;
              if (!isfinite(tau)) tt = 0.0;
              c = fast_rsqrt(fma(tt, tt, 1.0));
              sn = tt * c;
            }
          }
          plo[k] = lo_;
          phi[k] = (hi_ < b) ? hi_ : -1;
          pc[k] = c;
          ps[k] = sn;
          rot |= (sn != 0.0);
        }
        // a round of identity rotations leaves A and Q bit-for-bit unchanged: skip it
        if (!__syncthreads_or(rot)) continue;
        // (2) A' = J^T A J by 2x2 blocks, Q' = Q J by row / column pair
        for (int it = tid; it < nA + nQ; it += nt) {
          if (it < nA) {
            const int ab = tri[it], a = ab >> 8, bq = ab & 255;
            const int pa = plo[a], qa = phi[a], pb = plo[bq], qb = phi[bq];
            const double ca = pc[a], sa = ps[a], cb = pc[bq], sb = ps[bq];
            const double a00 = Ac[pa * lds + pb];
            const double a01 = (qb >= 0) ? Ac[pa * lds + qb] : 0.0;
            const double a10 = (qa >= 0) ? Ac[qa * lds + pb] : 0.0;
            const double a11 = (qa >= 0 && qb >= 0) ? Ac[qa * lds + qb] : 0.0;
            // columns: (p, q) -> (c p - s q, s p + c q)
            const double x00 = fma(-sb, a01, cb * a00), x01 = fma(sb, a00, cb * a01);
            const double x10 = fma(-sb, a11, cb * a10), x11 = fma(sb, a10, cb * a11);
            // rows
            const double y00 = fma(-sa, x10, ca * x00), y10 = fma(sa, x00, ca * x10);
            const double y01 = fma(-sa, x11, ca * x01);
            double y11 = fma(sa, x01, ca * x11);
            if (a == bq) {
              // diagonal block: the pair's off-diagonal is annihilated
              An[pa * lds + pa] = y00;
              if (qa >= 0) {
                const double off = (sa != 0.0) ? 0.0 : y01;
                An[pa * lds + qa] = off;
                An[qa * lds + pa] = off;
                An[qa * lds + qa] = y11;
              }
            } else {
              An[pa * lds + pb] = y00; An[pb * lds + pa] = y00;
              if (qb >= 0) { An[pa * lds + qb] = y01; An[qb * lds + pa] = y01; }
              if (qa >= 0) { An[qa * lds + pb] = y10; An[pb * lds + qa] = y10; }
              if (qa >= 0 && qb >= 0) { An[qa * lds + qb] = y11; An[qb * lds + qa] = y11; }
            }
          } else {
            const int e = it - nA, i = e / np, bq = e - i * np;
            const int pb = plo[bq], qb = phi[bq];
            const double cb = pc[bq], sb = ps[bq];
            const double q0 = Qc[i * lds + pb];
            const double q1 = (qb >= 0) ? Qc[i * lds + qb] : 0.0;
            Qn[i * lds + pb] = fma(-sb, q1, cb * q0);
            if (qb >= 0) Qn[i * lds + qb] = fma(sb, q0, cb * q1);
          }
        }
        __syncthreads();
        { double* tp = Ac; Ac = An; An = tp; tp = Qc; Qc = Qn; Qn = tp; }
      }
      ++sweeps;
    }
  }
  *Aout = Ac; *Qout = Qc;
  if (tid == 0) sflag[0] = sweeps;
  __syncthreads();
}

// Same as jacobi_eig2, executed by warp 0 alone (warp-synchronous).
__device__ void jacobi_eig2_warp(double* A, double* A2, double* Q, double* Q2, int b, int lds, double* cs,
                            int* tab, int* sflag, int nimp, double** Aout, double** Qout) {
  const int tid = threadIdx.x & 31, nt = 32;
  double f = 0.0;
  for (int e = tid; e < b * b; e += nt) {
    const int i = e / b, j = e % b;
    Q[i * lds + j] = (i == j) ? 1.0 : 0.0;
    const double v = A[i * lds + j];
    f = fma(v, v, f);
  }
  f = warp_sum(f);
  const int bb = b + (b & 1), np = bb / 2, R = bb - 1;
  // pairing table: tab[t * bb + i] = partner of i in round t (>= b: none)
  for (int e = tid; e < R * bb; e += nt) {
    const int t = e / bb, j = e % bb;
    if (j < np) {
      const int t0 = j, t1 = bb - 1 - j;
      const int p = (t0 == 0) ? 0 : 1 + (t0 - 1 + t) % R;
      const int q = 1 + (t1 - 1 + t) % R;
      tab[t * bb + p] = q;
      tab[t * bb + q] = p;
    }
  }
  __syncwarp();
  const double fro = sqrt(f);
  const double thr_imp = PDSDP_JAC_TOL_IMP * fro, thr_guard = PDSDP_JAC_TOL_GUARD * fro;
  double *Ac = A, *An = A2, *Qc = Q, *Qn = Q2;
  int sweeps = 0;
  if (b > 1) {
    for (int sweep = 0; sweep < 40; ++sweep) {
      int any = 0;
      for (int t = 0; t < R; ++t) {
        const int* pt = tab + t * bb;
        // (1) rotations, indexed by the smaller index of each pair
        for (int p = tid; p < b; p += nt) {
          const int q = pt[p];
          if (p < q) {
            double c = 1.0, sn = 0.0;
            if (q < b) {
              const double apq = Ac[p * lds + q];
              if (fabs(apq) > ((p < nimp) ? thr_imp : thr_guard)) {
                const double tau = (Ac[q * lds + q] - Ac[p * lds + p]) * fast_rcp(2.0 * apq);
                const double at = fabs(tau);
                double tt;
                if (at < 1e150) {
                  const double u = fma(tau, tau, 1.0);
                  tt = fast_rcp(at + u * fast_rsqrt(u));
                } else {
                  tt = 0.5 * fast_rcp(at);
                }
                tt = (tau >= 0.0) ? tt : -tt;
                if (!isfinite(tau)) tt = 0.0;
                c = fast_rsqrt(fma(tt, tt, 1.0));
                sn = tt * c;
                if (sn != 0.0) any = 1;
              }
            }
            cs[2 * p] = c;
            cs[2 * p + 1] = sn;
          }
        }
        __syncwarp();
        // (2) A' = J^T A J and Q' = Q J, element-wise
        for (int e = tid; e < 2 * b * b; e += nt) {
          const bool isQ = e >= b * b;
          const int ee = isQ ? e - b * b : e;
          const int i = ee / b, j = ee % b;
          const int pj = pt[j];
          double b0 = 1.0, b1 = 0.0;
          if (pj < b) {
            const int pp = min(j, pj);
            b0 = cs[2 * pp];
            b1 = (j == pp) ? -cs[2 * pp + 1] : cs[2 * pp + 1];
          }
          if (isQ) {
            double v = b0 * Qc[i * lds + j];
            if (pj < b) v = fma(b1, Qc[i * lds + pj], v);
            Qn[i * lds + j] = v;
            continue;
          }
          const int pi = pt[i];
          double a0 = 1.0, a1 = 0.0;
          if (pi < b) {
            const int pp = min(i, pi);
            a0 = cs[2 * pp];
            a1 = (i == pp) ? -cs[2 * pp + 1] : cs[2 * pp + 1];
          }
          double v = b0 * Ac[i * lds + j];
          if (pj < b) v = fma(b1, Ac[i * lds + pj], v);
          v *= a0;
          if (pi < b) {
            double w = b0 * Ac[pi * lds + j];
            if (pj < b) w = fma(b1, Ac[pi * lds + pj], w);
            v = fma(a1, w, v);
            if (pi == j && cs[2 * min(i, pi) + 1] != 0.0) v = 0.0;   // annihilated pair
          }
          An[i * lds + j] = v;
        }
        __syncwarp();
        { double* tp = Ac; Ac = An; An = tp; tp = Qc; Qc = Qn; Qn = tp; }
      }
      ++sweeps;
      if (!__any_sync(0xffffffffu, any)) break;
    }
  }
  *Aout = Ac; *Qout = Qc;
  if (tid == 0) sflag[0] = sweeps;
  __syncwarp();
}

}  // namespace pdsdp
