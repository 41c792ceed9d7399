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
__device__ void jacobi_eig(double* A, double* Q, int b, int lds, double* cs, int* pq, int* sflag) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < b * b; e += nt) Q[(e / b) * lds + e % b] = (e / b == e % b) ? 1.0 : 0.0;
  if (b == 1) { __syncthreads(); return; }
  const int bb = b + (b & 1);
  const int np = bb / 2;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (tid == 0) *sflag = 0;
    __syncthreads();
    for (int round = 0; round < bb - 1; ++round) {
      for (int j = tid; j < np; j += nt) {
        int t0 = j, t1 = bb - 1 - j;
        int p = (t0 == 0) ? 0 : 1 + (t0 - 1 + round) % (bb - 1);
        int q = 1 + (t1 - 1 + round) % (bb - 1);
        if (p > q) { int tmp = p; p = q; q = tmp; }
        double c = 1.0, s = 0.0;
        if (q < b) {
          double apq = A[p * lds + q];
          double app = A[p * lds + p], aqq = A[q * lds + q];
          double thr = 1.1102230246251565e-16 * sqrt(fabs(app) * fabs(aqq));
          if (fabs(apq) > thr && fabs(apq) > 1e-300) {
            double tau = (aqq - app) / (2.0 * apq);
            double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            if (!isfinite(tau)) t = 0.0;
            c = rsqrt(1.0 + t * t);
            s = t * c;
            if (t != 0.0) *sflag = 1;
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
    int f = *sflag;
    __syncthreads();
    if (!f) break;
  }
}

// Descending order of the diagonal of A: perm[rank] = index (ties by index).
__device__ void sort_desc(const double* A, int b, int lds, double* theta, int* perm) {
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
  for (int e = threadIdx.x; e < a * c; e += blockDim.x) {
    int i = e / c, j = e % c;
    double s = 0.0;
    for (int t = 0; t < k; ++t) s += A[i * lda + t] * B[t * ldb + j];
    C[i * ldc + j] = s;
  }
  __syncthreads();
}

}  // namespace pdsdp
