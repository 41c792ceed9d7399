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
  const double thr_imp = 1e-14 * fro, thr_guard = 1e-8 * fro;
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

}  // namespace pdsdp
