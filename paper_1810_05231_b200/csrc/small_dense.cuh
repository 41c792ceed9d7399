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
    int i = fdiv(e, c), j = e - i * c;
    double s = 0.0;
    for (int t = 0; t < k; ++t) s += A[i * lda + t] * B[t * ldb + j];
    C[i * ldc + j] = s;
  }
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

// In-place Cholesky G = L L^T (lower) of an SPD matrix scaled to unit
// diagonal first: G' = D G D, D = diag(G)^-1/2.  On exit G holds L' (lower,
// upper triangle zeroed) and dsc[i] = D_ii.  Returns false on breakdown.
// One __syncthreads per column: step j updates the trailing columns from the
// (final) column j without normalising it; the normalisation happens once at
// the end.  Fixed thread map: thread (i, p) owns row i and the columns
// k = j+1+p, j+1+p+P, ... of each step j (P = blockDim / b parts per row), so
// there is no per-element index division.
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
    const int i = fdiv(e, b), j = e - i * b;
    G[i * lds + j] = (j <= i) ? G[i * lds + j] * dsc[i] * dsc[j] : 0.0;
  }
  __syncthreads();
  const int P = max(1, fdiv(nt, b));
  const int ri = fdiv(tid, P), pp = tid - ri * P;
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
    const int i = fdiv(e, b), j = e - i * b;
    if (j < i) G[i * lds + j] = G[i * lds + j] / sqrt(G[j * lds + j]);
  }
  __syncthreads();
  for (int j = tid; j < b; j += nt) G[j * lds + j] = sqrt(G[j * lds + j]);
  __syncthreads();
  return true;
}

// X = L^{-1} (lower triangular), one barrier per column, with the fixed (row, part) thread map.
__device__ void tri_inv_lower_rows(const double* L, double* X, int b, int lds) {
  // every caller passes shared-memory workspaces: LDS/STS, not generic loads
  L = as_shared(L);
  X = as_shared(X);
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < b * b; e += nt) {
    const int i = fdiv(e, b), j = e - i * b;
    X[i * lds + j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int P = max(1, fdiv(nt, b));
  const int ri = fdiv(tid, P), pp = tid - ri * P;
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
    const int i = fdiv(e, b), c = e - i * b;
    X[i * lds + c] = (c <= i) ? X[i * lds + c] / L[i * lds + i] : 0.0;
  }
  __syncthreads();
}


// Second-order finish of a nearly diagonal A, in place of further Jacobi
// sweeps: with every off-diagonal entry small against its diagonal gap,
//   U = I + K,  K_ij = a_ij / (a_jj - a_ii)  (i != j),  columns normalised,
//   Q <- Q U,   A <- diag(a_jj + sum_i a_ij K_ij),
// leaves eigenvector errors O(a_ij^2 / gap) (first-order perturbation theory).
// K is antisymmetric, so U^T U = I + K^T K: the columns of U are orthogonal
// only up to the off-diagonal entries of K^T K, which are formed explicitly
// (three or more nearly equal eigenvalues make them large while every K_ij
// still passes the entrywise test).  Applied only when the eigenvector error
// is below a tenth of the pair's rotation threshold and every off-diagonal
// entry of K^T K is below PDSDP_JAC_PERTURB_ORTH, so the result meets the
// tolerance of the sweeps it replaces; otherwise returns false (An is
// scratch then, Ac / Qc / Qn are unchanged).  Three barriers instead of b - 1
// rounds of two.  An / Qn receive the new A / Q.
#ifndef PDSDP_JAC_PERTURB
#define PDSDP_JAC_PERTURB 1
#endif
#ifndef PDSDP_JAC_PERTURB_ORTH
#define PDSDP_JAC_PERTURB_ORTH 1e-14
#endif
__device__ bool jacobi_perturb_finish(const double* Ac, const double* Qc, double* An, double* Qn, int b, int lds,
                                      int nimp, double thr_imp, double thr_guard, double* cs) {
  const int tid = threadIdx.x, nt = blockDim.x;
  int bad = 0;
  for (int e = tid; e < b * b; e += nt) {
    const int i = fdiv(e, b), j = e - i * b;
    double k = 0.0;
    if (i != j) {
      const int lo_ = min(i, j), hi_ = max(i, j);
      const double a = Ac[lo_ * lds + hi_];
      const double gap = Ac[j * lds + j] - Ac[i * lds + i];
      const double thr = (lo_ < nimp) ? thr_imp : thr_guard;
      if (a == 0.0) {
        k = 0.0;              // exact zero (e.g. a pair just rotated): nothing to correct, and 0/0 with equal diagonals
      } else if (fabs(a) <= 1e-3 * fabs(gap)) {
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
  // (K^T K)_ij for every column pair: the diagonal gives the column norms,
  // the off-diagonal entries the loss of orthogonality of U
  for (int e = tid; e < b * b; e += nt) {
    const int i = fdiv(e, b), j = e - i * b;
    double g = 0.0;
    for (int l = 0; l < b; ++l) g = fma(An[l * lds + i], An[l * lds + j], g);
    if (i == j) {
      double l_ = Ac[j * lds + j];
      for (int l = 0; l < b; ++l)
        if (l != j) l_ = fma(An[l * lds + j], Ac[min(l, j) * lds + max(l, j)], l_);
      nrm[j] = 1.0 / sqrt(1.0 + g);
      lam[j] = l_;
    } else if (!(fabs(g) <= PDSDP_JAC_PERTURB_ORTH)) {
      bad = 1;
    }
  }
  if (__syncthreads_or(bad)) return false;
  for (int e = tid; e < b * b; e += nt) {
    const int i = fdiv(e, b), j = e - i * b;
    double acc = Qc[i * lds + j];
    for (int l = 0; l < b; ++l)
      if (l != j) acc = fma(Qc[i * lds + l], An[l * lds + j], acc);
    Qn[i * lds + j] = acc * nrm[j];
  }
  __syncthreads();
  for (int e = tid; e < b * b; e += nt) {
    const int i = fdiv(e, b), j = e - i * b;
    An[i * lds + j] = (i == j) ? lam[i] : 0.0;
  }
  __syncthreads();
  return true;
}

// Parallel-order cyclic Jacobi for the b x b (b <= 64) projected matrix,
// block-wide: two-sided rotations in round-robin order from a pairing table
// (tab: >= (bb-1) * bb ints of scratch), ping-pong buffers; on return *Aout /
// *Qout point at the buffers holding the diagonalised matrix and the
// eigenvectors, sflag[0] = sweeps.  Pairs touching an index < nimp are rotated
// down to PDSDP_JAC_TOL_IMP * ||A||_F, the others to PDSDP_JAC_TOL_GUARD.
// Structured for latency: per round, thread p (< b) writes the row coefficients (a0, a1) of
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
    const int i = fdiv(e, b), j = e - i * b;
    Q[i * lds + j] = (i == j) ? 1.0 : 0.0;
    const double v = A[i * lds + j];
    f = fma(v, v, f);
  }
  f = warp_sum(f);
  if ((tid & 31) == 0) fro_part[tid >> 5] = f;
  const int bb = b + (b & 1), np = bb / 2, R = bb - 1;
  for (int e = tid; e < R * bb; e += nt) {
    const int t = fdiv(e, bb), j = e - t * bb;
    if (j < np) {
      const int t0 = j, t1 = bb - 1 - j;
      // 0 <= t0 - 1 + t, t1 - 1 + t < 2 R: one conditional subtraction instead of %
      int pm = t0 - 1 + t, qm = t1 - 1 + t;
      if (pm >= R) pm -= R;
      if (qm >= R) qm -= R;
      const int p = (t0 == 0) ? 0 : 1 + pm;
      const int q = 1 + qm;
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
    const int i = fdiv(e, b), j = e - i * b;
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
          int pm = k - 1 + t, qm = bb - 2 - k + t;       // both in [-1, 2 R): no % needed
          if (pm >= R) pm -= R;
          if (qm >= R) qm -= R;
          const int p = (k == 0) ? 0 : 1 + pm;
          const int q = 1 + qm;
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
            const int e = it - nA, i = fdiv(e, np), bq = e - i * np;
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


}  // namespace pdsdp
