// One LR-PDHG iteration per thread-block cluster (one cluster per SDP
// instance): the body of the `for k` loop of the reference's
// solve_lr_pd_sdp (pkg/src/pdsdp/lowrank.py:140-150):
//
//   S      = X_k - alpha (C + M^T y_k)                        lowrank.py:97-98
//   X_k+1  = aproj_psd(S, r)  (top r+1 eigenpairs, clip)      symmat.py:229-245
//   y_k+1  = u - alpha proj_box(u/alpha), u = y + alpha M(2X_k+1 - X_k)
//                                                             pdhg.py:185-195
//   residual pieces (dual part + sparse-support primal part)  pdhg.py:198-208
//
// The dense part of the primal residual is finished by residual_kernel
// (residual.cuh) on the whole GPU.  Cross-CTA reductions go through L2 with
// one cluster barrier each (release/acquire at cluster scope); every CTA then
// sums the C partials in the same order, so all CTAs hold bit-identical
// reduced values and run the small dense algebra redundantly.
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"
#include "small_dense.cuh"

namespace cg = cooperative_groups;

namespace pdsdp {

// tolerances of the eigensolver (relative to the spectral scale)
#ifndef PDSDP_TOL_KEEP
#define PDSDP_TOL_KEEP 1e-12   // ARPACK's tol in the reference (symmat.py:33), relative to the spectral scale
#endif
#ifndef PDSDP_TOL_X
#define PDSDP_TOL_X 1e-12      // admissible per-iteration error of X+ (relative to ||X+||_F)
#endif
#define PDSDP_TOL_CERT 1e-8
#define PDSDP_TOL_CLIP 1e-6
#ifndef PDSDP_MMAX
#define PDSDP_MMAX 48          // largest filter degree per pass (slow clustered columns after a rank doubling)
#endif
// largest amplification of a column's contamination the filter may cause:
// CholQR2 re-orthonormalises blocks with condition up to ~1e8, so 1e5 keeps
// a 1000x margin (1e4 .. 3e5 measured within 0.4% of each other on config
// 2, 2% faster than 1e6: profiles/r01s4_spread_cap_sweep.txt)
#ifndef PDSDP_SPREAD_CAP
#define PDSDP_SPREAD_CAP 1e5
#endif
// contamination assumed for the first pass of an iteration (its residuals
// belong to the previous S): enters the spread cap only
#ifndef PDSDP_STALE_EPS
#define PDSDP_STALE_EPS 1e-3
#endif
// the same after an extrapolated start (PDSDP_EXTRAP below): the kept columns
// are then ~1e-8 from their targets and the trailing ones ~1e-5
#ifndef PDSDP_STALE_EPS_X
#define PDSDP_STALE_EPS_X 1e-3
#endif
#ifndef PDSDP_ONEPASS_RR
#define PDSDP_ONEPASS_RR 1
#endif
#ifndef PDSDP_JAC4_MIN
#define PDSDP_JAC4_MIN 24      // smallest block solved by the block-pair Jacobi (jacobi_eig4)
#endif
#ifndef PDSDP_ONEPASS_ETA
#define PDSDP_ONEPASS_ETA 0.5   // entrywise bound b * max|E| of the one-pass test (cond <= (1+eta)/(1-eta))
#endif
// Start block of the eigensolver: the eigenvectors move smoothly from one
// iteration to the next (on config 2 the second difference of V_k is ~1e-4
// and the third ~1e-7..1e-8 of the first, tools/gpu_warmstart_extrapolation.py),
// so the kept columns start from an extrapolation of the last blocks instead
// of V_k: 2 V_k - V_k-1 (order 1; V_k-1 is still in F when the iteration
// begins) or 3 V_k - 3 V_k-1 + V_k-2 (order 2; V_k-2 kept in Vp).  Only the
// starting point changes; the block is iterated to the same tolerances
// (tightened by PDSDP_QTOL on iterations that start at order 2).
#ifndef PDSDP_EXTRAP
#define PDSDP_EXTRAP 2
#endif
#ifndef PDSDP_QRETRY
#define PDSDP_QRETRY 128        // iterations at order 1 after an order-2 start needed a second pass
#endif
#ifndef PDSDP_QTOL
#define PDSDP_QTOL 0.1          // kept-pair tolerance factor of an iteration that starts at order 2
#endif
#ifndef PDSDP_EXTRAP_WHOLE
#define PDSDP_EXTRAP_WHOLE 1    // after an order-2 start the first pass filters the whole block (guards included)
#endif
#ifndef PDSDP_HINT_MIN
#define PDSDP_HINT_MIN 1        // smallest first-pass filter degree
#endif
#ifndef PDSDP_PROBE_AGE
#define PDSDP_PROBE_AGE 256     // iterations before a failed one-degree-down probe of the hint is retried (0: no probing)
#endif
#ifndef PDSDP_HINT_SAFETY
#define PDSDP_HINT_SAFETY 0     // degrees of slack kept when lowering the filter-degree hint
#endif

// Is Ritz pair i accurate enough?  i < r: kept in X+ (clipped at 0);
// i == r: the certificate eigenvalue lambda_{r+1} (only its value matters).
// factor on the kept-pair tolerances of the current iteration (1, or
// PDSDP_QTOL after an order-2 extrapolated start); block-uniform
__shared__ double g_tolf;

__device__ __forceinline__ bool col_ok(int i, double ri, const double* theta, int r, int b,
                                       double scale, double xnorm, double cert_tol) {
  const double th = theta[i];
  if (!(ri == ri) || !(th == th)) return true;          // non-finite: give up, reported as such
  // sentinel of an effective-rank block: only its sign matters -- the
  // eigenvalue within its residual must be negative (with margin)
  if (i == r && cert_tol < 0.0) return th < 0.0 && ri <= 0.1 * -th;
  // op-level aproj_psd returns lambda_{r+1} itself (symmat.py:242-245): the
  // tight certificate is held to the kept-pair residual whatever its sign
  if (i == r && cert_tol > 0.0 && cert_tol < PDSDP_TOL_CERT) return ri <= cert_tol * scale;
  // clipped / certificate passes -- only trusted once the pair is nearly
  // invariant (a Ritz value of an unconverged block can sit far below the
  // eigenvalue it will converge to)
  if (th + ri < 0.0 && ri <= PDSDP_TOL_CLIP * scale) return true;
  if (i < r) {
    if (ri <= PDSDP_TOL_KEEP * g_tolf * scale) return true;
    // remaining effect on X+: |dtheta| <= ri plus rotation ~ 2 theta ri / gap (Davis-Kahan)
    const double thr = (r < b) ? theta[r] : -1.0e308;
    const double gap = th - thr;
    const double impact = ri + 2.0 * fmax(th, 0.0) * fmin(1.0, ri * fast_rcp(fmax(gap, 1e-300)));
    return impact <= PDSDP_TOL_X * g_tolf * xnorm;
  }
  // cert_tol < 0: sentinel column of an effective-rank block -- it must be
  // certified non-positive (the clip rule above), its value is not needed
  return cert_tol == 0.0 || (cert_tol > 0.0 && ri <= cert_tol * scale);
}

struct Sm {
  ShPtr<double> A, Q, L, M, T;  // lds x lds each
  ShPtr<double> gsc;           // PDSDP_GRAM_SCR
  ShPtr<double> ys;            // staged operand block (n x ycw)
  ShPtr<double> SF;            // own rows of F
  ShPtr<int> szp;              // own rows of zptr
  ShPtr<int> gb;               // [C+1] first row of each CTA (multicast row groups)
  int own, sld;                // own-row buffers valid; their stride
  int ycap;                    // doubles in the staging buffer
  int ycw;                     // staged column chunk width (even; 0 = gather path)
  ShPtr<const int> zc;         // staged Z columns of own rows
  ShPtr<const double> zvs;     // staged Z values of own rows
  int zoff, zstaged;
  int pvalid;                  // leading columns of Vp valid after this iteration's prologue
  int q_used;                  // this iteration started from the order-2 extrapolation
  ShPtr<double> scr;           // NTHR
  ShPtr<double> theta, res, lamF, lamN, dsc, cs, red1;  // BMAX each (red1: 2*BMAX)
  ShPtr<int> perm, pq, flag;
  int lds;
  int gnext[17];               // operator step: next row group's first CTA after group g (thread 0 plans it)
  int gplan;                   // operand row stride the gnext plan was made for (-1: none)
};

__device__ __forceinline__ Sm& s_mut(const Sm& s) { return const_cast<Sm&>(s); }

struct Cta {
  int C, c, r0, r1, par;
};

__device__ __forceinline__ double* red_slot(const Inst& d, const Cta& x, int cc) {
  return d.red + ((size_t)x.par * x.C + cc) * PDSDP_RED_MAX;
}

// Sum of element i over the C partials of the current reduction slot; the C
// loads are issued together (one L2 round trip) and added in rank order.
__device__ __forceinline__ double cluster_sum(const Inst& d, const Cta& x, int i, bool is_max) {
  double v[16];
#pragma unroll
  for (int cc = 0; cc < 16; ++cc) v[cc] = (cc < x.C) ? __ldcg(red_slot(d, x, cc) + i) : 0.0;
  double s = is_max ? -1.0e308 : 0.0;
#pragma unroll
  for (int cc = 0; cc < 16; ++cc)
    if (cc < x.C) s = is_max ? fmax(s, v[cc]) : s + v[cc];
  return s;
}

// Finish a cluster reduction whose per-CTA partial (q_sum sums followed by
// q_max maxima) is already in red_slot(x, x.c).  Result -> dst (smem).
__device__ __forceinline__ void cluster_reduce(const Inst& d, Cta& x, int q_sum, int q_max, double* dst) {
  cg::this_cluster().sync();
  const int q = q_sum + q_max;
  for (int i = threadIdx.x; i < q; i += blockDim.x) dst[i] = cluster_sum(d, x, i, i >= q_sum);
  x.par ^= 1;
  __syncthreads();
}

#ifndef PDSDP_GRAM_SCR
#define PDSDP_GRAM_SCR 3072     // doubles of smem for the cross-warp Gram reduction (12 work items: one per warp; 2048 / 4096 measured slower)
#endif

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// gout[i*nb + j] = sum over own rows rho of A[rho, i] * B[rho, j]  (i < na, j < nb)
// on FP64 tensor cores: warps take (tile group, row chunk) work items, each
// accumulating up to four 8x8 DMMA tiles over its rows (k = 4 rows per
// mma.m8n8k4); chunks are then added in a fixed order through shared memory.
// SA / SB: A / B lie in this CTA's shared memory (LDS instead of generic loads).
template <bool SA = false, bool SB = false, bool CAT = false>
__device__ void gram_mma2(const double* __restrict__ A, int lda, int na, const double* __restrict__ B, int ldb,
                          int nb, int r0, int r1, double* gout, double* wsm,
                          const double* __restrict__ A2 = nullptr, int lda2 = 0, int na1 = 0);

__device__ __forceinline__ void gram_mma(const double* __restrict__ A, int na, const double* __restrict__ B, int nb,
                                         int ld, int r0, int r1, double* gout, double* wsm) {
  gram_mma2(A, ld, na, B, ld, nb, r0, r1, gout, wsm);
}

// CAT: A is the column concatenation [A (na1 columns) | A2 (na - na1 columns)]
template <bool SA, bool SB, bool CAT>
__device__ void gram_mma2(const double* __restrict__ A, int lda, int na, const double* __restrict__ B, int ldb,
                          int nb, int r0, int r1, double* gout, double* wsm,
                          const double* __restrict__ A2, int lda2, int na1) {
  if (SA) A = as_shared(A);
  if (SA && CAT) A2 = as_shared(A2);
  if (SB) B = as_shared(B);
  wsm = as_shared(wsm);
  const int q = na * nb;
  if (q == 0) return;
  const int mt = (na + 7) >> 3, ntl = (nb + 7) >> 3, tiles = mt * ntl;
  const int NG = (tiles + 3) >> 2;
  const int nw = blockDim.x >> 5;
  const int cap = PDSDP_GRAM_SCR / 256;          // work items whose partial tiles fit in wsm
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int nrows = r1 - r0;
  for (int g0 = 0; g0 < NG; g0 += cap) {
    const int ng = min(cap, NG - g0);
    const int chunks = max(1, fdiv(min(nw, cap), ng));
    const int clen = (fdiv(nrows + chunks - 1, chunks) + 3) & ~3;
    for (int wk = warp; wk < ng * chunks; wk += nw) {
      const int ch = fdiv(wk, ng), grp = g0 + wk - ch * ng;
      const int ra = r0 + ch * clen, rb = min(r1, ra + clen);
      double acc[4][2];
      int ti[4], tj[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        acc[t][0] = 0.0; acc[t][1] = 0.0;
        const int tt = grp * 4 + t;
        const int tq_ = fdiv(tt, ntl);
        ti[t] = (tt < tiles) ? tq_ * 8 + g : 1 << 30;
        tj[t] = (tt < tiles) ? (tt - tq_ * ntl) * 8 + g : 1 << 30;
      }
      PDSDP_TICK(43);
      for (int rho0 = ra; rho0 < rb; rho0 += 4) {
        const int rho = rho0 + tq;
        const bool rv = rho < rb;
        double av[4], bv[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (CAT)
            av[t] = (rv && ti[t] < na) ? (ti[t] < na1 ? A[(size_t)rho * lda + ti[t]] : A2[(size_t)rho * lda2 + ti[t] - na1]) : 0.0;
          else
            av[t] = (rv && ti[t] < na) ? A[(size_t)rho * lda + ti[t]] : 0.0;
          bv[t] = (rv && tj[t] < nb) ? B[(size_t)rho * ldb + tj[t]] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) dmma884(acc[t][0], acc[t][1], av[t], bv[t]);
      }
      PDSDP_TICK(44);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        double* w = wsm + ((size_t)(ch * ng + (grp - g0)) * 4 + t) * 64 + g * 8 + 2 * tq;
        w[0] = acc[t][0];
        w[1] = acc[t][1];
      }
    }
    PDSDP_TICK(40);
    __syncthreads();
    PDSDP_TICK(41);
    for (int o = threadIdx.x; o < q; o += blockDim.x) {
      const int i = fdiv(o, nb), j = o - i * nb;
      const int t = (i >> 3) * ntl + (j >> 3);
      const int grp = t >> 2;
      if (grp < g0 || grp >= g0 + ng) continue;
      const int slot = t & 3, el = (i & 7) * 8 + (j & 7);
      double sum = 0.0;
      for (int ch = 0; ch < chunks; ++ch) sum += wsm[((size_t)(ch * ng + (grp - g0)) * 4 + slot) * 64 + el];
      gout[o] = sum;
    }
    PDSDP_TICK(42);
    __syncthreads();
  }
}

// column sums of squares of (P[:, j] - th[j] * Q[:, j]) over own rows
__device__ void colres_partial(const double* __restrict__ P, const double* __restrict__ Qm,
                               const double* th, int b, int ld, int r0, int r1, double* gout, double* scr) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int S = fdiv(nt, b);
  const int sl = fdiv(tid, b), j = tid - sl * b;
  double s = 0.0;
  if (sl < S) {
    const double t = th[j];
    const int len = fdiv(r1 - r0 + S - 1, S);
    const int ra = r0 + sl * len, rb = min(r1, ra + len);
    double s1 = 0.0;
    int rho = ra;
    for (; rho + 2 <= rb; rho += 2) {
      const double v0 = P[(size_t)rho * ld + j] - t * Qm[(size_t)rho * ld + j];
      const double v1 = P[(size_t)(rho + 1) * ld + j] - t * Qm[(size_t)(rho + 1) * ld + j];
      s = fma(v0, v0, s);
      s1 = fma(v1, v1, s1);
    }
    for (; rho < rb; ++rho) {
      const double v = P[(size_t)rho * ld + j] - t * Qm[(size_t)rho * ld + j];
      s = fma(v, v, s);
    }
    s += s1;
  }
  scr[tid] = s;
  __syncthreads();
  if (tid < b) {
    double t = 0.0;
    for (int k = 0; k < S; ++k) t += scr[k * b + tid];
    gout[tid] = t;
  }
  __syncthreads();
}

// Columns [c0, c0+bc) of  out = ca * (S_d Yin) + cb * Yin + cd * Yprev  on own rows:
//   S_d Yin = F T_F + Vl T_V - alpha Z Yin
// with T (smem, (rF + nlock) x bc, flat) already scaled: T_F = diag(lamF) F^T Yin
// and T_V = -diag(theta) Vl^T Yin (deflation of locked Ritz pairs, nlock may be 0).
__device__ __forceinline__ void apply_rows(const Inst& d, const Cta& x, const Sm& s, const double* __restrict__ zv,
                           const double* __restrict__ Yin, const double* __restrict__ Yprev,
                           double* __restrict__ out, int c0, int bc, int rF, int nlock,
                           double ca, double cb, double cd) {
  const int ld = d.ld;
  const int nl = x.r1 - x.r0;
  const double alpha = d.alpha;
  // Z rows of this CTA: staged in shared memory when they fit, so the gather
  // addresses come from smem and only the Y loads go to L2
  const int* __restrict__ zcol = s.zstaged ? s.zc : d.zcol;
  const double* __restrict__ zval = s.zstaged ? s.zvs : zv;
  const int zoff = s.zstaged ? s.zoff : 0;
  // one (row, column) per thread: a warp covers 32/bc rows, each gathered
  // Y row segment is one coalesced transaction; 8 slots per round trip
  for (int it = threadIdx.x; it < nl * bc; it += blockDim.x) {
    const int lq_ = fdiv(it, bc);
    const int rho = x.r0 + lq_, jj = it - lq_ * bc, j = c0 + jj;
    const int e1 = d.zptr[rho + 1] - zoff;
    int e = d.zptr[rho] - zoff;
    double z = 0.0;
    for (; e + 8 <= e1; e += 8) {
      double y[8], v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) { v[u] = zval[e + u]; y[u] = Yin[(size_t)zcol[e + u] * ld + j]; }
#pragma unroll
      for (int u = 0; u < 8; ++u) z = fma(v[u], y[u], z);
    }
    if (e < e1) {
      double y[8], v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool ok = e + u < e1;
        v[u] = ok ? zval[e + u] : 0.0;
        y[u] = ok ? Yin[(size_t)zcol[e + u] * ld + j] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) z = fma(v[u], y[u], z);
    }
    const double yin = (cb != 0.0) ? Yin[(size_t)rho * ld + j] : 0.0;
    const double ypr = (cd != 0.0) ? Yprev[(size_t)rho * ld + j] : 0.0;
    double w = 0.0;
    const double* __restrict__ Fr = d.F + (size_t)rho * ld;
#pragma unroll 4
    for (int l = 0; l < rF; ++l) w = fma(Fr[l], s.T[l * bc + jj], w);
    const double* __restrict__ Vr = d.V + (size_t)rho * ld;
#pragma unroll 4
    for (int l = 0; l < nlock; ++l) w = fma(Vr[l], s.T[(rF + l) * bc + jj], w);
    w = fma(-alpha, z, w);
    double o = ca * w;
    if (cb != 0.0) o = fma(cb, yin, o);
    if (cd != 0.0) o = fma(cd, ypr, o);
    out[(size_t)rho * ld + j] = o;
  }
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
}

// --- TMA bulk multicast + mbarrier (cluster all-gather of the operand block) ---
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* mb, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* mb, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mb, unsigned phase) {
  asm volatile("{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n\t}"
               ::"r"(smem_u32(mb)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_multicast(void* dst_smem, const void* src_gmem, unsigned bytes,
                                               unsigned long long* mb, unsigned short mask) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
               " [%0], [%1], %2, [%3], %4;"
               ::"r"(smem_u32(dst_smem)), "l"(src_gmem), "r"(bytes), "r"(smem_u32(mb)), "h"(mask) : "memory");
}
// Cluster barrier with release / acquire semantics: this CTA's reads of its
// staging buffer happen-before the other CTAs' next multicast writes into it.
__device__ __forceinline__ void cluster_sync_relacq() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Same contract as apply_rows, but the operand block Yin is first copied
// into shared memory for ALL n rows (column chunks of width s.ycw, 16-byte
// cp.async, every load independent), so the sparse product reads its
// gathered rows from smem instead of issuing dependent L2 round trips.
__device__ __forceinline__ void apply_rows_staged(const Inst& d, const Cta& x, const Sm& s, const double* __restrict__ zv,
                                  const double* __restrict__ Yin, const double* __restrict__ Yprev,
                                  double* __restrict__ out, int c0, int bc, int rF, int nlock,
                                  double ca, double cb, double cd) {
  const int ld = d.ld, n = d.n;
  const int nl = x.r1 - x.r0;
  const double alpha = d.alpha;
  const int* __restrict__ zcol = s.zstaged ? s.zc : d.zcol;
  const double* __restrict__ zval = s.zstaged ? s.zvs : zv;
  const int zoff = s.zstaged ? s.zoff : 0;
  double* ys = s.ys;
  const int cw = s.ycw;                       // even
  const int a0 = c0 & ~1, a1 = c0 + bc;       // aligned column span [a0, a1)
  for (int cs0 = a0; cs0 < a1; cs0 += cw) {
    const int pairs = cw >> 1;
    for (int idx = threadIdx.x; idx < n * pairs; idx += blockDim.x) {
      const int row = fdiv(idx, pairs), pr = idx - row * pairs;
      cp_async16(ys + (size_t)row * cw + 2 * pr, Yin + (size_t)row * ld + cs0 + 2 * pr);
    }
    cp_async_wait_all();
    __syncthreads();
    const int jlo = max(cs0, c0), jhi = min(cs0 + cw, a1), w_ = jhi - jlo;
    for (int it = threadIdx.x; it < nl * w_; it += blockDim.x) {
      const int lq_ = fdiv(it, w_);
      const int rho = x.r0 + lq_, j = jlo + it - lq_ * w_, jj = j - c0, js = j - cs0;
      const int e1 = d.zptr[rho + 1] - zoff;
      int e = d.zptr[rho] - zoff;
      double z0 = 0.0, z1 = 0.0;
      for (; e + 2 <= e1; e += 2) {
        z0 = fma(zval[e], ys[(size_t)zcol[e] * cw + js], z0);
        z1 = fma(zval[e + 1], ys[(size_t)zcol[e + 1] * cw + js], z1);
      }
      if (e < e1) z0 = fma(zval[e], ys[(size_t)zcol[e] * cw + js], z0);
      const double z = z0 + z1;
      const double ypr = (cd != 0.0) ? Yprev[(size_t)rho * ld + j] : 0.0;
      double w = 0.0;
      const double* __restrict__ Fr = d.F + (size_t)rho * ld;
#pragma unroll 4
      for (int l = 0; l < rF; ++l) w = fma(Fr[l], s.T[l * bc + jj], w);
      const double* __restrict__ Vr = d.V + (size_t)rho * ld;
#pragma unroll 4
      for (int l = 0; l < nlock; ++l) w = fma(Vr[l], s.T[(rF + l) * bc + jj], w);
      w = fma(-alpha, z, w);
      double o = ca * w;
      if (cb != 0.0) o = fma(cb, ys[(size_t)rho * cw + js], o);
      if (cd != 0.0) o = fma(cd, ypr, o);
      out[(size_t)rho * ld + j] = o;
    }
    __syncthreads();
  }
}

// out = In * Msm (b x b in smem), own rows; In and out must differ.
__device__ __forceinline__ void rotate_rows(const Inst& d, const Cta& x, const double* __restrict__ In, const double* Msm,
                            int lds, double* __restrict__ out, int b) {
  const int ld = d.ld;
  const int nl = x.r1 - x.r0;
  for (int it = threadIdx.x; it < nl * b; it += blockDim.x) {
    const int lq_ = fdiv(it, b);
    const int rho = x.r0 + lq_, j = it - lq_ * b;
    const double* row = In + (size_t)rho * ld;
    double acc = 0.0;
#pragma unroll 8
    for (int t = 0; t < b; ++t) acc = fma(row[t], Msm[t * lds + j], acc);
    out[(size_t)rho * ld + j] = acc;
  }
}

// rows [0, nl) of a b-column block, global (stride ld) -> shared (stride b).
// With an even b (rows and dst 16-byte aligned) the copy is issued as 16-byte
// cp.async (global -> shared without a register stage): every transfer of the
// block is in flight at once, where a plain copy loop pays one L2 round trip
// per trip -- and holding several loads in registers instead spills in the
// Rayleigh-Ritz section.  The caller's copies are completed by copy_rows_wait().
__device__ __forceinline__ void copy_rows_in(const double* __restrict__ src, int ld, double* dst, int nl, int b) {
  if ((b & 1) == 0 && (ld & 1) == 0) {
    const int hp = b >> 1, tot = nl * hp;
    for (int it = threadIdx.x; it < tot; it += blockDim.x) {
      const int lr = fdiv(it, hp), j2 = it - lr * hp;
      cp_async16(dst + 2 * it, src + (size_t)lr * ld + 2 * j2);
    }
    return;
  }
  for (int it = threadIdx.x; it < nl * b; it += blockDim.x) {
    const int lr = fdiv(it, b), j = it - lr * b;
    dst[it] = src[(size_t)lr * ld + j];
  }
}
__device__ __forceinline__ void copy_rows_wait() { cp_async_wait_all(); }

// out (nl x b) = In (nl x b, shared memory) * Msm (b x b, shared memory) on
// FP64 tensor cores (mma.sync.m8n8k4.f64): one warp per 8-row tile, all
// 8-column tiles of the row tile at once (the A fragment is loaded once per
// k-step).  A scalar product reads 16 bytes of shared memory per FMA; this
// reads ~2 (the b x b rotations of a Rayleigh-Ritz pass were bound by it).
// With In2 / out2 a second block sharing Msm is rotated in the same sweep;
// with th != nullptr the column sums of (out2 - th .* out)^2 over the rows
// are accumulated (Ritz residual norms, fixed-order reduction) into gout[b].
__device__ void rot_mma(const double* __restrict__ In, int ldi, const double* __restrict__ In2, int ldi2,
                        const double* __restrict__ Msm, int lds, double* __restrict__ out, int ldo,
                        double* __restrict__ out2, int ldo2, int nl, int b, const double* __restrict__ th,
                        double* __restrict__ gout, double* __restrict__ scr) {
  // In, In2 and Msm always lie in this CTA's shared memory: LDS, not generic loads
  In = as_shared(In);
  if (In2) In2 = as_shared(In2);
  Msm = as_shared(Msm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int nw = blockDim.x >> 5;
  const int mt = (nl + 7) >> 3, ntl = (b + 7) >> 3;   // ntl <= 8
  double cres[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) { cres[q][0] = 0.0; cres[q][1] = 0.0; }
  for (int tm = warp; tm < mt; tm += nw) {
    const int row = tm * 8 + g;
    const bool rv = row < nl;
    double acc[8][2], acc2[8][2];
#pragma unroll
    for (int q = 0; q < 8; ++q) { acc[q][0] = acc[q][1] = 0.0; acc2[q][0] = acc2[q][1] = 0.0; }
    for (int t0 = 0; t0 < b; t0 += 4) {
      const int t = t0 + tq;
      const bool tv = t < b;
      const double a = (rv && tv) ? In[(size_t)row * ldi + t] : 0.0;
      const double a2 = (In2 && rv && tv) ? In2[(size_t)row * ldi2 + t] : 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (q < ntl) {
          const int col = q * 8 + g;
          const double bm = (tv && col < b) ? Msm[t * lds + col] : 0.0;
          dmma884(acc[q][0], acc[q][1], a, bm);
          if (In2) dmma884(acc2[q][0], acc2[q][1], a2, bm);
        }
      }
    }
    // D fragment: row tm*8+g, columns q*8 + 2tq + h
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q < ntl && rv) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = q * 8 + 2 * tq + h;
          if (col < b) {
            out[(size_t)row * ldo + col] = acc[q][h];
            if (out2) out2[(size_t)row * ldo2 + col] = acc2[q][h];
            if (th) {
              const double rr = acc2[q][h] - th[col] * acc[q][h];
              cres[q][h] = fma(rr, rr, cres[q][h]);
            }
          }
        }
      }
    }
  }
  if (th) {
    // lanes with the same tq hold the same columns: reduce over g (xor 4, 8, 16)
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double v = cres[q][h];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        cres[q][h] = v;
      }
    if (g == 0)
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = q * 8 + 2 * tq + h;
          if (col < b) scr[warp * PDSDP_BMAX + col] = cres[q][h];
        }
    __syncthreads();
    if ((int)threadIdx.x < b) {
      double tsum = 0.0;
      for (int w = 0; w < nw; ++w) tsum += scr[w * PDSDP_BMAX + threadIdx.x];
      gout[threadIdx.x] = tsum;
    }
  }
  __syncthreads();
}

// T (smem, (rF + nlock) x bc) <- [diag(lamF); -diag(theta)] .* T  (in place)
__device__ void scale_T(const Sm& s, int rF, int nlock, int bc) {
  for (int e = threadIdx.x; e < (rF + nlock) * bc; e += blockDim.x) {
    const int l = fdiv(e, bc);
    const double c = (l < rF) ? s.lamF[l] : -s.theta[l - rF];
    s.T[e] = (c == 0.0) ? 0.0 : s.T[e] * c;
  }
  __syncthreads();
}

// One operator product on columns [c0, c0+bc): reduction of [F | Vl]^T Yin
// (one cluster barrier, which also publishes Yin to every CTA), then rows.
__device__ __forceinline__ void operator_step(const Inst& d, Cta& x, const Sm& s, const double* zv, const double* Yin,
                              const double* Yprev, double* out, int c0, int bc, int rF, int nlock,
                              double ca, double cb, double cd, Prof& pf) {
  prof_mark(pf, 1);
  double* slot = red_slot(d, x, x.c);
  gram_mma(d.F, rF, Yin + c0, bc, d.ld, x.r0, x.r1, slot, s.gsc);
  gram_mma(d.V, nlock, Yin + c0, bc, d.ld, x.r0, x.r1, slot + rF * bc, s.gsc);
  prof_mark(pf, 2);
  cluster_reduce(d, x, (rF + nlock) * bc, 0, s.T);
  scale_T(s, rF, nlock, bc);
  prof_mark(pf, 3);
  if (s.ycw >= 2) apply_rows_staged(d, x, s, zv, Yin, Yprev, out, c0, bc, rF, nlock, ca, cb, cd);
  else apply_rows(d, x, s, zv, Yin, Yprev, out, c0, bc, rF, nlock, ca, cb, cd);
}

// Operator step of the Chebyshev recurrence.  The operand block Y_j (active
// columns, compact row stride bcp = bc rounded up to 4, global buffer Yc[p])
// is all-gathered inside the cluster with TMA bulk multicast: every CTA
// broadcasts its own rows into every CTA's staging buffer (one L2 read per
// row block), in row groups that fit the buffer.  Work items are (own row,
// 4-column chunk): each gathered Z slot feeds 4 FMAs from two 16-byte smem
// loads, and a running slot pointer per item walks the row's (column-sorted)
// slots group by group.  F's own rows stay in shared memory.  Y_{j+1} goes to
// global row-major (for Rayleigh-Ritz) and into Yc[p^1] over Y_{j-1}.
#ifndef PDSDP_OWN_ITEMS
#define PDSDP_OWN_ITEMS 3      // (row, 4-column chunk) items per thread
#endif
__device__ __forceinline__ int own_stride(int bc) { return (bc + 3) & ~3; }
// row stride of the compact operand block: the smallest odd number of 16-byte
// units that holds the bc columns, so the 16-byte loads of different rows at
// the same column chunk fall in different shared-memory bank groups (a
// multiple of 128 bytes put them all in the same group: 2-way conflicts on
// every operand load).  It may be shorter than the 4-column chunks' span
// (bc = 22: 22 doubles for 6 chunks): the last chunk's upper load then reads
// the next row's first two entries, which only feed discarded columns.  A
// tighter stride is fewer multicast bytes and more rows per staging group
// (n = 2000, rank 20: 3 row groups per operator step instead of 4).
__device__ __forceinline__ int own_ystr(int bc) {
  int u = (bc + 1) >> 1;
  if (!(u & 1)) ++u;
  return 2 * u;
}
// the locked pairs' own rows are copied next to F's in shared memory when
// they fit the row stride of SF
__device__ __forceinline__ bool own_lock_sm(int rFx, int nlock, int sl) { return nlock > 0 && rFx + nlock <= sl; }

// Sparse part of one operator-step row group: for every (own row, 4-column
// chunk) item of this thread, accumulate Z[row, q] * Y[q, chunk] over the
// row's slots whose column q lies in the staged rows [R0, R1).  The items of
// a thread run interleaved (independent chains) and the next slot's column
// is loaded before the current slot's products, so a thread keeps several
// shared-memory round trips in flight.  SZ: Z slots staged in shared memory.
template <bool SZ, int NI>
__device__ __forceinline__ void own_gather(const int* __restrict__ zcol, const double* __restrict__ zval,
                                           const double* ys, int R0, int R1, int cq, int ys_,
                                           int (&ep)[NI], const int (&ee)[NI],
                                           double (&zacc)[NI][4]) {
  constexpr int BIG = 0x7fffffff;
  int q[NI];
  // chunks 4..7 of a quarter warp read their upper 16 bytes first: the eight
  // first loads of a row's chunks then fall in eight distinct bank groups
  // (zacc holds the two halves swapped for those threads; the caller undoes it)
  const int sw = (cq >> 2) & 1;
  const double* yb = ys + 4 * cq + 2 * sw - (size_t)R0 * ys_;
  const int o2 = 2 - 4 * sw;
#pragma unroll
  for (int u = 0; u < NI; ++u) q[u] = (ep[u] < ee[u]) ? zcol[ep[u]] : BIG;
  if (SZ) {
    // Z slots and operand rows in shared memory: 32-bit shared addresses
    // kept in registers (the generic form recomputed 64-bit pointers per slot)
    const unsigned zc_a = smem_u32(zcol), zv_a = smem_u32(zval);
    const unsigned yb_a = smem_u32(ys) + 8u * (unsigned)(4 * cq + 2 * sw) - 8u * (unsigned)R0 * (unsigned)ys_;
    const unsigned rowb = 8u * (unsigned)ys_, o2b = 8u * (unsigned)o2;
    while (true) {
      bool any = false;
#pragma unroll
      for (int u = 0; u < NI; ++u) any |= q[u] < R1;
      if (!any) break;
#pragma unroll
      for (int u = 0; u < NI; ++u) {
        if (q[u] < R1) {
          const int e = ep[u];
          const unsigned a = yb_a + (unsigned)q[u] * rowb;
          double zv_, y0, y1, y2, y3;
          asm volatile("ld.shared.f64 %0, [%1];" : "=d"(zv_) : "r"(zv_a + 8u * (unsigned)e));
          asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(y0), "=d"(y1) : "r"(a));
          asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(y2), "=d"(y3) : "r"(a + o2b));
          int qn = BIG;
          if (e + 1 < ee[u]) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(qn) : "r"(zc_a + 4u * (unsigned)(e + 1)));
          ep[u] = e + 1;
          q[u] = qn;
          zacc[u][0] = fma(zv_, y0, zacc[u][0]); zacc[u][1] = fma(zv_, y1, zacc[u][1]);
          zacc[u][2] = fma(zv_, y2, zacc[u][2]); zacc[u][3] = fma(zv_, y3, zacc[u][3]);
        }
      }
    }
    return;
  }
  while (true) {
    bool any = false;
#pragma unroll
    for (int u = 0; u < NI; ++u) any |= q[u] < R1;
    if (!any) break;
#pragma unroll
    for (int u = 0; u < NI; ++u) {
      if (q[u] < R1) {
        const int e = ep[u];
        const double zv_ = zval[e];
        const double2 p0 = *reinterpret_cast<const double2*>(yb + (size_t)q[u] * ys_);
        const double2 p1 = *reinterpret_cast<const double2*>(yb + (size_t)q[u] * ys_ + o2);
        ep[u] = e + 1;
        q[u] = (e + 1 < ee[u]) ? zcol[e + 1] : BIG;
        zacc[u][0] = fma(zv_, p0.x, zacc[u][0]); zacc[u][1] = fma(zv_, p0.y, zacc[u][1]);
        zacc[u][2] = fma(zv_, p1.x, zacc[u][2]); zacc[u][3] = fma(zv_, p1.y, zacc[u][3]);
      }
    }
  }
}

template <int NI>
__device__ __forceinline__ void operator_step_own(const Inst& d, Cta& x, const Sm& s, const double* zv,
                                                  double* out, int c0, int bc, int rF, int nlock,
                                                  double ca, double cb, double cd, Prof& pf,
                                                  int& ycp, unsigned long long* mbar, unsigned& mphase,
                                                  bool& gram_ready, bool gram_next) {
  prof_mark(pf, 1);
  const int nl = x.r1 - x.r0, sl = s.sld, ld = d.ld, n = d.n, tid = threadIdx.x;
  const int bcp = own_stride(bc), nch = bcp >> 2, ys_ = own_ystr(bc);
  const size_t nld = (size_t)n * (ld + 4);
  const double* Ycur = d.Yc + (size_t)ycp * nld;
  double* Ynxt = d.Yc + (size_t)(ycp ^ 1) * nld;
  // work items: (own row, 4-column chunk).  Thread t takes chunk t % nch of
  // rows t / nch + u * rps (u < NI): its items share the column
  // chunk, so the dense epilogue loads each T entry once for all of them
  const int rps = fdiv(blockDim.x, nch), lr0 = fdiv(tid, nch), cq = tid - lr0 * nch;
  const int tstr = (bc + 1) & ~1;   // row stride of T in this step (even)
  const bool tact = lr0 < rps;
  if (!gram_ready) {     // [F | V_lock]^T Y_j partial of the own rows
    // own rows of Y_j into the (still idle) staging buffer first: a Gram
    // product reading L2 directly waits one round trip per k-step
    double* yo = s.ys;
    {
      const double* src = Ycur + (size_t)x.r0 * ys_;
      for (int i = tid; i < nl * ys_ / 2; i += blockDim.x) cp_async16(yo + 2 * i, src + 2 * i);   // all in flight, no register stage
      cp_async_wait_all();
    }
    __syncthreads();
    double* slot = red_slot(d, x, x.c);
    if (own_lock_sm(rF, nlock, sl)) {
      gram_mma2<true, true>(s.SF, sl, rF + nlock, yo, ys_, bc, 0, nl, slot, s.gsc);
    } else {
      gram_mma2<true, true>(s.SF, sl, rF, yo, ys_, bc, 0, nl, slot, s.gsc);
      gram_mma2<false, true>(d.V + (size_t)x.r0 * ld, ld, nlock, yo, ys_, bc, 0, nl, slot + rF * bc, s.gsc);
    }
  }
  gram_ready = false;
  if (tid == 0 && s.gplan != ys_) {   // row groups that fit the staging buffer (published by the barrier below)
    s_mut(s).gplan = ys_;
    const int rc = fdiv(s.ycap, ys_);
    for (int g0 = 0; g0 < x.C;) {
      int g1 = g0 + 1;
      while (g1 < x.C && s.gb[g1 + 1] - s.gb[g0] <= rc) ++g1;
      s_mut(s).gnext[g0] = g1;
      g0 = g1;
    }
  }
  prof_mark(pf, 2);
  cg::this_cluster().sync();                 // publishes Y_j rows and the partials
  prof_tick(pf, 20);
  const double alpha = d.alpha;
  const double* ys = s.ys;
  const int C = x.C;
  const unsigned short mask = (unsigned short)((1u << C) - 1u);
  const int* __restrict__ zcol = s.zstaged ? s.zc : d.zcol;
  const double* __restrict__ zval = s.zstaged ? s.zvs : zv;
  const int zoff = s.zstaged ? s.zoff : 0;
  double zacc[NI][4];
  int ep[NI], ee[NI];
#pragma unroll
  for (int u = 0; u < NI; ++u) {
    const int lr = lr0 + u * rps;
    const bool ok = tact && lr < nl;
    ep[u] = s.szp[ok ? lr : 0] - zoff;
    ee[u] = ok ? s.szp[lr + 1] - zoff : ep[u];
#pragma unroll
    for (int v = 0; v < 4; ++v) zacc[u][v] = 0.0;
  }
  int g0 = 0;
  bool first = true;
  while (g0 < C) {
    const int R0 = s.gb[g0];
    const int g1 = s.gnext[g0];
    const int R1 = s.gb[g1];
    if (tid == 0) {
      mbar_expect_tx(mbar, (unsigned)((R1 - R0) * ys_ * 8));
      if (x.c >= g0 && x.c < g1) {
        const char* src = reinterpret_cast<const char*>(Ycur + (size_t)x.r0 * ys_);
        char* dst = reinterpret_cast<char*>(s.ys + (size_t)(x.r0 - R0) * ys_);
        unsigned left = (unsigned)(nl * ys_ * 8), off = 0;
        while (left > 0) {
          const unsigned piece = left > 65536u ? 65536u : left;
          bulk_multicast(dst + off, src + off, piece, mbar, mask);
          off += piece; left -= piece;
        }
      }
    }
    prof_mark(pf, 13);
    mbar_wait(mbar, mphase);
    mphase ^= 1u;
    // reduce T once the first operand group has landed (its L2 reads would
    // otherwise queue behind the multicast traffic into this SM)
    if (first) {
      const int q = (rF + nlock) * bc;
      for (int i = tid; i < q; i += blockDim.x) {
        const int l = fdiv(i, bc);
        const double c = (l < rF) ? s.lamF[l] : -s.theta[l - rF];
        const double v = cluster_sum(d, x, i, false);
        s.T[l * tstr + (i - l * bc)] = (c == 0.0) ? 0.0 : v * c;   // even row stride: 16-byte rows
      }
      x.par ^= 1;
      first = false;
      prof_tick(pf, 21);
    }
    __syncthreads();
    prof_mark(pf, 14);
    if (s.zstaged) own_gather<true, NI>(s.zc, s.zvs, ys, R0, R1, cq, ys_, ep, ee, zacc);
    else own_gather<false, NI>(zcol, zval, ys, R0, R1, cq, ys_, ep, ee, zacc);
    g0 = g1;
    prof_tick(pf, 22);
    // the staging buffer is reused by the next group: the arrive must have
    // release semantics so that this CTA's shared-memory reads of the group
    // are ordered before the other CTAs' multicast writes of the next one
    // (a relaxed arrive orders nothing: write-after-read race)
    if (g0 < C) cluster_sync_relacq();
    prof_mark(pf, 3);
  }
  if ((cq >> 2) & 1) {        // own_gather kept this thread's chunk halves swapped
#pragma unroll
    for (int u = 0; u < NI; ++u) {
      double t = zacc[u][0]; zacc[u][0] = zacc[u][2]; zacc[u][2] = t;
      t = zacc[u][1]; zacc[u][1] = zacc[u][3]; zacc[u][3] = t;
    }
  }
#ifdef PDSDP_PROF_EPI
  prof_mark(pf, 10);
#endif
  // locked pairs' own rows sit after F's in SF when they fit (own_lock_sm)
  const int nsf = own_lock_sm(rF, nlock, sl) ? rF + nlock : rF;
  const int nglb = nsf == rF ? nlock : 0;
  // dense part [F | V_lock] T of all items: T entries loaded once per thread
  double w[NI][4];
#pragma unroll
  for (int u = 0; u < NI; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) w[u][v] = 0.0;
  if (tact) {
    const double* Fr[NI];
#pragma unroll
    for (int u = 0; u < NI; ++u) {
      const int lr = lr0 + u * rps;
      Fr[u] = s.SF + (size_t)(lr < nl ? lr : 0) * sl;
    }
    // entries past bc are never used; chunks 4..7 of a quarter warp read the
    // upper half of their chunk first (distinct bank groups for all seven
    // chunks of a row), w then holds those halves swapped until the end
    const int sw = (cq >> 2) & 1;
    const double* Tc = s.T + 4 * cq + 2 * sw;
    const int o2 = 2 - 4 * sw;
    for (int l = 0; l < nsf; ++l) {
      const double2 ta = *reinterpret_cast<const double2*>(Tc + l * tstr);
      const double2 tb = *reinterpret_cast<const double2*>(Tc + l * tstr + o2);
#pragma unroll
      for (int u = 0; u < NI; ++u) {
        const double f = Fr[u][l];
        w[u][0] = fma(f, ta.x, w[u][0]); w[u][1] = fma(f, ta.y, w[u][1]);
        w[u][2] = fma(f, tb.x, w[u][2]); w[u][3] = fma(f, tb.y, w[u][3]);
      }
    }
    if (sw) {
#pragma unroll
      for (int u = 0; u < NI; ++u) {
        double t = w[u][0]; w[u][0] = w[u][2]; w[u][2] = t;
        t = w[u][1]; w[u][1] = w[u][3]; w[u][3] = t;
      }
    }
  }
  prof_tick(pf, 23);
#pragma unroll
  for (int u = 0; u < NI; ++u) {
    const int lr = lr0 + u * rps;
    if (!tact || lr >= nl) break;
    const double* Vr = d.V + (size_t)(x.r0 + lr) * ld;
    const size_t oc = (size_t)(x.r0 + lr) * ys_ + 4 * cq;
    // recurrence terms Y_j, Y_{j-1} of the item, loaded before its stores
    // (which may alias them as far as the compiler knows: one L2 round trip
    // per item instead of one per element)
    double yc[4], yp[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const bool ok = 4 * cq + v < bc;
      yc[v] = (ok && cb != 0.0) ? __ldcg(Ycur + oc + v) : 0.0;
      yp[v] = (ok && cd != 0.0) ? __ldcg(Ynxt + oc + v) : 0.0;
    }
    for (int t = 0; t < nglb; ++t) {
      const double f = __ldcg(Vr + t);
      const double* Tl = s.T + (rF + t) * tstr + 4 * cq;
#pragma unroll
      for (int v = 0; v < 4; ++v) w[u][v] = fma(f, Tl[v], w[u][v]);
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int jj = 4 * cq + v;
      if (jj >= bc) break;
      const double wv = fma(-alpha, zacc[u][v], w[u][v]);
      double o = ca * wv;
      if (cb != 0.0) o = fma(cb, yc[v], o);
      if (cd != 0.0) o = fma(cd, yp[v], o);
      out[(size_t)(x.r0 + lr) * ld + c0 + jj] = o;
      Ynxt[oc + v] = o;
      zacc[u][v] = o;
    }
  }
#ifdef PDSDP_PROF_EPI
  prof_mark(pf, 12);
#endif
  prof_tick(pf, 24);
  fence_proxy_async();
  __syncthreads();
  prof_tick(pf, 25);
#ifdef PDSDP_PROF_EPI
  prof_mark(pf, 3);
#endif
  if (gram_next) {
    // the next step's Gram partial from a shared-memory copy of the own rows
    // of Y_{j+1} (the staging buffer is idle until the next cluster barrier)
    double* yo = s.ys;
#pragma unroll
    for (int u = 0; u < NI; ++u) {
      const int lr = lr0 + u * rps;
      if (!tact || lr >= nl) break;
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (4 * cq + v < ys_) yo[(size_t)lr * ys_ + 4 * cq + v] = (4 * cq + v < bc) ? zacc[u][v] : 0.0;
    }
    __syncthreads();
    prof_tick(pf, 27);
    double* slot = red_slot(d, x, x.c);
    if (own_lock_sm(rF, nlock, sl)) {
      gram_mma2<true, true>(s.SF, sl, rF + nlock, yo, ys_, bc, 0, nl, slot, s.gsc);
    } else {
      gram_mma2<true, true>(s.SF, sl, rF, yo, ys_, bc, 0, nl, slot, s.gsc);
      gram_mma2<false, true>(d.V + (size_t)x.r0 * ld, ld, nlock, yo, ys_, bc, 0, nl, slot + rF * bc, s.gsc);
    }
    gram_ready = true;
  }
  prof_tick(pf, 26);
  ycp ^= 1;
}

// Items per thread for this step: two when they cover the CTA's rows (fewer
// interleaved gather chains per thread, config 2: 3% faster), else
// PDSDP_OWN_ITEMS (the launch checked that those cover them).
__device__ __forceinline__ void operator_step_own_any(const Inst& d, Cta& x, const Sm& s, const double* zv,
                                                      double* out, int c0, int bc, int rF, int nlock,
                                                      double ca, double cb, double cd, Prof& pf,
                                                      int& ycp, unsigned long long* mbar, unsigned& mphase,
                                                      bool& gram_ready, bool gram_next) {
  const int rps = fdiv(blockDim.x, own_stride(bc) >> 2);
  if (x.r1 - x.r0 <= rps)
    operator_step_own<1>(d, x, s, zv, out, c0, bc, rF, nlock, ca, cb, cd, pf, ycp, mbar, mphase, gram_ready, gram_next);
  else if (PDSDP_OWN_ITEMS > 2 && x.r1 - x.r0 <= 2 * rps)
    operator_step_own<2>(d, x, s, zv, out, c0, bc, rF, nlock, ca, cb, cd, pf, ycp, mbar, mphase, gram_ready, gram_next);
  else
    operator_step_own<PDSDP_OWN_ITEMS>(d, x, s, zv, out, c0, bc, rF, nlock, ca, cb, cd, pf, ycp, mbar, mphase, gram_ready,
                                       gram_next);
}

// Convergence state of the Ritz block (identical in every thread).
struct Assess {
  int last_bad;     // last kept column (< r) still needing work, -1 if none
  bool cert_bad;    // lambda_{r+1} requested and not yet accurate
  bool tail_bad;    // lambda_{r+1} not clearly separated from the kept pairs
  double rho_k;     // residual reduction still needed on the kept columns
  double maxres;    // worst relative residual among columns needing work
};

// Warp-parallel per-column scans: every warp evaluates
// them independently (lanes stride the columns, fixed xor-shuffle trees), so
// all threads of all CTAs hold identical results without a barrier.  A
// sequential scan over up to 64 columns with FP64 divisions was several
// microseconds on the critical path of every pass.
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_maxi(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_mini(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// ||X+||_F estimate sqrt(sum_{i<min(r,b)} max(theta_i, 0)^2)
__device__ __forceinline__ double kept_norm_w(const double* theta, int r, int b) {
  const int lane = threadIdx.x & 31, nk = min(r, b);
  double acc = 0.0;
  for (int i = lane; i < nk; i += 32) { const double t = fmax(theta[i], 0.0); acc = fma(t, t, acc); }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return sqrt(acc);
}
__device__ Assess assess_w(const double* theta, const double* res, int r, int b, int k, double scale,
                           double xnorm, double cert_tol) {
  Assess a{-1, false, false, 1.0, 0.0};
  const int lane = threadIdx.x & 31;
  // reciprocals by rcp.approx + two Newton steps: the software FP64 division
  // sits on the critical path of every pass (planning needs a few digits)
  const double inv_scale = fast_rcp(scale);
  const double inv_tk = fast_rcp(g_tolf * fmax(PDSDP_TOL_KEEP * scale, PDSDP_TOL_X * xnorm));
  int last = -1, cert = 0;
  double mr = 0.0, rk = 1.0;
  for (int i = lane; i < k; i += 32) {
    const double ri = res[i];
    if (col_ok(i, ri, theta, r, b, scale, xnorm, cert_tol)) continue;
    mr = fmax(mr, ri * inv_scale);
    if (i < r) { last = max(last, i); rk = fmax(rk, ri * inv_tk); }
    else cert = 1;
  }
  a.last_bad = warp_maxi(last);
  a.cert_bad = warp_maxi(cert) != 0;
  a.maxres = warp_max(mr);
  a.rho_k = warp_max(rk);
  if (r < b && r < k + 1 && r >= 1) {
    const double lo_k = theta[r - 1] - 2.0 * res[r - 1];
    const double hi_t = theta[r] + 2.0 * res[r];
    if (!(hi_t < lo_k) && res[r] > PDSDP_TOL_CERT * scale &&
        !(theta[r] + res[r] < 0.0 && res[r] <= PDSDP_TOL_CLIP * scale) &&
        !(cert_tol < 0.0 && theta[r] < 0.0 && res[r] <= 0.1 * -theta[r])) {
      a.tail_bad = true;
      a.maxres = fmax(a.maxres, res[r] * inv_scale);
    }
  }
  return a;
}
// leading columns [0, n) that are col_ok, n <= lim
__device__ __forceinline__ int leading_ok_w(const double* theta, const double* res, int r, int b, int lim,
                                            double scale, double xnorm, double cert_tol) {
  const int lane = threadIdx.x & 31;
  int first_bad = lim;
  for (int i = lane; i < lim; i += 32)
    if (!col_ok(i, res[i], theta, r, b, scale, xnorm, cert_tol)) first_bad = min(first_bad, i);
  return warp_mini(first_bad);
}

// Filter-planning heuristics (degrees, caps, slack) need ~3 digits: FP32
// hardware approximations instead of the FP64 software log / acosh (each a
// few hundred dependent cycles, on the critical path of every pass).
__device__ __forceinline__ double plan_log(double x) {
  return (double)__logf((float)fmin(fmax(x, 1e-37), 1e37));
}
__device__ __forceinline__ double plan_acosh(double x) {   // x >= 1
  const float xf = (float)fmin(fmax(x, 1.0), 1e18);
  return (double)__logf(xf + sqrtf((xf - 1.0f) * (xf + 1.0f)));
}

// Chebyshev filter for columns [a0, a1): damp [lo, cut], scale at `top`;
// degree to reduce a column at `slow` by `rho`, and a cap keeping the
// amplification spread across the active columns below ~1e4/eps_rel
// (beyond that the filtered block loses rank and CholQR breaks down).
__device__ int cheb_plan(const double* theta, int a1, double lo, double top, double cut, double slow,
                         double rho, double scale, double eps_rel, int& mm, double& e_, double& c_,
                         double& s_) {
  const double lo_ = fmin(lo, cut);
  e_ = 0.5 * (cut - lo_);
  c_ = 0.5 * (cut + lo_);
  if (e_ < 1e-14 * scale) e_ = 1e-14 * scale;
  if (top - c_ <= e_) top = c_ + 1.0001 * e_;
  s_ = e_ * fast_rcp(top - c_);
  const double ie = fast_rcp(e_);
  const double ts = (slow - c_) * ie;
  const double at = (ts > 1.0 + 1e-6) ? plan_acosh(ts) : 0.0;
  mm = (at > 0.0) ? (int)ceilf(__fdividef((float)plan_acosh(fmax(rho, 1.0)), (float)at)) + 1 : 8;
  const double tb = (theta[a1 - 1] - c_) * ie;
  const double spread = plan_acosh(fmax((top - c_) * ie, 1.0 + 1e-6)) - ((tb > 1.0 + 1e-6) ? plan_acosh(tb) : 0.0);
  int mcap = PDSDP_MMAX;
  if (spread > 1e-3)
    mcap = (int)fminf((float)PDSDP_MMAX, floorf(__fdividef((float)plan_log(PDSDP_SPREAD_CAP * fast_rcp(fmin(fmax(eps_rel, 1e-16), 1.0))), (float)spread)));
  if (mcap < 2) mcap = 2;
  return mcap;
}

// ||dX||_F^2 for dX = V diag(lamN) V^T - F diag(lamF) F^T with orthonormal V
// (n x rN) and F (n x rF), from P = V^T F and G = F_perp^T F_perp, F_perp =
// F - V P:
//   dX = V A0 V^T - V B F_perp^T - F_perp B^T V^T - F_perp diag(lamF) F_perp^T,
//   A0 = diag(lamN) - P diag(lamF) P^T,  B = P diag(lamF),
// whose four blocks are mutually orthogonal (V^T F_perp = 0), so
//   ||dX||^2 = ||A0||^2 + 2 tr(B G B^T) + sum_jl lamF_j lamF_l G_jl^2.
// Every term is a sum of squares of small quantities: no cancellation against
// ||X||^2 (the expanded square ||X+||^2 - 2<X+, X> + ||X||^2 loses ~10 digits
// near the stopping tolerance).  Block-wide; deterministic fixed-order sums.
__device__ double dense_residual_lowrank(const double* P, const double* G, const double* lamN, const double* lamF,
                                         int rN, int rF, double* scr) {
  const int tid = threadIdx.x;
  double acc = 0.0;
  // ||A0||^2 : one entry (i, l) per work item
  for (int e = tid; e < rN * rN; e += blockDim.x) {
    const int i = fdiv(e, rN), l = e - i * rN;
    double a = (i == l) ? lamN[i] : 0.0;
    for (int j = 0; j < rF; ++j) a = fma(-P[i * rF + j] * lamF[j], P[l * rF + j], a);
    acc = fma(a, a, acc);
  }
  // 2 tr(B G B^T) = 2 sum_i sum_{j,l} B_ij G_jl B_il : one (i, j) per work item
  for (int e = tid; e < rN * rF; e += blockDim.x) {
    const int i = fdiv(e, rF), j = e - i * rF;
    const double bij = P[i * rF + j] * lamF[j];
    double t = 0.0;
    for (int l = 0; l < rF; ++l) t = fma(G[j * rF + l], P[i * rF + l] * lamF[l], t);
    acc = fma(2.0 * bij, t, acc);
  }
  // sum_jl lamF_j lamF_l G_jl^2
  for (int e = tid; e < rF * rF; e += blockDim.x) {
    const int j = fdiv(e, rF), l = e - j * rF;
    const double g = G[e];
    acc = fma(lamF[j] * lamF[l] * g, g, acc);
  }
  acc = warp_sum(acc);
  __syncthreads();
  if ((tid & 31) == 0) scr[tid >> 5] = acc;
  __syncthreads();
  double tot = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += scr[w];
  __syncthreads();
  return tot;
}

// a ring buffer free once the eigensolver passes are done (not V, F, AV)
__device__ __forceinline__ double* buf_free_after_passes(const Inst& d, int iav) {
  return iav == 2 ? d.Y1 : d.Y0;
}

// dynamic shared memory of lrpdhg_iterate_kernel (must match the carve-up below)
inline size_t iterate_smem_bytes(int lds, int zcap, int ycap, int owncap, int nlmax) {
  return (size_t)(5 * lds * (lds + 1) + PDSDP_NTHR + 13 * PDSDP_BMAX + PDSDP_GRAM_SCR + zcap + ycap + owncap) *
             sizeof(double) +
         (size_t)(3 * PDSDP_BMAX + 8 + 20 + zcap + (owncap ? nlmax + 2 : 0)) * sizeof(int) + 64;
}

// eigen block for k wanted pairs plus `extra` guard columns requested by the
// host (Ctl flags bits 8..11: instances whose iterations keep needing several
// filter passes get a wider block, see solver.py)
__device__ int choose_block(int k, int n, int extra) {
  int b = block_for(k, n) + extra;
  return b > n ? n : b;
}

__global__ void __launch_bounds__(PDSDP_NTHR, 1)
lrpdhg_iterate_kernel(const Inst* __restrict__ insts, const Ctl* __restrict__ ctls,
                      const int* __restrict__ active, int step0, int nsteps, int lcap, int zcap, int ycap,
                      int owncap, int nlmax) {
  const int lds = lcap + 1;   // odd stride of the b x b workspaces (no bank conflicts)
  extern __shared__ __align__(16) double smem[];
  cg::cluster_group cl = cg::this_cluster();
  Cta x;
  x.C = (int)cl.num_blocks();
  x.c = (int)cl.block_rank();
  const int inst_id = active[blockIdx.x / x.C];
  // the descriptor lives in shared memory: as a local struct it would sit in
  // (L1-backed) local memory, which every cluster barrier invalidates
  __shared__ __align__(16) Inst d_sm;
  {
    const int nw8 = (int)(sizeof(Inst) / 8);
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(insts + inst_id);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(&d_sm);
    for (int i = threadIdx.x; i < nw8; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const Inst& d = d_sm;
  if (*(volatile int*)d.stopf) return;            // an earlier launch of this chunk ended it
  const int flags0 = ctls[inst_id * PDSDP_KMAX + step0].flags;
  State* st = d.st;
  const int n = d.n, ld = d.ld, tid = threadIdx.x;
  x.r0 = (int)(((long long)n * x.c) / x.C);
  x.r1 = (int)(((long long)n * (x.c + 1)) / x.C);
  x.par = 0;

  __shared__ Prof pf_sm;                 // thread-0 phase timer (PDSDP_TRACE builds only)
  Prof& pf = pf_sm;
#if PDSDP_TRACE
  if (threadIdx.x == 0) {
    g_trace_prof = &pf_sm;
    pf.last = clock64(); pf.cur = 0;
    for (int q = 0; q < 16; ++q) pf.acc[q] = 0;
    pf.ntr = 0;
    pf.cap = PDSDP_TRACE_CAP;
    pf.trace = ((flags0 & 32) && x.c == 0) ? d.st->hdump : nullptr;
    if (flags0 & 64) { pf.trace = d.trace + (size_t)x.c * 2 * PDSDP_TRACE_CTA; pf.cap = PDSDP_TRACE_CTA - 1; }
  }
#else
  (void)flags0;
#endif
  prof_tick(pf, 29);
  __shared__ Sm s_sm;
  Sm& s = s_sm;
  if (threadIdx.x == 0) {
    s.lds = lds;
    double* p = smem;
    const int sq = lcap * lds;
    s.T = p; p += sq;
    s.scr = p; p += PDSDP_NTHR;
    s.theta = p; p += PDSDP_BMAX; s.res = p; p += PDSDP_BMAX; s.lamF = p; p += PDSDP_BMAX;
    s.lamN = p; p += PDSDP_BMAX; s.dsc = p; p += PDSDP_BMAX; s.cs = p; p += 4 * PDSDP_BMAX;
    // red1 receives cluster reductions of up to 3 + r^2 values: beyond 4 BMAX
    // doubles it runs on into gsc (and, above r ~ 57, into the Rayleigh-Ritz
    // workspaces), all of which are idle between a reduction and the reads of
    // its result in the residual phase -- keep red1, gsc, A.. in this order
    s.red1 = p; p += 4 * PDSDP_BMAX;
    s.gsc = p; p += PDSDP_GRAM_SCR;
    // A, Q, L, M are Rayleigh-Ritz workspaces: dead while the filter runs, so
    // the operand staging buffer starts at A and spans them too
    s.A = p; p += sq; s.Q = p; p += sq; s.L = p; p += sq; s.M = p; p += sq;
    s.ys = s.A; p += ycap;
    s.SF = p; p += owncap;
    double* zvs = p; p += zcap;
    int* ip = (int*)p;
    s.perm = ip; ip += PDSDP_BMAX; s.pq = ip; ip += 2 * PDSDP_BMAX; s.flag = ip; ip += 8;
    int* zc = ip; ip += zcap;
    s.szp = ip; ip += (owncap ? nlmax + 2 : 0);
    s.gb = ip; ip += 20;
    s.zc = zc; s.zvs = zvs;
    s.zoff = d.zptr[x.r0];
    s.zstaged = (d.zptr[x.r1] - s.zoff) <= zcap ? 1 : 0;
    int cw = (ycap + 4 * sq) / d.n;
    cw &= ~1;
    if (cw > d.ld) cw = d.ld;
    s.ycw = (cw >= 2) ? cw : 0;
    s.sld = lcap;
    s.ycap = ycap + 4 * sq;
    {
      const int nl = x.r1 - x.r0, sp = own_ystr(lcap);
      s.own = (owncap > 0 && nl * lcap <= owncap && nl <= nlmax && nl * sp <= s.ycap &&
               nl <= PDSDP_OWN_ITEMS * (PDSDP_NTHR / (own_stride(lcap) / 4))) ? 1 : 0;
    }
  }
  __shared__ __align__(8) unsigned long long mbar_sm;   // completion barrier of the operand all-gather
  if (threadIdx.x == 0) mbar_init(&mbar_sm, 1);
  unsigned mphase = 0;
  __syncthreads();

  auto buf = [&](int i) -> double* {
    return i == 0 ? d.V : i == 1 ? d.AV : i == 2 ? d.Y0 : i == 3 ? d.Y1 : d.Y2;
  };
  const int own_base = s.own;
  // launch invariants: Z column indices of the own rows, row pointers, groups
  if (s.zstaged) {
    const int nzl = d.zptr[x.r1] - s.zoff;
    for (int e = tid; e < nzl; e += blockDim.x) const_cast<int*>(static_cast<const int*>(s.zc))[e] = d.zcol[s.zoff + e];
  }
  if (own_base) {
    for (int lr = tid; lr <= x.r1 - x.r0; lr += blockDim.x) s.szp[lr] = d.zptr[x.r0 + lr];
    for (int c = tid; c <= x.C; c += blockDim.x) s.gb[c] = (int)(((long long)n * c) / x.C);
  }
  if (tid == 0) s.gplan = -1;   // the operator step plans its row groups per operand stride
  __syncthreads();

  // Persistent over the chunk: one launch runs the chunk's iterations until
  // the host's control logic may act (the stop flag set by CTA 0 at the end
  // of an iteration); iterations are separated by one cluster barrier, which
  // publishes the iterate to every CTA of the cluster.
  for (int step = step0; step < step0 + nsteps; ++step) {
  const Ctl ctl = ctls[inst_id * PDSDP_KMAX + step];

  // ---------------- prologue: F <- V[:, :rF] (X_k), block setup ----------------
  // flags: bit0 cold start; bit1 the certificate eigenvalue lambda_{r+1} must be
  // accurate (checkpoint iterations); bit2 re-run of the last iteration from
  // the same (X_k, y_k) (F, lamF, Z_k kept) -- used when a checkpoint turns up
  // in an iteration that ran without bit1.
  // Effective rank: X+ keeps only positive eigenpairs among the top r, so
  // when S has far fewer than r positive eigenvalues the block only needs
  // them plus one "sentinel" pair certified non-positive -- then lambda_{r+1}
  // <= sentinel <= 0 and the certificate (n-r) max(lambda_{r+1}, 0) is 0, as
  // in the reference.  The block grows in-kernel whenever the sentinel's Ritz
  // value is positive (Cauchy interlacing: theta_i <= lambda_i).
  const int r_t = ctl.r;
  const bool tight = (ctl.flags & 8) != 0;
  int r = r_t;
  {
    const int np = st->npos;
    if (!tight && (r_t >= np + 8 || min(r_t + 1, n) > lcap)) r = min(r_t, np + 2);
  }
  int k = (r + 1 < n) ? r + 1 : n;
  const bool need_cert = (ctl.flags & 2) != 0;
  // bit3: certificate eigenpair to the kept-pair tolerance (op-level aproj_psd)
  const double cert_tol0 = need_cert ? ((ctl.flags & 8) ? PDSDP_TOL_KEEP : PDSDP_TOL_CERT) : 0.0;
  double cert_tol = (r < r_t) ? -1.0 : cert_tol0;
  const bool rerun = (ctl.flags & 4) != 0;
  const bool cold = !rerun && ((ctl.flags & 1) || st->b == 0);
  const int rF = cold ? 0 : (rerun ? st->rF_used : st->rF);
  const int b_old = cold ? 0 : st->b;
  const int gextra = (ctl.flags >> 8) & 15;
  int b = choose_block(k, n, gextra);
  if (b > lcap) b = lcap;
  if (b < b_old) b = b_old;
  int iav = cold ? 1 : st->iav;   // physical buffer holding AV
  if (iav < 1 || iav > 4) iav = 1;
  bool theta_valid = !cold && st->theta_valid && b == b_old;
  for (int i = tid; i < PDSDP_BMAX; i += blockDim.x) {
    double th = (!cold && i < b_old) ? st->theta[i] : 0.0;
    s.theta[i] = th;
    s.lamF[i] = rerun ? st->lamF[i] : ((i < rF && th > 0.0) ? th : 0.0);
    // dense rank-one rows ride along as extra factor columns of S:
    // -alpha * sig * y_k[row] * u u^T  (column rF + q of F holds u)
    if (i >= rF && i < rF + d.nd) {
      const double* yk0 = (ctl.ypar & 1) ? d.ybuf1 : d.ybuf0;
      const int q = i - rF;
      s.lamF[i] = -d.alpha * d.dsig[q] * yk0[d.drow[q]];
    }
    s.res[i] = (!cold && i < b_old) ? st->res[i] : 1.0e300;
  }
  if (tid == 0) s.own = (own_base && rF + d.nd <= s.sld) ? 1 : 0;
  __syncthreads();
  const int rFx = rF + d.nd;       // factor columns of the operator S = F_x diag(lamF) F_x^T - alpha Z
  // Chebyshev interval floor: Gershgorin bound of -alpha Z, tightened by the
  // Lanczos estimate of lambda_max(Z) when available (zbound.cuh)
  const double lo = (st->zlam_ok == 1.0) ? fmax(st->lo_par[ctl.ypar & 1], -d.alpha * st->zlam)
                                         : st->lo_par[ctl.ypar & 1];
  const double alpha = d.alpha;
  const double* zv = (ctl.ypar & 1) ? d.zbuf1 : d.zbuf0;     // Z_k  = C + M^T y_k
  double* zvn = (ctl.ypar & 1) ? d.zbuf0 : d.zbuf1;          // Z_k+1
  // Z_k values of the own rows: the previous iteration of this launch left
  // them in shared memory (its adjoint gather), otherwise stage them
  if (s.zstaged && (step == step0 || rerun)) {
    const int nzl = d.zptr[x.r1] - s.zoff;
    for (int e = tid; e < nzl; e += blockDim.x) const_cast<double*>(static_cast<const double*>(s.zvs))[e] = zv[s.zoff + e];
  }
  // F <- V[:, :rF] masked by the clip (own rows; also into shared memory).
  // Four loads are issued before their stores: a plain copy loop pays one L2
  // round trip per trip (the stores may alias the loads for the compiler).
  // columns [0, nex) of F still hold V_k-1 and columns [0, nex2) of Vp hold
  // V_k-2: extrapolated start (PDSDP_EXTRAP)
  const int nex = (PDSDP_EXTRAP && !cold && !rerun && b == b_old && st->theta_valid) ? min(st->fvalid, rF) : 0;
  // order 2 while it pays: an order-2 start that needed a second pass (its
  // error feedback is 7x the previous errors against 3x at order 1, which
  // some spectra turn into a period-2 cycle above the tolerance) puts the
  // instance back to order 1 for PDSDP_QRETRY iterations
  const int nex2 = (PDSDP_EXTRAP >= 2 && st->q_age >= (double)PDSDP_QRETRY) ? min(nex, st->pvalid) : 0;
  if (tid == 0) {
    s.pvalid = rerun ? st->pvalid : nex;     // Vp after this prologue (written to the state at the end)
    s.q_used = nex2 > 0;
    g_tolf = (nex2 > 0) ? PDSDP_QTOL : 1.0;
  }
  if (rF > 0) {
    const int tot = (x.r1 - x.r0) * rF;
    const double* srcm = rerun ? d.F : d.V;
    for (int it0 = tid; it0 < tot; it0 += 4 * blockDim.x) {
      double v[4], fo[4], po[4];
      int lr_[4], j_[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int it = it0 + u * blockDim.x;
        lr_[u] = fdiv(min(it, tot - 1), rF);
        j_[u] = min(it, tot - 1) - lr_[u] * rF;
        const size_t o = (size_t)(x.r0 + lr_[u]) * ld + j_[u];
        v[u] = __ldcg(srcm + o);
        fo[u] = (j_[u] < nex) ? __ldcg(d.F + o) : 0.0;
        po[u] = (j_[u] < nex2) ? __ldcg(d.Vp + o) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int it = it0 + u * blockDim.x;
        if (it < tot) {
          const size_t o = (size_t)(x.r0 + lr_[u]) * ld + j_[u];
          const double f = (rerun || s.lamF[j_[u]] != 0.0) ? v[u] : 0.0;
          if (!rerun) d.F[o] = f;
          if (s.own) s.SF[(size_t)lr_[u] * s.sld + j_[u]] = f;
          if (j_[u] < nex) {
            d.V[o] = (j_[u] < nex2) ? 3.0 * (v[u] - fo[u]) + po[u] : 2.0 * v[u] - fo[u];
            if (PDSDP_EXTRAP >= 2) d.Vp[o] = fo[u];
          }
        }
      }
    }
  }
  if (b > b_old)      // fresh block columns (cold start, rank change)
    for (int it = tid; it < (x.r1 - x.r0) * (b - b_old); it += blockDim.x) {
      const int lq_ = fdiv(it, b - b_old);
      const int rho = x.r0 + lq_, j = b_old + it - lq_ * (b - b_old);
      d.V[(size_t)rho * ld + j] = hash_uniform(0x5EEDull + (uint64_t)st->seed, (uint64_t)rho, (uint64_t)j);
    }
  for (int it = tid; it < (x.r1 - x.r0) * d.nd; it += blockDim.x) {
    const int rho = x.r0 + it / d.nd, q = it % d.nd;
    const double u = d.du[(size_t)q * n + rho];
    d.F[(size_t)rho * ld + rF + q] = u;
    if (s.own) s.SF[(size_t)(rho - x.r0) * s.sld + rF + q] = u;
  }
  __syncthreads();
  if (x.c == 0 && tid < PDSDP_BMAX) st->lamF[tid] = s.lamF[tid];
  if (x.c == 0 && tid == 0) st->rF_used = rF;
  int grow_err = 0, since_grow = 0;
  prof_tick(pf, 30);

  // ---------------- eigensolver: warm-started Chebyshev-filtered subspace iteration ----
  bool av_valid = false;
  int passes = 0, matvecs = 0, converged = 0;
  double prev_maxres = 1.0e300, maxres = 1.0e300;
  const int maxpass = ctl.maxpass > 0 ? ctl.maxpass : 60;
  int force_m = -1, msucc = 0, fails = 0, slack = 0;
  const int hint = (int)st->mhint;
  for (int pass = 0; pass < maxpass; ++pass) {
    // ---- pass plan (identical in every thread): degree m, active columns
    //      [c0, c0+bc) to filter, nlock locked (deflated) leading pairs ----
    int m = 0, c0 = 0, bc = b, nlock = 0;
    double fe = 1.0, fc = 0.0, sig1 = 1.0;
    if (theta_valid && b < n) {
      const double scale = fmax(fmax(fabs(s.theta[0]), fabs(lo)), 1e-300);
      const double xnorm = kept_norm_w(s.theta, r, b);
      const Assess as = assess_w(s.theta, s.res, r, b, k, scale, xnorm, cert_tol);
      const bool stale = (pass == 0 && !rerun);   // residuals belong to the previous S
      const double eps_rel = fmax(as.maxres, stale ? (nex > 0 ? PDSDP_STALE_EPS_X : PDSDP_STALE_EPS) : 0.0);
      int mcap = PDSDP_MMAX;
      // leading pairs already converged to the kept tolerance: deflate them
      // and filter the rest of the block (a small spread admits the degree the
      // slow column needs, and the trailing columns track the eigenvalues
      // just below the cut instead of riding along unfiltered)
      int nconv = 0;
      if (!stale && as.last_bad >= 0)
        nconv = leading_ok_w(s.theta, s.res, r, b, as.last_bad, scale, xnorm, cert_tol);
      if (nconv >= 1) {
        nlock = nconv; c0 = nconv; bc = b - nconv;
        mcap = cheb_plan(s.theta, b, lo, s.theta[nconv], s.theta[b - 1], s.theta[as.last_bad], as.rho_k, scale,
                         eps_rel, m, fe, fc, sig1);
        if (m < 2) m = 2;
        if (m > mcap) m = mcap;
      } else if (as.last_bad >= 0 || stale || (!as.cert_bad && !as.tail_bad)) {
        // kept columns; guards filtered too unless that would collapse the block
        int a1 = (as.last_bad >= 0) ? as.last_bad + 1 : r;
        if (a1 > b - 1) a1 = b - 1;
        if (a1 < 1) a1 = 1;
        const double slow = s.theta[(as.last_bad >= 0) ? as.last_bad : a1 - 1];
        double e1, c1, s1, e2, c2, s2;
        int m1, m2;
        const int cap1 = cheb_plan(s.theta, a1, lo, s.theta[0], s.theta[a1], slow, as.rho_k, scale, eps_rel, m1, e1, c1, s1);
        const int cap2 = cheb_plan(s.theta, b, lo, s.theta[0], s.theta[b - 1], slow, as.rho_k, scale, eps_rel, m2, e2, c2, s2);
        int want2 = stale ? (hint > 0 ? hint : 4) : max(m2, 2);
        int want1 = stale ? (hint > 0 ? hint : 4) : max(m1, 2);
        if (cap2 >= min(want2, 6) || (PDSDP_EXTRAP_WHOLE && stale && nex2 > 0)) { m = min(want2, cap2); mcap = cap2; c0 = 0; bc = b; fe = e2; fc = c2; sig1 = s2; }
        else { m = min(want1, cap1); mcap = cap1; c0 = 0; bc = a1; fe = e1; fc = c1; sig1 = s1; }
      } else if (as.cert_bad || as.tail_bad) {
        // kept pairs converged: lock (deflate) them and filter the tail
        nlock = r; c0 = r; bc = b - r;
        const double ct = (cert_tol < 0.0) ? 0.05 * fabs(s.theta[r]) / scale
                                            : fmax(cert_tol, PDSDP_TOL_CERT * 1e-4);
        const double rr = s.res[r] / fmax(ct * scale, 1e-300);
        mcap = cheb_plan(s.theta, b, lo, s.theta[r], s.theta[b - 1], s.theta[r], rr, scale, eps_rel, m, fe, fc, sig1);
        if (m > mcap) m = mcap;
      }
      if (force_m >= 0) m = force_m;                        // retry after a breakdown
      if (m > mcap) m = mcap;
      if (m > PDSDP_MMAX) m = PDSDP_MMAX;
      const int last_bad = as.last_bad;
      if (x.c == 0 && tid == 0 && pass < 32) {
        double* g = st->dbg[pass];
        g[0] = m; g[1] = maxres; g[2] = last_bad; g[3] = c0 + 1000.0 * r; g[4] = bc + 1000.0 * b; g[5] = lo; g[6] = fc - fe;
        g[7] = xnorm;
      }
    }
    force_m = -1;
    prof_tick(pf, 31);
    // ---- Chebyshev filter on the active columns:  Y_m = p_m(S_d) V ----
    int iy = 0;                       // buffer index holding Y_j (0 == V)
    int iyp = -1;                     // buffer holding Y_{j-1}
    // the three buffers other than V and AV (ring for the recurrence)
    auto fre = [&](int t) -> int { const int q = 1 + t; return q >= iav ? q + 1 : q; };
    if (m > 0 && s.own) {
      // own rows of V (the recurrence's Y_0) into the compact multicast source
      const int nl = x.r1 - x.r0;
      const int bcp = own_ystr(bc);   // compact row stride
      const size_t nld = (size_t)n * (ld + 4);
      int ycp = 0;
      bool gram_ready = false;
      if (((bc | c0) & 1) == 0) {
        // bounce through the (idle) staging buffer: cp.async in, 16-byte stores out
        double* yb_ = s.ys;
        const int hp = bc >> 1;
        for (int it = tid; it < nl * hp; it += blockDim.x) {
          const int lr = fdiv(it, hp), j2 = it - lr * hp;
          cp_async16(yb_ + (size_t)lr * bcp + 2 * j2, d.V + (size_t)(x.r0 + lr) * ld + c0 + 2 * j2);
        }
        cp_async_wait_all();
        __syncthreads();
        for (int it = tid; it < nl * hp; it += blockDim.x) {
          const int lr = fdiv(it, hp), j2 = it - lr * hp;
          *reinterpret_cast<double2*>(d.Yc + (size_t)(x.r0 + lr) * bcp + 2 * j2) =
              *reinterpret_cast<const double2*>(yb_ + (size_t)lr * bcp + 2 * j2);
        }
      } else {
        for (int it = tid; it < nl * bc; it += blockDim.x) {
          const int lr = fdiv(it, bc), jj = it - lr * bc;
          d.Yc[(size_t)(x.r0 + lr) * bcp + jj] = d.V[(size_t)(x.r0 + lr) * ld + c0 + jj];
        }
      }
      if (own_lock_sm(rFx, nlock, s.sld))
        for (int it = tid; it < nl * nlock; it += blockDim.x) {
          const int lr = fdiv(it, nlock), t = it - lr * nlock;
          s.SF[(size_t)lr * s.sld + rFx + t] = d.V[(size_t)(x.r0 + lr) * ld + t];
        }
      fence_proxy_async();
      __syncthreads();
      double sg = sig1;
      for (int j = 1; j <= m; ++j) {
        int io = fre((j - 1) % 3);
        if (j == 1) {
          const double ife = fast_rcp(fe), ca = sig1 * ife, cb = -fc * sig1 * ife;
          if (av_valid) {
            for (int it = tid; it < nl * bc; it += blockDim.x) {
              const int lr = fdiv(it, bc), jj = it - lr * bc, jc = c0 + jj;
              const size_t o = (size_t)(x.r0 + lr) * ld + jc;
              const double v = fma(ca, buf(iav)[o], cb * d.V[o]);
              buf(io)[o] = v;
              d.Yc[nld + (size_t)(x.r0 + lr) * bcp + jj] = v;
            }
            fence_proxy_async();
            __syncthreads();
            ycp = 1;
          } else {
            operator_step_own_any(d, x, s, zv, buf(io), c0, bc, rFx, nlock, ca, cb, 0.0, pf, ycp, &mbar_sm, mphase,
                              gram_ready, j < m);
            ++matvecs;
          }
        } else {
          // recurrence coefficients by rcp.approx + Newton (identical in every CTA)
          const double sn = fast_rcp(2.0 * fast_rcp(sig1) - sg), ife = fast_rcp(fe);
          const double ca = 2.0 * sn * ife, cb = -2.0 * sn * fc * ife, cd = -sg * sn;
          operator_step_own_any(d, x, s, zv, buf(io), c0, bc, rFx, nlock, ca, cb, cd, pf, ycp, &mbar_sm, mphase,
                            gram_ready, j < m);
          ++matvecs;
          sg = sn;
        }
        iyp = iy;
        iy = io;
        __syncthreads();
      }
      if (bc < b) {
        for (int it = tid; it < (x.r1 - x.r0) * b; it += blockDim.x) {
          const int lq_ = fdiv(it, b), jj = it - lq_ * b;
          if (jj >= c0 && jj < c0 + bc) continue;
          const size_t o = (size_t)(x.r0 + lq_) * ld + jj;
          buf(iy)[o] = d.V[o];
        }
        __syncthreads();
      }
    } else if (m > 0) {
      double sg = sig1;
      for (int j = 1; j <= m; ++j) {
        int io = fre((j - 1) % 3);
        if (j == 1) {
          const double ife = fast_rcp(fe), ca = sig1 * ife, cb = -fc * sig1 * ife;
          if (av_valid) {
            for (int it = tid; it < (x.r1 - x.r0) * bc; it += blockDim.x) {
              const int lq_ = fdiv(it, bc);
              const size_t o = (size_t)(x.r0 + lq_) * ld + c0 + it - lq_ * bc;
              buf(io)[o] = fma(ca, buf(iav)[o], cb * d.V[o]);
            }
          } else {
            operator_step(d, x, s, zv, d.V, nullptr, buf(io), c0, bc, rFx, nlock, ca, cb, 0.0, pf);
            ++matvecs;
          }
        } else {
          // recurrence coefficients by rcp.approx + Newton (identical in every CTA)
          const double sn = fast_rcp(2.0 * fast_rcp(sig1) - sg), ife = fast_rcp(fe);
          const double ca = 2.0 * sn * ife, cb = -2.0 * sn * fc * ife, cd = -sg * sn;
          operator_step(d, x, s, zv, buf(iy), buf(iyp < 0 ? 0 : iyp), buf(io), c0, bc, rFx, nlock, ca, cb, cd, pf);
          ++matvecs;
          sg = sn;
        }
        iyp = iy;
        iy = io;
        __syncthreads();
      }
      // passive columns ride along unfiltered
      if (bc < b) {
        for (int it = tid; it < (x.r1 - x.r0) * b; it += blockDim.x) {
          const int lq_ = fdiv(it, b), jj = it - lq_ * b;
          if (jj >= c0 && jj < c0 + bc) continue;
          const size_t o = (size_t)(x.r0 + lq_) * ld + jj;
          buf(iy)[o] = d.V[o];
        }
        __syncthreads();
      }
    }
    // ---- R1: G1 = Y^T Y, T = F^T Y ; W = S Y ----
    const int iw = (iy == 0) ? fre(0) : fre((m) % 3);          // free of {Y_m, Y_{m-1}} ring
    int iw1 = -1;
    for (int q2 = 0; q2 < 3; ++q2) if (fre(q2) != iy && fre(q2) != iw) { iw1 = fre(q2); break; }
    if (s.own) {
      // W = S Y through the own-row operator step (multicast all-gather of the
      // block, smem-resident F rows); G1 = Y^T Y rides in the step's reduction
      const int nl = x.r1 - x.r0, bcp = own_ystr(b);   // compact row stride
      prof_mark(pf, 1);
      double* yo = s.ys;   // own rows for the G1 product (staging buffer idle until the step's barrier)
      if ((b & 1) == 0) {
        // global -> shared by cp.async (every transfer in flight, no registers), then
        // shared -> the compact multicast source; a copy loop through registers
        // waits for one L2 round trip per trip
        const int hp = b >> 1;
        for (int it = tid; it < nl * hp; it += blockDim.x) {
          const int lr = fdiv(it, hp), j2 = it - lr * hp;
          cp_async16(yo + (size_t)lr * bcp + 2 * j2, buf(iy) + (size_t)(x.r0 + lr) * ld + 2 * j2);
        }
        cp_async_wait_all();
        __syncthreads();
        for (int it = tid; it < nl * hp; it += blockDim.x) {
          const int lr = fdiv(it, hp), j2 = it - lr * hp;
          *reinterpret_cast<double2*>(d.Yc + (size_t)(x.r0 + lr) * bcp + 2 * j2) =
              *reinterpret_cast<const double2*>(yo + (size_t)lr * bcp + 2 * j2);
        }
      } else {
        for (int it = tid; it < nl * b; it += blockDim.x) {
          const int lr = fdiv(it, b), jj = it - lr * b;
          const double v = buf(iy)[(size_t)(x.r0 + lr) * ld + jj];
          d.Yc[(size_t)(x.r0 + lr) * bcp + jj] = v;
          yo[(size_t)lr * bcp + jj] = v;
        }
      }
      fence_proxy_async();
      __syncthreads();
      // [F_x | Y]^T Y in one Gram: the step's T partial (rows < rFx) and G1 = Y^T Y
      // (rows rFx ..) -- the layout the step's reduction and G1 read
      gram_mma2<true, true, true>(s.SF, s.sld, rFx + b, yo, bcp, b, 0, nl, red_slot(d, x, x.c), s.gsc, yo, bcp, rFx);
      int ycp_rr = 0;
      bool gr = true;
      operator_step_own_any(d, x, s, zv, buf(iw), 0, b, rFx, 0, 1.0, 0.0, 0.0, pf, ycp_rr, &mbar_sm, mphase, gr, false);
      __syncthreads();
      Cta xp = x;
      xp.par ^= 1;    // the step's reduction slot
      for (int i = tid; i < b * b; i += blockDim.x) s.A[fdiv(i, b) * lds + (i - fdiv(i, b) * b)] = cluster_sum(d, xp, rFx * b + i, false);
      __syncthreads();
    } else {
      {
        double* slot = red_slot(d, x, x.c);
        prof_mark(pf, 1);
        gram_mma(buf(iy), b, buf(iy), b, ld, x.r0, x.r1, slot, s.gsc);
        gram_mma(d.F, rFx, buf(iy), b, ld, x.r0, x.r1, slot + b * b, s.gsc);
        // reduce T now; G1 after the product (whose staging buffer overlays A)
        cg::this_cluster().sync();
        for (int i = tid; i < rFx * b; i += blockDim.x) s.T[i] = cluster_sum(d, x, b * b + i, false);
        __syncthreads();
      }
      scale_T(s, rFx, 0, b);
      prof_mark(pf, 3);
      if (s.ycw >= 2) apply_rows_staged(d, x, s, zv, buf(iy), nullptr, buf(iw), 0, b, rFx, 0, 1.0, 0.0, 0.0);
      else apply_rows(d, x, s, zv, buf(iy), nullptr, buf(iw), 0, b, rFx, 0, 1.0, 0.0, 0.0);
      __syncthreads();
      for (int i = tid; i < b * b; i += blockDim.x) s.A[fdiv(i, b) * lds + (i - fdiv(i, b) * b)] = cluster_sum(d, x, i, false);
      x.par ^= 1;
      __syncthreads();
    }
    prof_mark(pf, 8);
    ++matvecs;
    const int nlr = x.r1 - x.r0;
    const bool rsm = 3 * nlmax * b <= ycap;
    double* S0 = s.A + 4 * (size_t)lcap * lds;
    double* S1 = S0 + (size_t)nlr * b;
    double* S2 = S1 + (size_t)nlr * b;
    // one-pass Rayleigh-Ritz when the filtered block is already well
    // conditioned: D G1 D within 0.5/b of identity entrywise (cond <= 3 by
    // Gershgorin), so the pairs of (Y^T S Y, Y^T Y) through L1 are as accurate
    // as CholQR2's, and V = Y D L1^-T Q -- the rotations Y M1, W M1 and the
    // second Gram are skipped
    bool onep = false;
#if PDSDP_ONEPASS_RR
    if (rsm) {
      for (int i = tid; i < b; i += blockDim.x) {
        const double g = s.A[i * lds + i];
        s.dsc[i] = (g > 0.0 && isfinite(g)) ? rsqrt(g) : 0.0;
      }
      __syncthreads();
      const double eta = PDSDP_ONEPASS_ETA / b;
      int big = 0;
      for (int e = tid; e < b * b; e += blockDim.x) {
        const int i = fdiv(e, b), j = e - i * b;
        big |= !(fabs(fma(s.A[i * lds + j] * s.dsc[i], s.dsc[j], (i == j) ? -1.0 : 0.0)) <= eta);
      }
      onep = !__syncthreads_or(big);
    }
#endif
    // ---- small: M1 = D L^-T ----
    bool okc = chol_scaled_rows(s.A, b, lds, s.dsc);
    if (!okc) {
      // breakdown: the filtered block lost rank; retry from V with half the degree
      if (++fails >= 8 || m == 0) break;
      force_m = m / 2;
      __syncthreads();
      continue;
    }
    prof_mark(pf, 9);
    tri_inv_lower_rows(s.A, s.L, b, lds);
    for (int e = tid; e < b * b; e += blockDim.x) {
      int i = fdiv(e, b), j = e - i * b;
      s.M[i * lds + j] = s.dsc[i] * s.L[j * lds + i];   // (L^-1)^T scaled
    }
    __syncthreads();
    bool g2s = false;
    if (onep) {
      prof_mark(pf, 5);
      copy_rows_in(buf(iy) + (size_t)x.r0 * ld, ld, S1, nlr, b);
      copy_rows_in(buf(iw) + (size_t)x.r0 * ld, ld, S2, nlr, b);
      copy_rows_wait();
      __syncthreads();
      gram_mma2<true, true>(S1, b, b, S2, b, b, 0, nlr, red_slot(d, x, x.c), s.gsc);   // H0 = Y^T W
      prof_mark(pf, 4);
      cg::this_cluster().sync();
      for (int i = tid; i < b * b; i += blockDim.x) s.Q[fdiv(i, b) * lds + (i - fdiv(i, b) * b)] = cluster_sum(d, x, i, false);
      x.par ^= 1;
      __syncthreads();
      msucc += m;
      prof_mark(pf, 9);
    } else {
    // Y1 = Y M1 ; W1 = W M1 -- in shared memory (own rows) when they fit
    // after the Rayleigh-Ritz workspaces, else in buf(iav) / buf(iw1)
    prof_mark(pf, 5);
    if (rsm) {
      copy_rows_in(buf(iy) + (size_t)x.r0 * ld, ld, S0, nlr, b);
      copy_rows_wait();
      __syncthreads();
      rot_mma(S0, b, nullptr, 0, s.M, lds, S1, b, nullptr, 0, nlr, b, nullptr, nullptr, nullptr);
      copy_rows_in(buf(iw) + (size_t)x.r0 * ld, ld, S0, nlr, b);
      copy_rows_wait();
      __syncthreads();
      rot_mma(S0, b, nullptr, 0, s.M, lds, S2, b, nullptr, 0, nlr, b, nullptr, nullptr, nullptr);
    } else {
      rotate_rows(d, x, buf(iy), s.M, lds, buf(iav), b);
      rotate_rows(d, x, buf(iw), s.M, lds, buf(iw1), b);
    }
    __syncthreads();
    // ---- R2: G2 = Y1^T Y1, H = Y1^T W1 ----
    {
      double* slot = red_slot(d, x, x.c);
      if (rsm) {
        gram_mma2<true, true>(S1, b, b, S1, b, b, 0, nlr, slot, s.gsc);
        gram_mma2<true, true>(S1, b, b, S2, b, b, 0, nlr, slot + b * b, s.gsc);
      } else {
        gram_mma(buf(iav), b, buf(iav), b, ld, x.r0, x.r1, slot, s.gsc);
        gram_mma(buf(iav), b, buf(iw1), b, ld, x.r0, x.r1, slot + b * b, s.gsc);
      }
      prof_mark(pf, 4);
      cg::this_cluster().sync();
      const int q = 2 * b * b;
      for (int i = tid; i < q; i += blockDim.x) {
        const double acc = cluster_sum(d, x, i, false);
        if (i < b * b) s.A[fdiv(i, b) * lds + (i - fdiv(i, b) * b)] = acc;
        else { int e = i - b * b; s.Q[fdiv(e, b) * lds + (e - fdiv(e, b) * b)] = acc; }
      }
      x.par ^= 1;
      __syncthreads();
    }
    // L2 = chol(G2 scaled); H' = L2^-1 D H D L2^-T ; eig ; B = D L2^-T Qe.
    // After the first CholQR the scaled G2 = D G2 D is I + E with E at the
    // level of u kappa^2; when max|E| <= 1e-5 the second Cholesky is replaced
    // by the series (I + E)^(-1/2) = I - E/2 + 3/8 E^2 + O(E^3) (symmetric
    // K instead of the triangular L2^-1; V^T V = I + O(E^3)).
    prof_mark(pf, 8);
    {
      for (int i = tid; i < b; i += blockDim.x) {
        const double g = s.A[i * lds + i];
        s.dsc[i] = (g > 0.0 && isfinite(g)) ? rsqrt(g) : 0.0;
      }
      __syncthreads();
      int big = 0;
      for (int e = tid; e < b * b; e += blockDim.x) {
        const int i = fdiv(e, b), j = e - i * b;
        const double v = fma(s.A[i * lds + j] * s.dsc[i], s.dsc[j], (i == j) ? -1.0 : 0.0);
        s.L[i * lds + j] = v;
        big |= !(fabs(v) <= 1e-5);
      }
      g2s = !__syncthreads_or(big);
    }
    if (g2s) {
      sm_gemm(s.L, lds, s.L, lds, s.M, lds, b, b, b);            // E^2
      for (int e = tid; e < b * b; e += blockDim.x) {
        const int i = fdiv(e, b), j = e - i * b;
        s.L[i * lds + j] = fma(0.375, s.M[i * lds + j], fma(-0.5, s.L[i * lds + j], (i == j) ? 1.0 : 0.0));
      }
      __syncthreads();
    } else {
      okc = chol_scaled_rows(s.A, b, lds, s.dsc);
      if (!okc) {
        if (++fails >= 8 || m == 0) break;
        force_m = m / 2;
        continue;
      }
    }
    msucc += m;     // total degree of the iteration (the next first pass takes min(hint, spread cap))
    prof_mark(pf, 9);
    if (!g2s) tri_inv_lower_rows(s.A, s.L, b, lds);            // L = L2^-1
    }
    prof_mark(pf, 10);
    for (int e = tid; e < b * b; e += blockDim.x) {   // Q <- D H D
      int i = fdiv(e, b), j = e - i * b;
      s.Q[i * lds + j] *= s.dsc[i] * s.dsc[j];
    }
    __syncthreads();
    sm_gemm(s.L, lds, s.Q, lds, s.M, lds, b, b, b);            // M = L^-1 (DHD)
    for (int e = tid; e < b * b; e += blockDim.x) {           // A = M L^-T
      int i = fdiv(e, b), j = e - i * b;
      double acc = 0.0;
      for (int t = 0; t < b; ++t) acc += s.M[i * lds + t] * s.L[j * lds + t];
      s.A[i * lds + j] = acc;
    }
    __syncthreads();
    for (int e = tid; e < b * b; e += blockDim.x) {           // symmetrise
      int i = fdiv(e, b), j = e - i * b;
      if (j > i) { double v = 0.5 * (s.A[i * lds + j] + s.A[j * lds + i]); s.A[i * lds + j] = v; s.A[j * lds + i] = v; }
    }
    __syncthreads();
    if ((ctl.flags & 16) && x.c == 0) {
      for (int e = tid; e < b * b; e += blockDim.x) st->hdump[e] = s.A[fdiv(e, b) * lds + (e - fdiv(e, b) * b)];
      if (tid == 0) st->hdump[PDSDP_BMAX * PDSDP_BMAX] = b;
    }
    prof_mark(pf, 11);
    // pairs among the trailing guard columns only need loose accuracy (their
    // Ritz pairs are not used; residuals are recomputed honestly below)
    double *Aj, *Qj;
    // block-pair updates pay off once the per-element traffic dominates the
    // per-round latency (tools/microbench/small_dense_probe.cu: 1.4x at b = 28)
    if (b >= PDSDP_JAC4_MIN)
      jacobi_eig4(s.A, s.M, s.Q, s.T, b, lds, s.cs, reinterpret_cast<int*>(static_cast<double*>(s.gsc)), s.flag, need_cert ? b : min(b, r + 1), &Aj, &Qj);
    else
      jacobi_eig3(s.A, s.M, s.Q, s.T, b, lds, s.cs, reinterpret_cast<int*>(static_cast<double*>(s.gsc)), s.flag, need_cert ? b : min(b, r + 1), &Aj, &Qj);
    prof_mark(pf, 12);
#if PDSDP_TRACE
    if (x.c == 0 && tid == 0) st->prof[15] += s.flag[0];   // Jacobi sweeps
#endif
    sort_desc(Aj, b, lds, s.theta, s.perm);
    // B = D L^-T Q[:, perm]  -> the Jacobi scratch that does not hold Q
    double* Bm = (Qj == s.Q) ? s.M : s.Q;
    for (int e = tid; e < b * b; e += blockDim.x) {
      int i = fdiv(e, b), j = e - i * b;
      const int pj = s.perm[j];
      double acc = 0.0;
      for (int t = g2s ? 0 : i; t < b; ++t) acc += s.L[t * lds + i] * Qj[t * lds + pj];   // L2^-T (lower) or K
      Bm[i * lds + j] = s.dsc[i] * acc;
    }
    __syncthreads();
    // V = Y1 B ; AV = W1 B  (AV goes to buf(iw), which becomes the AV buffer)
    prof_mark(pf, 5);
    if (rsm) {
      // V = Y1 B, AV = W1 B and the Ritz residual partials in one DMMA sweep
      rot_mma(S1, b, S2, b, Bm, lds, d.V + (size_t)x.r0 * ld, ld, buf(iw) + (size_t)x.r0 * ld, ld, nlr, b,
              s.theta, red_slot(d, x, x.c), s.gsc);
      prof_mark(pf, 4);
    } else {
      rotate_rows(d, x, buf(iav), Bm, lds, d.V, b);
      rotate_rows(d, x, buf(iw1), Bm, lds, buf(iw), b);
      __syncthreads();
      prof_mark(pf, 4);
      colres_partial(buf(iw), d.V, s.theta, b, ld, x.r0, x.r1, red_slot(d, x, x.c), s.scr);
    }
    iav = iw;
    av_valid = true;
    theta_valid = true;
    // ---- R3: residual norms ----
    cluster_reduce(d, x, b, 0, s.red1);
    prof_tick(pf, 70);
    ++passes;
    {
      double scale = fmax(fmax(fabs(s.theta[0]), fabs(lo)), 1e-300);
      const double xnorm = kept_norm_w(s.theta, r, b);
      for (int i = tid; i < b; i += blockDim.x) s.res[i] = sqrt(fmax(s.red1[i], 0.0));
      __syncthreads();
      const Assess as = assess_w(s.theta, s.res, r, b, k, scale, xnorm, cert_tol);
      prof_tick(pf, 71);
      maxres = as.maxres;
      ++since_grow;
      if (r < r_t) {
        // effective-rank block: grow when the sentinel is positive, or when it
        // will not certify (an eigenvalue at ~0 -- move the sentinel deeper)
        int np = 0;
        for (int i = 0; i < b; ++i) np += (s.theta[i] > 0.0) ? 1 : 0;
        const bool sent_ok = s.theta[r] < 0.0 && s.res[r] <= 0.1 * -s.theta[r];
        if (s.theta[r] > 0.0 || (!sent_ok && since_grow >= 4)) {
          const int rn = min(r_t, max(np + 2, r + 4));
          const int kn = min(rn + 1, n);
          if (kn > lcap) { grow_err = 1; break; }
          int bn = choose_block(kn, n, gextra);
          if (bn > lcap) bn = lcap;
          if (bn < b) bn = b;
          __syncthreads();
          for (int it = tid; it < (x.r1 - x.r0) * bn; it += blockDim.x) {
            const int rho = x.r0 + it / bn, j = it % bn;
            if (j >= b) d.V[(size_t)rho * ld + j] = hash_uniform(0x5EEDull + (uint64_t)st->seed, (uint64_t)rho, (uint64_t)j);
          }
          for (int i = b + tid; i < bn; i += blockDim.x) { s.theta[i] = 0.0; s.res[i] = 1.0e300; }
          r = rn; k = kn; b = bn;
          cert_tol = (r < r_t) ? -1.0 : cert_tol0;
          theta_valid = false;
          av_valid = false;
          since_grow = 0;
          prev_maxres = 1.0e300;
          __syncthreads();
          continue;
        }
      }
      // a block that was not filtered in this pass (cold RR) is not trusted
      if (as.last_bad < 0 && !as.cert_bad && !as.tail_bad && (m > 0 || b >= n)) {
        converged = 1;
        // degrees of slack: how many fewer filter degrees would still have met
        // each kept column's tolerance (Chebyshev gain acosh(t) per degree)
        if (m > 0 && pass == 0) {
          double sl = 1.0e300;
          const double tol = g_tolf * fmax(PDSDP_TOL_KEEP * scale, PDSDP_TOL_X * xnorm);
          const double ife = fast_rcp(fe);
          for (int i = (tid & 31); i < r && i < b; i += 32) {
            const double t = (s.theta[i] - fc) * ife;
            if (t <= 1.0 + 1e-6) { sl = 0.0; continue; }
            sl = fmin(sl, (double)__fdividef((float)plan_log(tol * fast_rcp(fmax(s.res[i], 1e-300))), (float)plan_acosh(t)));
          }
          sl = -warp_max(-sl);
          slack = (sl > 0.0 && sl < 64.0) ? (int)floor(sl) : (sl >= 64.0 ? 64 : 0);
        }
        break;
      }
      // stagnation at the rounding floor
      if (pass >= 2 && maxres > 0.5 * prev_maxres && maxres < 1e-10) { converged = 2; break; }
      prev_maxres = maxres;
    }
  }
  prof_tick(pf, 72);
  for (int i = tid; i < PDSDP_BMAX; i += blockDim.x) s.lamN[i] = (i < r && i < b && s.theta[i] > 0.0) ? s.theta[i] : 0.0;
  __syncthreads();

  prof_mark(pf, 6);
  // ---------------- dual step: y+ = u - alpha proj_box(u/alpha) ----------------
  const double* yk = ctl.ypar ? d.ybuf1 : d.ybuf0;
  double* yn = ctl.ypar ? d.ybuf0 : d.ybuf1;
  const int rN = (r < b) ? r : b;
  // Own rows of V (= X_k+1's factor) into shared memory for the residual
  // algebra below (P = V^T F, F_perp = F - V P, G = F_perp^T F_perp): the
  // staging area is idle after the eigensolver, and Gram products / row
  // updates fed from L2 wait one round trip per step.  Four loads in flight.
  const int nlo = x.r1 - x.r0;
  const bool tsm = s.own && 3 * nlmax * lcap <= ycap;
  double* SV = s.A + 4 * (size_t)lcap * lds;      // nlo x rN
  double* SFp = SV + (size_t)nlo * lcap;          // nlo x rF
  if (tsm) {
    const int tot = nlo * rN;
    for (int it0 = tid; it0 < tot; it0 += 4 * blockDim.x) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int it = min(it0 + u * (int)blockDim.x, tot - 1);
        const int lr = fdiv(it, rN);
        v[u] = __ldcg(d.V + (size_t)(x.r0 + lr) * ld + (it - lr * rN));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int it = it0 + u * blockDim.x;
        if (it < tot) SV[it] = v[u];
      }
    }
    // visible to the Gram product after the dual step's barrier
  }
  // dense rank-one rows: <D, X> = sig u^T X u from p = V^T u (X+) and q = F^T u (X_k)
  __shared__ double dsum_sm[2 * PDSDP_NDMAX];   // [2q]: sig u^T(2X+ - X)u, [2q+1]: sig u^T(X+ - X)u
  if (d.nd > 0) {
    const int nq = rN + rF, qt = d.nd * nq;
    const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
    double* slot = red_slot(d, x, x.c);
    for (int o = warp; o < qt; o += nw) {
      const int q = o / nq, l = o % nq;
      const double* U = (l < rN) ? d.V + l : d.F + (l - rN);
      const double* u = d.du + (size_t)q * n;
      double a = 0.0;
      for (int rho = x.r0 + lane; rho < x.r1; rho += 32) a = fma(U[(size_t)rho * ld], u[rho], a);
      a = warp_sum(a);
      if (lane == 0) slot[o] = a;
    }
    __syncthreads();
    cluster_reduce(d, x, qt, 0, s.red1);
    if (tid < d.nd) {
      double xn = 0.0, xo = 0.0;
      for (int l = 0; l < rN; ++l) { const double pv = s.red1[tid * nq + l]; xn = fma(s.lamN[l] * pv, pv, xn); }
      for (int l = 0; l < rF; ++l) { const double qv = s.red1[tid * nq + rN + l]; xo = fma(s.lamF[l] * qv, qv, xo); }
      dsum_sm[2 * tid] = d.dsig[tid] * (2.0 * xn - xo);
      dsum_sm[2 * tid + 1] = d.dsig[tid] * (xn - xo);
    }
    __syncthreads();
  }
  double ed2 = 0.0, fin = 1.0, dysd = 0.0;   // dysd: <dy, M(X+ - X)> = <M^T dy, dX>
  prof_tick(pf, 60);
  {
    const int G = d.group;
    const int gsh = __ffs(G) - 1;                 // G is a power of two (<= 32)
    const int lane = tid & 31, sub = lane & (G - 1);
    const int gid = tid >> gsh, ng = blockDim.x >> gsh;
    const int a0 = d.asplit[x.c], a1 = d.asplit[x.c + 1];
    for (int i0 = a0; i0 < a1; i0 += ng) {
      const int i = i0 + gid;
      double s2 = 0.0, sd = 0.0;
      if (i < a1) {
        for (int e = __ldg(d.aptr + i) + sub; e < __ldg(d.aptr + i + 1); e += G) {
          const int p = __ldg(d.ai + e), q = __ldg(d.aj + e);
          const double* Vp = d.V + (size_t)p * ld; const double* Vq = d.V + (size_t)q * ld;
          const double* Fp = d.F + (size_t)p * ld; const double* Fq = d.F + (size_t)q * ld;
          double xn = 0.0, xo = 0.0;
          for (int l = 0; l < rN; ++l) if (s.lamN[l] != 0.0) xn = fma(Vp[l] * s.lamN[l], Vq[l], xn);
          for (int l = 0; l < rF; ++l) if (s.lamF[l] != 0.0) xo = fma(Fp[l] * s.lamF[l], Fq[l], xo);
          const double g = __ldg(d.ag + e);
          s2 = fma(g, 2.0 * xn - xo, s2);
          sd = fma(g, xn - xo, sd);
        }
      }
      for (int o = G >> 1; o > 0; o >>= 1) {
        s2 += __shfl_down_sync(0xffffffffu, s2, o, G);
        sd += __shfl_down_sync(0xffffffffu, sd, o, G);
      }
      if (i < a1 && sub == 0) {
        for (int q = 0; q < d.nd; ++q)
          if (i == d.drow[q]) { s2 = dsum_sm[2 * q]; sd = dsum_sm[2 * q + 1]; }
        const double u = yk[i] + alpha * s2;
        const double pr = (i < d.m) ? d.bv[i] : fmin(u / alpha, d.hv[i - d.m]);
        const double ynew = u - alpha * pr;
        const double dyi = ynew - yk[i];
        yn[i] = ynew;
        d.dy[i] = dyi;
        const double t = dyi / alpha - sd;
        ed2 = fma(t, t, ed2);
        dysd = fma(dyi, sd, dysd);
        if (!isfinite(ynew)) fin = 0.0;
      }
    }
  }
  prof_tick(pf, 61);
  // block reduce ed2, dysd (sums), fin (min -> max of negatives)
  {
    double v = warp_sum(ed2);
    double v2 = warp_sum(dysd);
    double f = fin;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) f = fmin(f, __shfl_xor_sync(0xffffffffu, f, o));
    if ((tid & 31) == 0) { s.scr[tid >> 5] = v; s.scr[32 + (tid >> 5)] = f; s.scr[64 + (tid >> 5)] = v2; }
    __syncthreads();
    // P = V^T F (own rows) rides along: the dense part of the primal residual
    // is evaluated in factored form (see dense_residual_lowrank)
    prof_tick(pf, 50);
    if (tsm) gram_mma2<true, true>(SV, rN, rN, s.SF, s.sld, rF, 0, nlo, red_slot(d, x, x.c) + 2, s.gsc);
    else gram_mma(d.V, rN, d.F, rF, ld, x.r0, x.r1, red_slot(d, x, x.c) + 2, s.gsc);
    prof_tick(pf, 51);
    if (tid == 0) {
      double a = 0.0, a2 = 0.0, ff = 1.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a += s.scr[w]; a2 += s.scr[64 + w]; ff = fmin(ff, s.scr[32 + w]); }
      double* slot = red_slot(d, x, x.c);
      slot[0] = a;
      slot[1] = a2;
      slot[2 + rN * rF] = -ff;   // max of -fin
    }
    __syncthreads();
  }
  cluster_reduce(d, x, 2 + rN * rF, 1, s.red1);
  const double ed2_tot = s.red1[0];
  const double dysd_tot = s.red1[1];
  double fin_tot = -s.red1[2 + rN * rF];
  // keep P (rN x rF, row-major) and form the own rows of F_perp = F - V P
  // in a free ring buffer
  double* Pm = s.T;
  for (int i = tid; i < rN * rF; i += blockDim.x) Pm[i] = s.red1[2 + i];
  double* Fp = buf_free_after_passes(d, iav);
  __syncthreads();
  if (tsm) {
    for (int it = tid; it < nlo * rF; it += blockDim.x) {
      const int lr = fdiv(it, rF), j = it - lr * rF;
      const double* Vr = SV + (size_t)lr * rN;
      double a = s.SF[(size_t)lr * s.sld + j];
      for (int l = 0; l < rN; ++l) a = fma(-Vr[l], Pm[l * rF + j], a);
      SFp[it] = a;
    }
  } else {
    for (int it = tid; it < (x.r1 - x.r0) * rF; it += blockDim.x) {
      const int lq_ = fdiv(it, rF);
      const int rho = x.r0 + lq_, j = it - lq_ * rF;
      const double* Vr = d.V + (size_t)rho * ld;
      double a = d.F[(size_t)rho * ld + j];
      for (int l = 0; l < rN; ++l) a = fma(-Vr[l], Pm[l * rF + j], a);
      Fp[(size_t)rho * ld + j] = a;
    }
  }
  __syncthreads();
  prof_tick(pf, 53);
  for (int i = 0; i < rN; ++i) if (s.theta[i] > 0.0 && !isfinite(s.theta[i])) fin_tot = 0.0;

  prof_mark(pf, 7);
  // ---------------- adjoint gather: Z_{k+1} = C + M^T y+, support correction ----------------
  double corr = 0.0;
  double cu[PDSDP_NDMAX] = {0.0, 0.0};   // <M^T dy (sparse part), u u^T> per dense row
  {
    // the slot tables are read-only for the kernel's lifetime (__ldg: the
    // loads may move ahead of the stores below); y+ / dy come from other
    // CTAs of the cluster (coherent L2 loads)
    // only the slots M^T y touches change (the others hold C in both Z
    // buffers and in the staged copy)
    const int k0 = __ldg(d.dptr + x.r0), k1 = __ldg(d.dptr + x.r1);
    double* zsm = s.zstaged ? const_cast<double*>(static_cast<const double*>(s.zvs)) - s.zoff : nullptr;   // Z_k is dead: keep Z_k+1 here too
    for (int kk = k0 + tid; kk < k1; kk += blockDim.x) {
      const int e = __ldg(d.dslot + kk);
      double z = __ldg(d.cval + e), a = 0.0;
      const int t0 = __ldg(d.tptr + e), t1 = __ldg(d.tptr + e + 1);
      for (int t = t0; t < t1; ++t) {
        const int row = __ldg(d.trow + t);
        const double cf = __ldg(d.tcoef + t);
        z = fma(__ldcg(yn + row), cf, z);
        a = fma(__ldcg(d.dy + row), cf, a);
      }
      zvn[e] = z;
      if (zsm) zsm[e] = z;
      const int i = __ldg(d.zrow + e), j = __ldg(d.zcol + e);
      if (j >= i) {
        const double w = (i == j) ? 1.0 : 2.0;
        corr = fma(w * a, a, corr);
        for (int q = 0; q < d.nd; ++q) cu[q] = fma(w * a, d.du[(size_t)q * n + i] * d.du[(size_t)q * n + j], cu[q]);
      }
    }
  }
  prof_tick(pf, 80);
  __syncthreads();
  prof_tick(pf, 81);
  double gmax = 0.0;
  {
    const double* zsrc = s.zstaged ? (const double*)s.zvs - s.zoff : zvn;
    for (int rho = x.r0 + tid; rho < x.r1; rho += blockDim.x) {
      double sacc = __ldg(d.zsabs + rho);
      for (int kk = __ldg(d.dptr + rho); kk < __ldg(d.dptr + rho + 1); ++kk) sacc += fabs(zsrc[__ldg(d.dslot + kk)]);
      gmax = fmax(gmax, sacc);
    }
  }
  prof_tick(pf, 82);
  {
    double v = warp_sum(corr);
    double g = gmax;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) g = fmax(g, __shfl_xor_sync(0xffffffffu, g, o));
    double cw[PDSDP_NDMAX];
    for (int q = 0; q < d.nd; ++q) cw[q] = warp_sum(cu[q]);
    if ((tid & 31) == 0) {
      s.scr[tid >> 5] = v; s.scr[32 + (tid >> 5)] = g;
      for (int q = 0; q < d.nd; ++q) s.scr[64 + 32 * q + (tid >> 5)] = cw[q];
    }
    __syncthreads();
    prof_tick(pf, 54);
    if (tsm) gram_mma2<true, true>(SFp, rF, rF, SFp, rF, rF, 0, nlo, red_slot(d, x, x.c) + 1 + d.nd, s.gsc);
    else gram_mma(Fp, rF, Fp, rF, ld, x.r0, x.r1, red_slot(d, x, x.c) + 1 + d.nd, s.gsc);
    prof_tick(pf, 55);
    if (tid == 0) {
      double a = 0.0, gg = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a += s.scr[w]; gg = fmax(gg, s.scr[32 + w]); }
      double* slot = red_slot(d, x, x.c);
      slot[0] = a;
      for (int q = 0; q < d.nd; ++q) {
        double c = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) c += s.scr[64 + 32 * q + w];
        slot[1 + q] = c;
      }
      slot[1 + d.nd + rF * rF] = gg;
    }
    __syncthreads();
  }
  cluster_reduce(d, x, 1 + d.nd + rF * rF, 1, s.red1);
  // dense part ||dX||_F^2 of the primal residual from P and G (CTA 0 reports)
  const double dense_a2 = (x.c == 0) ? dense_residual_lowrank(Pm, s.red1 + 1 + d.nd, s.lamN, s.lamF, rN, rF, s.scr)
                                     : 0.0;
  prof_tick(pf, 57);
  // Support correction of the primal residual  eps_p^2 = ||dX/alpha||^2 + corr,
  // corr = ||A||^2 - 2 <A, dX>/alpha with A = M^T dy; the cross term is
  // <dy, M(dX)> from the dual step (adjoint identity).  Dense rank-one rows:
  // A = A_s + sum_q dlt_q u_q u_q^T, dlt_q = sig_q dy_q, so
  //   ||A||^2 = ||A_s||^2 + 2 sum_q dlt_q <A_s, u_q u_q^T> + sum_{q,l} dlt_q dlt_l (u_q^T u_l)^2,
  // and lambda_max(Z+) <= gersh(Z_s) + sum_q max(0, sig_q y+_q) ||u_q||^2.
  double corr_tot = s.red1[0] - 2.0 * dysd_tot / alpha, gmax_tot = s.red1[1 + d.nd + rF * rF];
  for (int q = 0; q < d.nd; ++q) {
    const double dyq = d.dy[d.drow[q]], dlt = d.dsig[q] * dyq;
    corr_tot += 2.0 * dlt * s.red1[1 + q];
    for (int l = 0; l < d.nd; ++l) corr_tot += dlt * d.dsig[l] * d.dy[d.drow[l]] * d.duu[q * PDSDP_NDMAX + l];
    gmax_tot += fmax(0.0, d.dsig[q] * yn[d.drow[q]]) * d.dun2[q];
  }

  // ---------------- epilogue: state for the next iteration + scalars ----------------
  prof_mark(pf, 0);
#if PDSDP_TRACE
  if (x.c == 0 && tid == 0) {
    for (int q = 0; q < 15; ++q) st->prof[q] = (double)pf.acc[q];
    if (pf.trace && !(ctl.flags & 64)) { prof_tick(pf, 99); st->hdump[PDSDP_BMAX * PDSDP_BMAX + 7] = pf.ntr; }
  }
  if (tid == 0 && (ctl.flags & 64)) {
    prof_tick(pf, 99);
    pf.trace[2 * PDSDP_TRACE_CTA - 1] = pf.ntr;
  }
#endif
  if (x.c == 0) {
    for (int i = tid; i < PDSDP_BMAX; i += blockDim.x) {
      st->theta[i] = (i < b) ? s.theta[i] : 0.0;
      st->res[i] = (i < b) ? s.res[i] : 0.0;
      st->lamN[i] = s.lamN[i];
    }
    if (tid == 0) {
      st->b = b;
      st->rF = rN;
      st->r_cur = r;
      int np = 0;
      for (int i = 0; i < rN; ++i) np += (s.theta[i] > 0.0) ? 1 : 0;
      st->npos = np;
      st->theta_valid = theta_valid ? 1 : 0;
      {   // leading columns of F (this iteration's X_k factor) that were not clipped
        int fv = 0;
        while (fv < rF && s.lamF[fv] != 0.0) ++fv;
        st->fvalid = fv;
        st->pvalid = s.pvalid;
      }
      // degree hint for the next iteration's first pass: after a single-pass
      // convergence drop the measured slack (less a safety degree), else the
      // total degree this iteration needed.  Residuals at the rounding floor
      // (~64 eps scale; the usual case after an extrapolated start) show no
      // slack however many degrees were surplus, so without measured slack
      // the hint is probed one degree down; a probe that costs a second pass
      // is not repeated for PDSDP_PROBE_AGE iterations.
      if (!rerun && msucc > 0) {
        const int hused = (int)st->mhint;
        int fl = (int)st->mfloor, age = (int)st->mfloor_age + 1;
        int h;
        if (passes == 1 && converged == 1 && fails == 0) {
          h = max(PDSDP_HINT_MIN, msucc - max(0, slack - PDSDP_HINT_SAFETY));
          if (PDSDP_PROBE_AGE > 0 && h == msucc && msucc > PDSDP_HINT_MIN) {
            if (age > PDSDP_PROBE_AGE) fl = 0;
            if (msucc - 1 >= fl) h = msucc - 1;
          }
        } else {
          h = msucc;
          if (hused > 0) { fl = hused + 1; age = 0; }
        }
        st->mhint = h;
        st->mfloor = fl;
        st->mfloor_age = min(age, 1 << 20);
        st->q_age = (s.q_used && (passes > 1 || fails > 0)) ? 0.0 : fmin(st->q_age + 1.0, 1048576.0);
      }
      st->iav = iav;
      st->ed2 = ed2_tot;
      st->corr = corr_tot;
      st->lo_par[(ctl.ypar & 1) ^ 1] = -alpha * gmax_tot;
      st->finite = fin_tot;
      double* o = d.out + step * PDSDP_OUT_LEN;
      o[O_LAM] = s.theta[k - 1];
      o[O_FIN] = fin_tot;
      o[O_PASSES] = passes;
      o[O_MATVECS] = matvecs;
      o[O_EIGCONV] = converged;
      o[O_EIGRES] = maxres;
      o[O_ED2] = ed2_tot;
      o[O_CORR] = corr_tot;
      o[O_BLK] = b;
      o[O_ERR] = grow_err;
      // primal / dual residuals (reference pdhg.py:198-208)
      const double dense = dense_a2 / (alpha * alpha);
      const double ep = sqrt(fmax(dense + corr_tot, 0.0)), ed = sqrt(fmax(ed2_tot, 0.0));
      o[O_DENSE] = dense;
      o[O_EPS_P] = ep;
      o[O_EPS_D] = ed;
      o[O_DONE] = 1.0;
      // pause the chunk where the host's control logic may act (lowrank.py:145-185)
      const double ec = ep + ed;
      if (grow_err || fin_tot != 1.0 || ec <= ctl.conv_thr || ec >= ctl.stall_thr) *d.stopf = 1;
    }
  }
  // publish the iterate (and the stop flag) to the whole cluster
  cg::this_cluster().sync();
  if (*(volatile int*)d.stopf) break;
  }   // step loop
}

}  // namespace pdsdp
