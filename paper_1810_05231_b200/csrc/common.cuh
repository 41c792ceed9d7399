// Shared device-side definitions for the B200 LR-PD-SDP hot path.
//
// Layout in HBM (per SDP instance, everything FP64, row-major n x ld blocks):
//   V, AV        Ritz basis of the current PSD-projection argument and S*V
//   Yb[0..2]     Chebyshev filter recurrence buffers
//   F            factor of the current iterate X_k = F diag(lamF) F^T
//   Z CSR        sparse symmetric matrix  Z = C + M^T(y)  in dense (i, j)
//                coordinates (both triangles), values refreshed every
//                iteration by the adjoint gather; pattern = union of the
//                patterns of C and of every constraint row.
// The projection argument S = X_k - alpha (C + M^T y) is never formed:
//     S * Y = F (lamF .* (F^T Y)) - alpha * Z * Y
// which is exact because X_k is the rank-r truncated projection of the
// previous step (reference symmat.py:212-220 builds it as sum lam u u^T).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define PDSDP_BMAX 64          // largest eigen block (k = r+1 plus guard vectors)
#ifndef PDSDP_NTHR
#define PDSDP_NTHR 384         // threads per CTA of the cluster kernel (168 registers each)
#endif
#ifndef PDSDP_CTA_ROWS
#define PDSDP_CTA_ROWS 128     // cluster size: smallest power of 2 with C * CTA_ROWS >= n (C <= 16)
#endif
#define PDSDP_RED_MAX (2 * PDSDP_BMAX * PDSDP_BMAX + 64)
#define PDSDP_OUT_LEN 16       // doubles per instance and step in the host-mapped output
#define PDSDP_KMAX 128         // iterations per pdsdp_iterate_many call
#define PDSDP_NDMAX 2          // dense rank-one constraint rows handled as vectors

// Eigen block for k = r+1 wanted pairs: k plus max(GUARD_MIN, k / GUARD_DIV)
// guard columns, rounded up to BLOCK_ROUND, <= min(BMAX, n).  One guard
// (b = 12 at r = 10, 22 at r = 20) measured 11% faster on config 2 than
// max(4, k/4) (16 / 28): the per-column cost of every operator step and
// Rayleigh-Ritz pass outweighs the slower convergence (profiles/r01s4_block_sweep.txt).
#ifndef PDSDP_GUARD_MIN
#define PDSDP_GUARD_MIN 1
#endif
#ifndef PDSDP_GUARD_DIV
#define PDSDP_GUARD_DIV 100
#endif
#ifndef PDSDP_BLOCK_ROUND
#define PDSDP_BLOCK_ROUND 2
#endif

namespace pdsdp {

__host__ __device__ inline int block_for(int k, int n) {
  int g = k / PDSDP_GUARD_DIV;
  if (g < PDSDP_GUARD_MIN) g = PDSDP_GUARD_MIN;
  int b = (k + g + PDSDP_BLOCK_ROUND - 1) / PDSDP_BLOCK_ROUND * PDSDP_BLOCK_ROUND;
  if (b > PDSDP_BMAX) b = PDSDP_BMAX;
  if (b > n) b = n;
  return b;
}

struct State {
  int b;            // current eigen block size
  int rF;           // columns of the factor produced by the last iteration
  int theta_valid;  // theta[0..b) are Ritz values of the current V
  int iav;          // physical buffer (1..4) holding S*V
  int rF_used;      // columns of F (= X_k) used by the last iteration
  int r_cur;        // columns of V (= X_k+1) produced by the last iteration
  int npos;         // positive kept Ritz values of the last iteration (effective-rank hint)
  int fvalid;       // leading columns of F holding eigenvectors of the iteration before (not clipped to zero)
  int pvalid;       // leading columns of Vp holding the eigenvectors of two iterations before
  int pad2;
  double theta[PDSDP_BMAX];
  double res[PDSDP_BMAX];
  double lamF[PDSDP_BMAX];   // eigenvalues of X_k   (clipped)
  double lamN[PDSDP_BMAX];   // eigenvalues of X_k+1 (clipped)
  double lo_par[2]; // lower bound of spec(S) for Z in zbuf[par] (Chebyshev interval)
  double ed2;       // sum (dy/alpha - M dX)^2
  double corr;      // sparse-support correction of the primal residual
  double finite;    // 1 when y+ and theta are finite
  double seed;
  double mhint;     // total filter degree used by the previous iteration
  double mfloor;    // first-pass degree below which a probe of the hint failed recently
  double mfloor_age;  // iterations since that failure
  double q_age;     // iterations since an order-2 extrapolated start last needed a second pass (or since the reset)
  double dbg[32][8];  // per pass: m, worst rel residual, slow column, theta, t, lo, cut, xnorm
  double prof[16];    // SM cycles of CTA 0 per phase in the last launch
  double hdump[PDSDP_BMAX * PDSDP_BMAX + 8];  // diagnostic: last projected matrix H' (flag bit4)
  double zlam;        // Lanczos estimate of lambda_max(Z) plus margin (zbound.cuh)
  double zlam_ok;     // 1 when zlam is valid
};

// thread-0 phase timer (clock64 deltas; diagnostic only).  With a trace
// buffer (flag bit 5, CTA 0) every mark / tick is also logged as
// (label, cycle) pairs for a per-step timeline.
#define PDSDP_TRACE_CAP 2040
#define PDSDP_TRACE_CTA 1024
// Pointer into this CTA's dynamic shared memory.  Workspace pointers are
// carved out once and kept in a shared struct; loaded back from there, the
// compiler no longer knows their address space and emits generic 64-bit
// loads (LD.E, long scoreboard).  ShPtr keeps the byte offset instead and
// rebuilds the pointer from the extern shared array on every use, so the
// accesses compile to LDS/STS with 32-bit addressing.  (An assumed
// __isShared() on the generic pointer miscompiles in cluster launches.)
extern __shared__ __align__(16) unsigned char pdsdp_dsm[];
template <class T>
struct ShPtr {
  unsigned off;
  __device__ __forceinline__ ShPtr& operator=(T* q) {
    off = (unsigned)(reinterpret_cast<const unsigned char*>(q) - pdsdp_dsm);
    return *this;
  }
  __device__ __forceinline__ operator T*() const { return reinterpret_cast<T*>(pdsdp_dsm + off); }
};
// The same pointer rebuilt from the extern shared array (p must point into
// this CTA's dynamic shared memory): accesses through it compile to LDS/STS.
template <class T>
__device__ __forceinline__ T* as_shared(T* p) {
  const unsigned o = (unsigned)__cvta_generic_to_shared(p) - (unsigned)__cvta_generic_to_shared(pdsdp_dsm);
  return reinterpret_cast<T*>(pdsdp_dsm + o);
}

struct Prof {
  long long last;
  long long acc[16];
  int cur;
  int ntr;
  int cap;
  double* trace;
};
// Compiled in only with -DPDSDP_TRACE=1 (tools/gpu_trace*.py builds): the
// production kernel carries no clock64 reads or trace stores.
#ifndef PDSDP_TRACE
#define PDSDP_TRACE 0
#endif
#if PDSDP_TRACE
__device__ __forceinline__ void prof_log(Prof& p, int label, long long now) {
  if (p.trace && p.ntr < p.cap) {
    p.trace[2 * p.ntr] = label;
    p.trace[2 * p.ntr + 1] = (double)now;
    ++p.ntr;
  }
}
__device__ __forceinline__ void prof_mark(Prof& p, int phase) {
  if (threadIdx.x == 0) {
    const long long now = clock64();
    p.acc[p.cur] += now - p.last;
    p.last = now;
    p.cur = phase;
    prof_log(p, phase, now);
  }
}
__device__ __forceinline__ void prof_tick(Prof& p, int label) {
  if (threadIdx.x == 0) prof_log(p, label, clock64());
}
// ticks from helpers that do not receive the Prof handle (trace builds only)
__shared__ Prof* g_trace_prof;
#define PDSDP_TICK(label) prof_tick(*g_trace_prof, (label))
#else
__device__ __forceinline__ void prof_mark(Prof&, int) {}
__device__ __forceinline__ void prof_tick(Prof&, int) {}
#define PDSDP_TICK(label) ((void)0)
#endif

// Per-instance descriptor (device resident).  Sizes and pointers only.
struct Inst {
  int n, m, p, mp, ld, C;
  int nz;              // slots of the symmetric Z CSR
  int group;           // lanes per constraint row in the A-map
  int nd;              // low-rank dense constraint rows (D = sig u u^T), kept out of the CSR
  int drow[PDSDP_NDMAX];
  int pad0;
  double dsig[PDSDP_NDMAX];                 // sign sigma of each dense row
  double dun2[PDSDP_NDMAX];                 // ||u||^2
  double duu[PDSDP_NDMAX * PDSDP_NDMAX];    // (u_k^T u_l)^2
  const double* du;    // [nd][n] the vectors u
  const int* zptr;     // [n+1]
  const int* zcol;     // [nz]
  const int* zrow;     // [nz]
  const double* cval;  // [nz] objective entry C_ij at the slot
  const int* tptr;     // [nz+1] contributors of M^T y to the slot
  const int* trow;     // constraint row of each contributor
  const double* tcoef; // scatter coefficient (packed value / s, s = 1 or sqrt 2)
  const int* dptr;     // [n+1] slots with contributors ("dynamic") in rows < i
  const int* dslot;    // dynamic slot indices, row order (the others hold C for ever)
  const double* zsabs; // [n] sum over the row's static slots of |C|
  double* zbuf0;       // [nz] Z = C + M^T y for y in ybuf0
  double* zbuf1;       // [nz] ... for y in ybuf1
  const int* aptr;     // [mp+1] constraint rows in dense coordinates
  const int* ai;
  const int* aj;
  const double* ag;    // gather coefficient (packed value * s)
  const int* asplit;   // [C+1] constraint-row range of each CTA
  const double* bv;    // [m]
  const double* hv;    // [p]
  double alpha;
  double* V;
  double* AV;
  double* Y0;
  double* Y1;
  double* Y2;
  double* F;
  double* Vp;          // eigenvector block of two iterations before (start-block extrapolation)
  double* Yc;          // 2 x compact (stride = active width) copies of the filter block (TMA multicast sources)
  double* ybuf0;
  double* ybuf1;
  double* dy;
  double* red;         // [2][C][RED_MAX] cluster reduction scratch
  double* rpart;       // residual kernel tile partials
  unsigned int* rcount;
  State* st;
  double* out;         // host-mapped [KMAX][OUT_LEN]
  int* stopf;          // device flag: an event may fire, skip the remaining steps
  double* trace;       // [C][2 * PDSDP_TRACE_CTA] per-CTA (label, cycle) log (flag bit 6)
};

static_assert(sizeof(Inst) % 8 == 0, "Inst is copied as 8-byte words");

// Per-launch control for one instance.
struct Ctl {
  int r;       // target rank for this iteration
  int ypar;    // y_k lives in ybuf[ypar], y_{k+1} goes to ybuf[ypar^1]
  int flags;   // bit0 cold, bit1 certificate, bit2 re-run, bit3 tight certificate, bit4 dump
  int maxpass;
  double conv_thr;    // stop when eps_p + eps_d <= conv_thr  (lowrank.py:161)
  double stall_thr;   // stop when eps_p + eps_d >= stall_thr (lowrank.py:64-69, 181)
};

// output slots
enum { O_EPS_P = 0, O_EPS_D, O_LAM, O_FIN, O_PASSES, O_MATVECS, O_EIGCONV, O_EIGRES,
       O_DENSE, O_CORR, O_ED2, O_BLK, O_DONE, O_ERR, O_DENSE_EXACT };

// a / b for 0 <= a < 2^21, 1 <= b <= 2^10 through the FP32 reciprocal: the
// emulated 32-bit integer division is a ~100-cycle dependent chain, and the
// short latency-bound phases of the iteration kernel start with several of
// them (index arithmetic).  Exact: (a + 0.5) / b is at least 0.5 / b away from
// an integer, the float product is within 2^-22 (a + 0.5) / b of it.
__device__ __forceinline__ int fdiv(int a, int b) {
  return __float2int_rz((__int2float_rn(a) + 0.5f) * __frcp_rn(__int2float_rn(b)));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// deterministic counter-based uniform(-1, 1)
__device__ __forceinline__ double hash_uniform(uint64_t seed, uint64_t a, uint64_t b) {
  uint64_t x = seed * 0x9E3779B97F4A7C15ull ^ (a * 0xBF58476D1CE4E5B9ull) ^ (b * 0x94D049BB133111EBull + 0x632BE59BD9B4E019ull);
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27; x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return ((double)(x >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
}

}  // namespace pdsdp
