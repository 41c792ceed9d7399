// Host runtime + C ABI of the B200 LR-PD-SDP hot path (see include/pdsdp_b200.h).
//
// Responsibilities:
//   * one-time re-indexing of the reference's packed problem layout
//     (problem.py:119-137) into dense (i, j) coordinates: the symmetric Z
//     pattern, per-slot adjoint contributor lists, constraint rows with
//     gather coefficients, the touched-position space of the operator norm;
//   * one device arena per instance, descriptors, host-mapped outputs;
//   * launching the cluster iteration kernel and the whole-GPU residual kernel.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pdsdp_b200.h"
#include "common.cuh"
#include "dense_path.cuh"
#include "iterate.cuh"
#include "opnorm.cuh"
#include "residual.cuh"
#include "zbound.cuh"

// Iterations between lambda_max(Z) estimates: Z = C + M^T y drifts quickly
// while y builds up and ever more slowly afterwards, so the refresh interval
// grows with the iteration count, k / 8 clamped to [ZL_EVERY, ZL_EVERY_MAX]
// (a stale estimate costs filter efficiency, never accuracy: zbound.cuh;
// config 2: fixed 256 -> 7.56 s, 1024 -> 7.42 s, 4096 -> 7.37 s to tolerance).
#ifndef PDSDP_ZL_EVERY
#define PDSDP_ZL_EVERY 256
#endif
#ifndef PDSDP_ZL_EVERY_MAX
#define PDSDP_ZL_EVERY_MAX 4096
#endif

using namespace pdsdp;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(PDSDP_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
  } while (0)

struct Arena {
  char* base = nullptr;
  size_t off = 0, cap = 0;
  template <class T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base + off);
    off += count * sizeof(T) + 16;
    return p;
  }
};

struct Instance {
  int n = 0, m = 0, p = 0, mp = 0, ld = 0;
  int bmax = 0;          // largest eigen block used so far (smem workspace size)
  long long nz = 0;
  int group = 1;
  int ntile = 0;
  // host copies of the re-indexed problem
  std::vector<int> zptr, zcol, zrow, tptr, trow, aptr, ai, aj, dptr, dslot;
  std::vector<double> cval, tcoef, ag, bv, hv, zsabs;
  // dense rank-one constraint rows  D_r = sig u u^T  (kept out of the CSR)
  int nd = 0;
  int drow[PDSDP_NDMAX] = {0};
  double dsig[PDSDP_NDMAX] = {0}, dun2[PDSDP_NDMAX] = {0}, duu[PDSDP_NDMAX * PDSDP_NDMAX] = {0};
  std::vector<double> du;
  // operator-norm T-space
  std::vector<long long> tpos;
  std::vector<int> o_seg_lo, o_seg_hi, o_row_seg, o_mcol, o_tptr, o_trow;
  std::vector<double> o_mval, o_tval;
  // device
  void* dmem = nullptr;
  size_t dbytes = 0;
  Inst desc{};
  OpnormDev od{};
  double* d_packed = nullptr;   // scratch packed vector (op-level maps)
  long long zl_age = 1LL << 40;  // iterations since the last lambda_max(Z) estimate
  long long iters_total = 0;     // iterations since the last reset
  long long P = 0;
  // dense-iterate mode (dense_path.cuh): X_k as a dense n x n matrix, full eigendecomposition
  int dense_mode = 0;
  int dcur = 0;                  // dd.X[dcur] holds X_k
  void* dense_mem = nullptr;
  DenseDev dd{};
  double* d_rowt = nullptr;      // per-row scratch of the dense kernels
};

}  // namespace

struct pdsdp_batch {
  std::vector<Instance*> inst;
  int C = 1, lds = 4;
  size_t smem = 0;
  cudaStream_t stream = nullptr;
  Inst* d_insts = nullptr;
  Ctl* h_ctl = nullptr;
  Ctl* d_ctl = nullptr;
  int* h_active = nullptr;
  int* d_active = nullptr;
  double* h_out = nullptr;   // mapped pinned, count * KMAX * OUT_LEN
  int* d_stop = nullptr;     // per-instance chunk stop flags
  int* h_zl = nullptr;       // lambda_max(Z) estimate list (instance, y parity)
  int* d_zl = nullptr;
  double* d_out = nullptr;
  double* d_objpart = nullptr;
  unsigned* d_objcnt = nullptr;
  double* d_objres = nullptr;
  int max_tiles = 1;
  long long zmax = 0;    // largest per-CTA slice of Z rows over the batch
  int nmax = 0, ldmax = 0;
  int timing = 0;
  int verify_residual = 0;   // also run residual_kernel (exact dense term) after each step
  int dense_no_tma = 0;      // PDSDP_DENSE_NO_TMA=1: plain-load Jacobi rounds (A/B of the bulk-copy kernel)
  int dense_no_block = 0;    // PDSDP_DENSE_NO_BLOCK=1: scalar-rotation rounds for every n (A/B of the blocked kernel)
  int bj_nmin = PDSDP_BJ_NMIN;   // smallest n taking the blocked rounds (PDSDP_DENSE_BLOCK_NMIN overrides: tests)
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  double t_iter = 0.0, n_iter = 0.0, t_res = 0.0, n_res = 0.0, n_launch = 0.0;
  cudaEvent_t tev[PDSDP_KMAX + 1] = {};
  // asynchronous per-instance chunks (pdsdp_chunk_*): one stream + event per slot
  std::vector<cudaStream_t> slot_stream;
  std::vector<cudaEvent_t> slot_event;
  int* d_ident = nullptr;    // d_ident[i] = i: the active list of a one-instance launch
};

namespace {

inline long long packed_len(long long n) { return n * (n + 1) / 2; }

int build_instance(const pdsdp_problem& pr, Instance& I) {
  const int n = pr.n, m = pr.m, p = pr.p;
  if (n < 1) return fail(PDSDP_EINVAL, "matrix dimension must be positive");
  if (m < 0 || p < 0) return fail(PDSDP_EINVAL, "negative constraint count");
  if (!pr.C_packed) return fail(PDSDP_EINVAL, "C_packed is NULL");
  const int mp = m + p;
  const long long P = packed_len(n);
  I.n = n; I.m = m; I.p = p; I.mp = mp; I.P = P;
  const int bcap = std::min(n, PDSDP_BMAX);
  I.ld = (bcap + 1) & ~1;
  std::vector<long long> rstart(n + 1);
  for (long long i = 0; i <= n; ++i) rstart[i] = i * n - i * (i - 1) / 2;
  auto coords = [&](long long pos, int& i, int& j) {
    int ii = (int)(std::upper_bound(rstart.begin(), rstart.begin() + n, pos) - rstart.begin()) - 1;
    i = ii;
    j = (int)(pos - rstart[ii] + ii);
  };
  const long long nnz = mp ? pr.row_ptr[mp] : 0;
  if (mp && (!pr.row_ptr || (nnz && (!pr.row_idx || !pr.row_val))))
    return fail(PDSDP_EINVAL, "constraint arrays are NULL");
  for (int r = 0; r < mp; ++r) {
    if (pr.row_ptr[r + 1] < pr.row_ptr[r]) return fail(PDSDP_EINVAL, "row_ptr not monotone");
    for (long long e = pr.row_ptr[r]; e < pr.row_ptr[r + 1]; ++e) {
      if (pr.row_idx[e] < 0 || pr.row_idx[e] >= P) return fail(PDSDP_EINVAL, "constraint row index out of range");
      if (e > pr.row_ptr[r] && pr.row_idx[e] <= pr.row_idx[e - 1])
        return fail(PDSDP_EINVAL, "indices must be strictly increasing");
    }
  }
  // ---- dense rank-one rows: a row whose matrix D (D_ii = a, D_ij = a/sqrt 2,
  //      the adjoint's scatter coefficients) is exactly sig u u^T is applied
  //      through u: M^T y gets y sig u u^T, <D, X> = sig u^T X u.  Its n^2/2
  //      entries would otherwise turn Z into a dense matrix (an equipartition
  //      row <11^T, X> = 0, BASELINE configs[2]). ----
  std::vector<char> dense(mp, 0);
  I.nd = 0;
  I.du.clear();
  for (int r = 0; r < mp && I.nd < PDSDP_NDMAX; ++r) {
    const long long a0 = pr.row_ptr[r], a1 = pr.row_ptr[r + 1];
    if (a1 - a0 < std::max<long long>(2LL * n, 64)) continue;
    std::vector<double> dg(n, 0.0), col(n, 0.0);
    double dmax = 0.0;
    for (long long e = a0; e < a1; ++e) {
      int i, j;
      coords(pr.row_idx[e], i, j);
      const double v = (i == j) ? pr.row_val[e] : pr.row_val[e] / std::sqrt(2.0);
      if (i == j) dg[i] = v;
      dmax = std::max(dmax, std::fabs(v));
    }
    int piv = 0;
    for (int i = 1; i < n; ++i) if (std::fabs(dg[i]) > std::fabs(dg[piv])) piv = i;
    if (dg[piv] == 0.0 || !std::isfinite(dmax)) continue;
    for (long long e = a0; e < a1; ++e) {
      int i, j;
      coords(pr.row_idx[e], i, j);
      const double v = (i == j) ? pr.row_val[e] : pr.row_val[e] / std::sqrt(2.0);
      if (j == piv) col[i] = v;
      if (i == piv) col[j] = v;
    }
    const double sg = dg[piv] > 0.0 ? 1.0 : -1.0, sq = std::sqrt(std::fabs(dg[piv]));
    std::vector<double> u(n);
    long long nzu = 0;
    for (int i = 0; i < n; ++i) { u[i] = col[i] / (sg * sq); if (u[i] != 0.0) ++nzu; }
    bool ok = true;
    long long nzv = 0;
    for (long long e = a0; e < a1 && ok; ++e) {
      int i, j;
      coords(pr.row_idx[e], i, j);
      const double v = (i == j) ? pr.row_val[e] : pr.row_val[e] / std::sqrt(2.0);
      if (v == 0.0) continue;
      ++nzv;
      if (std::fabs(v - sg * u[i] * u[j]) > 1e-13 * dmax) ok = false;
    }
    if (!ok || nzv != nzu * (nzu + 1) / 2) continue;   // every pair with u_i u_j != 0 present
    dense[r] = 1;
    I.drow[I.nd] = r;
    I.dsig[I.nd] = sg;
    double n2 = 0.0;
    for (int i = 0; i < n; ++i) n2 += u[i] * u[i];
    I.dun2[I.nd] = n2;
    I.du.insert(I.du.end(), u.begin(), u.end());
    ++I.nd;
  }
  for (int k = 0; k < I.nd; ++k)
    for (int l = 0; l < I.nd; ++l) {
      double g = 0.0;
      for (int i = 0; i < n; ++i) g += I.du[(size_t)k * n + i] * I.du[(size_t)l * n + i];
      I.duu[k * PDSDP_NDMAX + l] = g * g;
    }
  if (I.nd) I.ld = (std::min(n, PDSDP_BMAX) + I.nd + 1) & ~1;   // F holds the u's after its rF columns
  // ---- support = nonzeros of C  U  positions of all (sparse) constraint entries ----
  std::vector<int> sid(P, -1);
  std::vector<long long> spos;
  {
    std::vector<unsigned char> mark(P, 0);
    for (long long q = 0; q < P; ++q) if (pr.C_packed[q] != 0.0) mark[q] = 1;
    for (int r = 0; r < mp; ++r)
      if (!dense[r])
        for (long long e = pr.row_ptr[r]; e < pr.row_ptr[r + 1]; ++e) mark[pr.row_idx[e]] = 1;
    for (long long q = 0; q < P; ++q) if (mark[q]) { sid[q] = (int)spos.size(); spos.push_back(q); }
  }
  const long long U = (long long)spos.size();
  // contributors per support entry
  std::vector<int> ccount(U + 1, 0);
  for (int r = 0; r < mp; ++r)
    if (!dense[r])
      for (long long e = pr.row_ptr[r]; e < pr.row_ptr[r + 1]; ++e) ccount[sid[pr.row_idx[e]] + 1]++;
  for (long long u = 0; u < U; ++u) ccount[u + 1] += ccount[u];
  std::vector<int> crow(ccount[U]);
  std::vector<double> ccoef(ccount[U]);
  {
    std::vector<int> fillp(ccount.begin(), ccount.end() - 1);
    for (int r = 0; r < mp; ++r)
      if (!dense[r])
      for (long long e = pr.row_ptr[r]; e < pr.row_ptr[r + 1]; ++e) {
        int i, j;
        coords(pr.row_idx[e], i, j);
        const int u = sid[pr.row_idx[e]];
        crow[fillp[u]] = r;
        ccoef[fillp[u]] = (i == j) ? pr.row_val[e] : pr.row_val[e] / std::sqrt(2.0);
        fillp[u]++;
      }
  }
  // ---- symmetric CSR in dense coordinates ----
  std::vector<int> si(U), sj(U);
  std::vector<long long> rowcnt(n + 1, 0);
  for (long long u = 0; u < U; ++u) {
    int i, j;
    coords(spos[u], i, j);
    si[u] = i; sj[u] = j;
    rowcnt[i + 1]++;
    if (i != j) rowcnt[j + 1]++;
  }
  for (int i = 0; i < n; ++i) rowcnt[i + 1] += rowcnt[i];
  const long long nz = rowcnt[n];
  if (nz >= (1ll << 31) || nnz >= (1ll << 31)) return fail(PDSDP_EINVAL, "problem too large for int32 indexing");
  I.nz = nz;
  I.zptr.assign(rowcnt.begin(), rowcnt.end());
  I.zcol.resize(nz); I.zrow.resize(nz); I.cval.resize(nz);
  std::vector<long long> slot_u(nz);
  {
    std::vector<long long> fillp(rowcnt.begin(), rowcnt.end() - 1);
    for (long long u = 0; u < U; ++u) {
      const int i = si[u], j = sj[u];
      const double c = (i == j) ? pr.C_packed[spos[u]] : pr.C_packed[spos[u]] / std::sqrt(2.0);
      long long s = fillp[i]++;
      I.zcol[s] = j; I.zrow[s] = i; I.cval[s] = c; slot_u[s] = u;
      if (i != j) {
        s = fillp[j]++;
        I.zcol[s] = i; I.zrow[s] = j; I.cval[s] = c; slot_u[s] = u;
      }
    }
  }
  I.tptr.assign(nz + 1, 0);
  for (long long s = 0; s < nz; ++s) I.tptr[s + 1] = I.tptr[s] + (ccount[slot_u[s] + 1] - ccount[slot_u[s]]);
  if ((long long)I.tptr[nz] >= (1ll << 31)) return fail(PDSDP_EINVAL, "too many adjoint contributors");
  I.trow.resize(I.tptr[nz]); I.tcoef.resize(I.tptr[nz]);
  for (long long s = 0; s < nz; ++s) {
    const long long u = slot_u[s];
    int o = I.tptr[s];
    for (int c = ccount[u]; c < ccount[u + 1]; ++c, ++o) { I.trow[o] = crow[c]; I.tcoef[o] = ccoef[c]; }
  }
  // slots touched by M^T y, per row; the others keep their C value in both Z buffers
  I.dptr.assign(n + 1, 0);
  I.dslot.clear();
  I.zsabs.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    for (long long s = I.zptr[i]; s < I.zptr[i + 1]; ++s) {
      if (I.tptr[s + 1] > I.tptr[s]) I.dslot.push_back((int)s);
      else I.zsabs[i] += std::fabs(I.cval[s]);
    }
    I.dptr[i + 1] = (int)I.dslot.size();
  }
  // ---- constraint rows in dense coordinates (dense rank-one rows left empty) ----
  I.aptr.assign(mp + 1, 0);
  I.ai.clear(); I.aj.clear(); I.ag.clear();
  int maxrow = 0;
  for (int r = 0; r < mp; ++r) {
    if (!dense[r])
      for (long long e = pr.row_ptr[r]; e < pr.row_ptr[r + 1]; ++e) {
        int i, j;
        coords(pr.row_idx[e], i, j);
        I.ai.push_back(i); I.aj.push_back(j);
        I.ag.push_back((i == j) ? pr.row_val[e] : pr.row_val[e] * std::sqrt(2.0));
      }
    I.aptr[r + 1] = (int)I.ai.size();
    maxrow = std::max(maxrow, I.aptr[r + 1] - I.aptr[r]);
  }
  I.group = 1;
  while (I.group < maxrow && I.group < 32) I.group <<= 1;
  I.bv.assign(pr.b, pr.b + m);
  I.hv.assign(pr.h, pr.h + p);
  // ---- operator-norm T-space ----
  {
    std::vector<int> tid_of(P, -1);
    for (long long e = 0; e < nnz; ++e) {
      const long long q = pr.row_idx[e];
      if (tid_of[q] < 0) { tid_of[q] = 0; }
    }
    I.tpos.clear();
    for (long long q = 0; q < P; ++q) if (tid_of[q] == 0) { tid_of[q] = (int)I.tpos.size(); I.tpos.push_back(q); }
    const int nT = (int)I.tpos.size();
    I.o_mcol.resize(nnz); I.o_mval.resize(nnz);
    for (long long e = 0; e < nnz; ++e) { I.o_mcol[e] = tid_of[pr.row_idx[e]]; I.o_mval[e] = pr.row_val[e]; }
    I.o_row_seg.assign(mp + 1, 0);
    I.o_seg_lo.clear(); I.o_seg_hi.clear();
    for (int r = 0; r < mp; ++r) {
      long long a = pr.row_ptr[r], bnd = pr.row_ptr[r + 1];
      if (a == bnd) { I.o_seg_lo.push_back((int)a); I.o_seg_hi.push_back((int)a); }
      for (long long s = a; s < bnd; s += SEG_LEN) {
        I.o_seg_lo.push_back((int)s);
        I.o_seg_hi.push_back((int)std::min(bnd, s + SEG_LEN));
      }
      I.o_row_seg[r + 1] = (int)I.o_seg_lo.size();
    }
    I.o_tptr.assign(nT + 1, 0);
    for (long long e = 0; e < nnz; ++e) I.o_tptr[tid_of[pr.row_idx[e]] + 1]++;
    for (int t = 0; t < nT; ++t) I.o_tptr[t + 1] += I.o_tptr[t];
    I.o_trow.resize(nnz); I.o_tval.resize(nnz);
    std::vector<int> fillp(I.o_tptr.begin(), I.o_tptr.end() - 1);
    for (int r = 0; r < mp; ++r)
      for (long long e = pr.row_ptr[r]; e < pr.row_ptr[r + 1]; ++e) {
        const int t = tid_of[pr.row_idx[e]];
        I.o_trow[fillp[t]] = r; I.o_tval[fillp[t]] = pr.row_val[e]; fillp[t]++;
      }
  }
  const int nt = (n + RES_TILE - 1) / RES_TILE;
  I.ntile = nt * (nt + 1) / 2;
  return PDSDP_OK;
}

template <class T>
int upload(Arena& a, T*& dst, const std::vector<T>& src, size_t min_count = 1) {
  dst = a.take<T>(std::max(src.size(), min_count));
  if (!src.empty()) CK(cudaMemcpy(dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
  return PDSDP_OK;
}

int alloc_instance(Instance& I, int C, double* out_dev) {
  const size_t nld = (size_t)I.n * I.ld;
  const int nseg = (int)I.o_seg_lo.size();
  size_t bytes = 0;
  auto add = [&](size_t b) { bytes += ((b + 16) + 255) & ~size_t(255); };
  add((I.n + 1) * 4); add(I.nz * 4); add(I.nz * 4); add(I.nz * 8); add((I.nz + 1) * 4);
  add(I.trow.size() * 4 + 4); add(I.tcoef.size() * 8 + 8); add(I.nz * 8); add(I.nz * 8);
  add((I.n + 1) * 4); add(I.dslot.size() * 4 + 4); add(I.n * 8 + 8);
  add((I.mp + 1) * 4); add(I.ai.size() * 4 + 4); add(I.aj.size() * 4 + 4); add(I.ag.size() * 8 + 8);
  add((C + 1) * 4); add(I.bv.size() * 8 + 8); add(I.hv.size() * 8 + 8);
  for (int k = 0; k < 7; ++k) add(nld * 8);
  add(2 * (size_t)I.n * (I.ld + 4) * 8);
  add(I.mp * 8 + 8); add(I.mp * 8 + 8); add(I.mp * 8 + 8);
  add((size_t)2 * C * PDSDP_RED_MAX * 8);
  add((size_t)I.ntile * 8 + 8); add(64); add(sizeof(State));
  // opnorm
  add(nseg * 4 + 4); add(nseg * 4 + 4); add((I.mp + 1) * 4); add(I.o_mcol.size() * 4 + 4);
  add(I.o_mval.size() * 8 + 8); add(I.o_tptr.size() * 4 + 4); add(I.o_trow.size() * 4 + 4);
  add(I.o_tval.size() * 8 + 8); add(I.tpos.size() * 8 + 8); add(I.mp * 8 + 8); add(nseg * 8 + 8);
  add(2 * NORM_BLOCKS * 8); add(64); add(4096 * 8);
  add((size_t)I.P * 8);
  add(I.du.size() * 8 + 8);
  add((size_t)C * 2 * PDSDP_TRACE_CTA * 8);
  bytes += 4096;
  CK(cudaMalloc(&I.dmem, bytes));
  I.dbytes = bytes;
  CK(cudaMemset(I.dmem, 0, bytes));
  Arena a{(char*)I.dmem, 0, bytes};
  Inst& d = I.desc;
  d.n = I.n; d.m = I.m; d.p = I.p; d.mp = I.mp; d.ld = I.ld; d.C = C;
  d.nz = (int)I.nz; d.group = I.group;
  d.nd = I.nd;
  for (int k = 0; k < PDSDP_NDMAX; ++k) { d.drow[k] = I.drow[k]; d.dsig[k] = I.dsig[k]; d.dun2[k] = I.dun2[k]; }
  for (int k = 0; k < PDSDP_NDMAX * PDSDP_NDMAX; ++k) d.duu[k] = I.duu[k];
  int rc;
  int* zptr; int* zcol; int* zrow; double* cval; int* tptr; int* trow; double* tcoef;
  if ((rc = upload(a, zptr, I.zptr))) return rc;
  if ((rc = upload(a, zcol, I.zcol))) return rc;
  if ((rc = upload(a, zrow, I.zrow))) return rc;
  if ((rc = upload(a, cval, I.cval))) return rc;
  if ((rc = upload(a, tptr, I.tptr))) return rc;
  if ((rc = upload(a, trow, I.trow))) return rc;
  if ((rc = upload(a, tcoef, I.tcoef))) return rc;
  d.zptr = zptr; d.zcol = zcol; d.zrow = zrow; d.cval = cval; d.tptr = tptr; d.trow = trow; d.tcoef = tcoef;
  {
    int *dp, *ds; double* za;
    if ((rc = upload(a, dp, I.dptr))) return rc;
    if ((rc = upload(a, ds, I.dslot))) return rc;
    if ((rc = upload(a, za, I.zsabs))) return rc;
    d.dptr = dp; d.dslot = ds; d.zsabs = za;
  }
  d.zbuf0 = a.take<double>(I.nz + 1);
  d.zbuf1 = a.take<double>(I.nz + 1);
  int *aptr, *ai, *aj; double* ag;
  if ((rc = upload(a, aptr, I.aptr))) return rc;
  if ((rc = upload(a, ai, I.ai))) return rc;
  if ((rc = upload(a, aj, I.aj))) return rc;
  if ((rc = upload(a, ag, I.ag))) return rc;
  d.aptr = aptr; d.ai = ai; d.aj = aj; d.ag = ag;
  // constraint-row split across the C CTAs, balanced by entries
  std::vector<int> split(C + 1, I.mp);
  {
    const long long tot = I.aptr[I.mp] + I.mp;
    int r = 0;
    split[0] = 0;
    for (int c = 1; c < C; ++c) {
      const long long target = tot * c / C;
      while (r < I.mp && (long long)I.aptr[r] + r < target) ++r;
      split[c] = r;
    }
    split[C] = I.mp;
  }
  int* asplit;
  if ((rc = upload(a, asplit, split))) return rc;
  d.asplit = asplit;
  double *bv, *hv;
  if ((rc = upload(a, bv, I.bv))) return rc;
  if ((rc = upload(a, hv, I.hv))) return rc;
  d.bv = bv; d.hv = hv;
  d.V = a.take<double>(nld); d.AV = a.take<double>(nld); d.Y0 = a.take<double>(nld);
  d.Y1 = a.take<double>(nld); d.Y2 = a.take<double>(nld); d.F = a.take<double>(nld);
  d.Vp = a.take<double>(nld);
  d.Yc = a.take<double>(2 * (size_t)I.n * (I.ld + 4));
  d.ybuf0 = a.take<double>(I.mp + 1); d.ybuf1 = a.take<double>(I.mp + 1); d.dy = a.take<double>(I.mp + 1);
  d.red = a.take<double>((size_t)2 * C * PDSDP_RED_MAX);
  d.rpart = a.take<double>(I.ntile + 1);
  d.rcount = a.take<unsigned>(16);
  d.st = a.take<State>(1);
  d.trace = a.take<double>((size_t)C * 2 * PDSDP_TRACE_CTA);
  d.out = out_dev;
  d.alpha = 1.0;
  // opnorm
  OpnormDev& o = I.od;
  o.mp = I.mp; o.nT = (int)I.tpos.size(); o.nseg = nseg;
  int *slo, *shi, *rseg, *mcol, *otp, *otr; double *mval, *otv;
  if ((rc = upload(a, slo, I.o_seg_lo))) return rc;
  if ((rc = upload(a, shi, I.o_seg_hi))) return rc;
  if ((rc = upload(a, rseg, I.o_row_seg))) return rc;
  if ((rc = upload(a, mcol, I.o_mcol))) return rc;
  if ((rc = upload(a, mval, I.o_mval))) return rc;
  if ((rc = upload(a, otp, I.o_tptr))) return rc;
  if ((rc = upload(a, otr, I.o_trow))) return rc;
  if ((rc = upload(a, otv, I.o_tval))) return rc;
  o.seg_lo = slo; o.seg_hi = shi; o.row_seg = rseg; o.mcol = mcol; o.mval = mval;
  o.tptr = otp; o.trow = otr; o.tval = otv;
  o.x = a.take<double>(I.tpos.size() + 1);
  o.y = a.take<double>(I.mp + 1);
  o.seg_part = a.take<double>(nseg + 1);
  o.norm_part = a.take<double>(2 * NORM_BLOCKS);
  o.scal = a.take<double>(8);
  o.s_hist = a.take<double>(4096);
  I.d_packed = a.take<double>((size_t)I.P);
  double* du;
  if ((rc = upload(a, du, I.du))) return rc;
  d.du = du;
  if (a.off > bytes) return fail(PDSDP_ENOMEM, "arena overflow");
  return PDSDP_OK;
}

int check_inst(pdsdp_batch* b, int inst) {
  if (!b) return fail(PDSDP_EINVAL, "batch is NULL");
  if (inst < 0 || inst >= (int)b->inst.size()) return fail(PDSDP_EINVAL, "instance index out of range");
  return PDSDP_OK;
}

int launch_iterate(pdsdp_batch* b, int nact, int lds, int step0, int nsteps, cudaStream_t stream = nullptr,
                   const int* d_active = nullptr) {
  // shared memory plan beyond the fixed workspaces, in priority order:
  // (1) the CTA's Z rows (all-or-nothing; they feed every sparse product),
  // (2) own rows of F, Y_j, Y_{j-1} (smem-resident filter recurrence),
  // (3) the staged operand block (n rows x up to 16 columns, >= 2 columns).
  const int nlmax = (b->nmax + b->C - 1) / b->C;
  const size_t limit = b->smem;
  const size_t base = iterate_smem_bytes(lds, 0, 0, 0, 0);
  size_t avail = limit > base ? limit - base : 0;
  int zcap = (int)std::min<long long>(b->zmax, (long long)(avail / 12));
  if (zcap < b->zmax) zcap = 0;
  avail -= (size_t)zcap * 12;
  int owncap = nlmax * lds;
  size_t need_own = iterate_smem_bytes(lds, 0, 0, owncap, nlmax) - base;
  if (need_own + 16 * (size_t)b->nmax > avail) { owncap = 0; need_own = 0; }
  avail -= need_own;
  long long want = (long long)b->nmax * std::min(b->ldmax, 16);
  int ycap = (int)std::min<long long>(want, (long long)(avail / 8));
  ycap &= ~1;
  if (ycap + 4LL * lds * (lds + 1) < 2LL * b->nmax) { ycap = 0; owncap = 0; }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nact * b->C);
  cfg.blockDim = dim3(PDSDP_NTHR);
  cfg.dynamicSmemBytes = iterate_smem_bytes(lds, zcap, ycap, owncap, nlmax);
  cfg.stream = stream ? stream : b->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = b->C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, lrpdhg_iterate_kernel, (const Inst*)b->d_insts, (const Ctl*)b->d_ctl,
                        d_active ? d_active : (const int*)b->d_active, step0, nsteps, lds, zcap, ycap, owncap, nlmax));
  return PDSDP_OK;
}

// Resident clusters of the iteration kernel on this device (cluster size C,
// one CTA per SM): the number of per-instance chunks that can run side by side.
int max_active_clusters(pdsdp_batch* b, int* out) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(b->C);
  cfg.blockDim = dim3(PDSDP_NTHR);
  cfg.dynamicSmemBytes = b->smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = b->C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  CK(cudaOccupancyMaxActiveClusters(&n, lrpdhg_iterate_kernel, &cfg));
  *out = std::max(1, n);
  return PDSDP_OK;
}

// Fill the control block of one instance's next K steps (host side).
void fill_ctl(pdsdp_batch* b, int k, int rank, int ypar0, int flags, int maxpass, int K, double conv_thr,
              const double* stall_thr) {
  for (int j = 0; j < K; ++j) {
    Ctl& c = b->h_ctl[(size_t)k * PDSDP_KMAX + j];
    c.r = rank;
    c.ypar = (ypar0 ^ j) & 1;
    c.flags = flags;
    c.maxpass = maxpass;
    c.conv_thr = conv_thr;
    c.stall_thr = stall_thr ? stall_thr[j] : HUGE_VAL;
    double* o = b->h_out + ((size_t)k * PDSDP_KMAX + j) * PDSDP_OUT_LEN;
    o[O_DONE] = 0.0;
    o[O_DENSE_EXACT] = NAN;
    o[O_ERR] = 0.0;
  }
}

// The lambda_max(Z) refresh of one instance on `stream`, when due (zbound.cuh).
int maybe_zlanczos(pdsdp_batch* b, int k, int ypar, cudaStream_t stream) {
  Instance* I = b->inst[k];
  const long long every = std::min<long long>(PDSDP_ZL_EVERY_MAX, std::max<long long>(PDSDP_ZL_EVERY, I->iters_total / 8));
  if (I->zl_age < every || I->n > PDSDP_ZL_NMAX) return PDSDP_OK;
  b->h_zl[2 * k] = k;
  b->h_zl[2 * k + 1] = ypar & 1;
  I->zl_age = 0;
  CK(cudaMemcpyAsync(b->d_zl + 2 * k, b->h_zl + 2 * k, 2 * sizeof(int), cudaMemcpyHostToDevice, stream));
  const size_t zsm = (size_t)3 * std::max(2, I->n) * sizeof(double);
  CK(cudaFuncSetAttribute(zlanczos_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zsm));
  zlanczos_kernel<<<1, PDSDP_ZL_THREADS, zsm, stream>>>(b->d_insts, b->d_zl + 2 * k);
  CK(cudaGetLastError());
  b->n_launch += 1;
  return PDSDP_OK;
}


// ---- dense-iterate mode (dense_path.cuh) ----
#define DENSE_GRID 512

int dense_alloc(Instance* I) {
  if (I->dense_mem) return PDSDP_OK;
  const size_t n = I->n, nn = n * n;
  if (2 * n * sizeof(double) > 220 * 1024)
    return fail(PDSDP_ENOMEM, "dense eigensolver stages two matrix rows in shared memory: n <= 14080");
  const size_t rowt = std::max<size_t>(std::max<size_t>(3 * (size_t)I->mp, 2 * n), 2 * (size_t)PDSDP_NDMAX * n) + 16;
  size_t bytes = 0;
  auto add = [&](size_t b) { bytes += (b + 255) & ~size_t(255); };
  add(nn * 8); add(nn * 8); add(nn * 8); add(n * 8); add(n * 8); add(n * 4); add(n * 8);
  add(4 * DENSE_PART_MAX * 8); add(DENSE_SCAL * 8); add(64); add(64); add(rowt * 8);
  CK(cudaMalloc(&I->dense_mem, bytes + 4096));
  CK(cudaMemset(I->dense_mem, 0, bytes + 4096));
  Arena a{(char*)I->dense_mem, 0, bytes + 4096};
  DenseDev& D = I->dd;
  D.n = I->n;
  D.X[0] = a.take<double>(nn - 2); D.X[1] = a.take<double>(nn - 2); D.W = a.take<double>(nn - 2);
  D.lam = a.take<double>(n); D.lams = a.take<double>(n); D.idx = a.take<int>(n); D.rowsum = a.take<double>(n);
  D.part = a.take<double>(4 * DENSE_PART_MAX); D.scal = a.take<double>(DENSE_SCAL);
  D.rot = a.take<unsigned>(4);
  D.maxoff = a.take<unsigned long long>(2);
  I->d_rowt = a.take<double>(rowt - 2);
  return PDSDP_OK;
}

int dense_objective(pdsdp_batch* b, Instance* I, int which, double* out) {
  const DenseDev& D = I->dd;
  dense_objective_kernel<<<DENSE_GRID, 256, 0, b->stream>>>(I->n, (int)I->nz, I->desc.zrow, I->desc.zcol, I->desc.cval,
                                                           D.X[which ? (I->dcur ^ 1) : I->dcur], D.part);
  reduce_sum_kernel<<<1, 256, 0, b->stream>>>(D.part, DENSE_GRID, D.scal + DS_DENSE);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, D.scal + DS_DENSE, sizeof(double), cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return PDSDP_OK;
}

}  // namespace

extern "C" {

const char* pdsdp_last_error(void) { return g_err.c_str(); }

const char* pdsdp_strerror(int code) {
  switch (code) {
    case PDSDP_OK: return "ok";
    case PDSDP_EINVAL: return "invalid argument";
    case PDSDP_ECUDA: return "CUDA error";
    case PDSDP_ENOMEM: return "out of memory";
    case PDSDP_ERANK: return "target rank exceeds the eigen block limit";
    default: return "unknown error";
  }
}

int pdsdp_version(void) { return 1; }

int pdsdp_batch_create(int count, const pdsdp_problem* problems, pdsdp_batch** out) {
  if (!out || !problems || count < 1) return fail(PDSDP_EINVAL, "bad batch arguments");
  *out = nullptr;
  int dev;
  CK(cudaGetDevice(&dev));
  pdsdp_batch* b = new pdsdp_batch();
  if (const char* e = getenv("PDSDP_DENSE_NO_TMA")) b->dense_no_tma = atoi(e);
  if (const char* e = getenv("PDSDP_DENSE_NO_BLOCK")) b->dense_no_block = atoi(e);
  if (const char* e = getenv("PDSDP_DENSE_BLOCK_NMIN")) b->bj_nmin = std::max(BJ_B2, atoi(e));
  int maxn = 0;
  for (int k = 0; k < count; ++k) maxn = std::max(maxn, (int)problems[k].n);
  int cta_rows = PDSDP_CTA_ROWS;
  const char* rows_env = getenv("PDSDP_CTA_ROWS");
  if (rows_env) cta_rows = std::max(32, atoi(rows_env));
  int C = 1;
  while (C < 16 && C * cta_rows < maxn) C <<= 1;
  b->C = C;
  int lds = std::min(maxn, PDSDP_BMAX);
  b->lds = lds < 4 ? 4 : lds;
  {
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, lrpdhg_iterate_kernel));
    b->smem = 227 * 1024 - fa.sharedSizeBytes;   // dynamic limit next to the static part
  }
  // A batch with more instances than clusters of that size can be resident
  // runs on clusters of half the size: each instance is slower, twice as many
  // run side by side (config 5: 32 instances 12.7 -> 9.8 s, 128 instances
  // ~43 -> 29.5 s; a further halving gains nothing, profiles/r02_cfg5_cluster_size.txt)
  if (!rows_env && count > 1 && C >= 2) {
    int slots = 1;
    int rc = max_active_clusters(b, &slots);
    if (rc) { delete b; return rc; }
    if (count > slots) b->C = C = C / 2;
  }
  CK(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking));
  const size_t outn = (size_t)count * PDSDP_KMAX * PDSDP_OUT_LEN;
  CK(cudaHostAlloc((void**)&b->h_out, outn * sizeof(double), cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer((void**)&b->d_out, b->h_out, 0));
  memset(b->h_out, 0, outn * sizeof(double));
  CK(cudaHostAlloc((void**)&b->h_ctl, (size_t)count * PDSDP_KMAX * sizeof(Ctl), 0));
  memset(b->h_ctl, 0, (size_t)count * PDSDP_KMAX * sizeof(Ctl));
  CK(cudaMalloc(&b->d_stop, (size_t)count * sizeof(int)));
  CK(cudaMalloc(&b->d_zl, (size_t)2 * count * sizeof(int)));
  b->h_zl = new int[2 * (size_t)count];
  CK(cudaMemset(b->d_stop, 0, (size_t)count * sizeof(int)));
  CK(cudaHostAlloc((void**)&b->h_active, (size_t)count * sizeof(int), 0));
  CK(cudaMalloc(&b->d_ctl, (size_t)count * PDSDP_KMAX * sizeof(Ctl)));
  CK(cudaMalloc(&b->d_active, (size_t)count * sizeof(int)));
  CK(cudaMalloc(&b->d_insts, (size_t)count * sizeof(Inst)));
  CK(cudaMalloc(&b->d_objpart, (size_t)count * 256 * sizeof(double)));
  CK(cudaMalloc(&b->d_objcnt, (size_t)count * sizeof(unsigned)));
  CK(cudaMemset(b->d_objcnt, 0, (size_t)count * sizeof(unsigned)));
  CK(cudaMalloc(&b->d_objres, (size_t)count * sizeof(double)));
  std::vector<Inst> descs(count);
  for (int k = 0; k < count; ++k) {
    Instance* I = new Instance();
    b->inst.push_back(I);
    int rc = build_instance(problems[k], *I);
    if (rc) { pdsdp_batch_destroy(b); return rc; }
    rc = alloc_instance(*I, C, b->d_out + (size_t)k * PDSDP_KMAX * PDSDP_OUT_LEN);
    I->desc.stopf = b->d_stop + k;
    if (rc) { std::string e = g_err; pdsdp_batch_destroy(b); g_err = e; return rc; }
    descs[k] = I->desc;
    b->max_tiles = std::max(b->max_tiles, I->ntile);
    b->nmax = std::max(b->nmax, I->n);
    b->ldmax = std::max(b->ldmax, I->ld);
    for (int c = 0; c < C; ++c) {
      const long long r0 = (long long)I->n * c / C, r1 = (long long)I->n * (c + 1) / C;
      b->zmax = std::max<long long>(b->zmax, (long long)I->zptr[r1] - I->zptr[r0]);
    }
  }
  CK(cudaMemcpy(b->d_insts, descs.data(), count * sizeof(Inst), cudaMemcpyHostToDevice));
  if (C > 8) CK(cudaFuncSetAttribute(lrpdhg_iterate_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(lrpdhg_iterate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b->smem));
  const size_t rsm = (size_t)2 * RES_TILE * (RES_KMAX + 1) * sizeof(double);
  CK(cudaFuncSetAttribute(residual_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm));
  for (int k = 0; k < count; ++k) {
    int rc = pdsdp_reset(b, k, 0.0);
    if (rc) { std::string e = g_err; pdsdp_batch_destroy(b); g_err = e; return rc; }
  }
  *out = b;
  return PDSDP_OK;
}

int pdsdp_batch_destroy(pdsdp_batch* b) {
  if (!b) return PDSDP_OK;
  if (b->stream) cudaStreamSynchronize(b->stream);
  for (Instance* I : b->inst) {
    if (I->dmem) cudaFree(I->dmem);
    if (I->dense_mem) cudaFree(I->dense_mem);
    delete I;
  }
  if (b->h_out) cudaFreeHost(b->h_out);
  if (b->h_ctl) cudaFreeHost(b->h_ctl);
  if (b->h_active) cudaFreeHost(b->h_active);
  if (b->d_ctl) cudaFree(b->d_ctl);
  if (b->d_active) cudaFree(b->d_active);
  if (b->d_insts) cudaFree(b->d_insts);
  if (b->d_objpart) cudaFree(b->d_objpart);
  if (b->d_objcnt) cudaFree(b->d_objcnt);
  if (b->d_objres) cudaFree(b->d_objres);
  if (b->d_stop) cudaFree(b->d_stop);
  if (b->d_zl) cudaFree(b->d_zl);
  if (b->d_ident) cudaFree(b->d_ident);
  for (cudaStream_t st : b->slot_stream) { cudaStreamSynchronize(st); cudaStreamDestroy(st); }
  for (cudaEvent_t ev : b->slot_event) cudaEventDestroy(ev);
  delete[] b->h_zl;
  for (int k = 0; k < 3; ++k) if (b->ev[k]) cudaEventDestroy(b->ev[k]);
  for (int k = 0; k <= PDSDP_KMAX; ++k) if (b->tev[k]) cudaEventDestroy(b->tev[k]);
  if (b->stream) cudaStreamDestroy(b->stream);
  delete b;
  return PDSDP_OK;
}

int pdsdp_batch_info(const pdsdp_batch* b, int inst, int64_t* info) {
  if (!b || !info || inst < 0 || inst >= (int)b->inst.size()) return fail(PDSDP_EINVAL, "bad info arguments");
  const Instance* I = b->inst[inst];
  info[0] = I->n; info[1] = I->nz; info[2] = (int64_t)I->tpos.size(); info[3] = b->C;
  info[4] = I->ld; info[5] = I->group; info[6] = (int64_t)b->smem; info[7] = (int64_t)I->dbytes;
  return PDSDP_OK;
}

void* pdsdp_batch_stream(pdsdp_batch* b) { return b ? (void*)b->stream : nullptr; }

int pdsdp_opnorm_positions(pdsdp_batch* b, int inst, int64_t* pos_out, int64_t* count) {
  int rc = check_inst(b, inst);
  if (rc) return rc;
  const Instance* I = b->inst[inst];
  if (count) *count = (int64_t)I->tpos.size();
  if (pos_out) for (size_t t = 0; t < I->tpos.size(); ++t) pos_out[t] = I->tpos[t];
  return PDSDP_OK;
}

// One cooperative launch for `iters` power iterations (opnorm.cuh).
static int opnorm_chunk(pdsdp_batch* b, Instance* I, int iters) {
  OpnormDev o = I->od;
  int dev = 0, sms = 148, per_sm = 1;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, opnorm_power_kernel, 256, 0));
  const long long want = std::max<long long>(std::max<long long>(o.nseg, ((long long)std::max(o.nT, o.mp) + 255) / 256), 1);
  const int grid = (int)std::max<long long>(1, std::min<long long>((long long)sms * std::max(per_sm, 1), want));
  double* hist = o.s_hist;
  void* args[] = {(void*)&o, (void*)&iters, (void*)&hist};
  CK(cudaLaunchCooperativeKernel((void*)opnorm_power_kernel, dim3(grid), dim3(256), args, 0, b->stream));
  b->n_launch += 1;
  return PDSDP_OK;
}

int pdsdp_opnorm_run(pdsdp_batch* b, int inst, const double* x0, int iters, double* s_out) {
  int rc = check_inst(b, inst);
  if (rc) return rc;
  if (iters < 1 || iters > 4096 || !s_out) return fail(PDSDP_EINVAL, "iters must lie in [1, 4096]");
  Instance* I = b->inst[inst];
  if (I->od.nT == 0 || I->o_mval.empty()) return fail(PDSDP_EINVAL, "all constraint rows are zero; operator norm is 0");
  if (x0) CK(cudaMemcpyAsync(I->od.x, x0, I->tpos.size() * sizeof(double), cudaMemcpyHostToDevice, b->stream));
  if ((rc = opnorm_chunk(b, I, iters))) return rc;
  CK(cudaMemcpyAsync(s_out, I->od.s_hist, iters * sizeof(double), cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return PDSDP_OK;
}

int pdsdp_set_alpha(pdsdp_batch* b, int inst, double alpha) {
  int rc = check_inst(b, inst);
  if (rc) return rc;
  if (!(alpha > 0.0) || !std::isfinite(alpha)) return fail(PDSDP_EINVAL, "alpha must be positive");
  Instance* I = b->inst[inst];
  I->desc.alpha = alpha;
  CK(cudaMemcpyAsync(&b->d_insts[inst].alpha, &I->desc.alpha, sizeof(double), cudaMemcpyHostToDevice, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return PDSDP_OK;
}

__global__ void init_finalize_kernel(const Inst* insts, int inst, double seed) {
  State* st = insts[inst].st;
  const double g = st->lo_par[0];
  st->lo_par[0] = -insts[inst].alpha * g;
  st->lo_par[1] = st->lo_par[0];
  st->seed = seed;
  st->b = 0; st->rF = 0; st->theta_valid = 0; st->iav = 1; st->rF_used = 0; st->r_cur = 0;
}

int pdsdp_reset(pdsdp_batch* b, int inst, double seed) {
  int rc = check_inst(b, inst);
  if (rc) return rc;
  Instance* I = b->inst[inst];
  I->bmax = 0;
  I->zl_age = 1LL << 40;
  I->iters_total = 0;
  I->dense_mode = 0;
  CK(cudaMemsetAsync(I->desc.st, 0, sizeof(State), b->stream));
  CK(cudaMemsetAsync(I->desc.V, 0, (size_t)I->n * I->ld * sizeof(double), b->stream));
  CK(cudaMemsetAsync(I->desc.F, 0, (size_t)I->n * I->ld * sizeof(double), b->stream));
  init_kernel<<<148, 256, 0, b->stream>>>(b->d_insts, inst, seed);
  init_finalize_kernel<<<1, 1, 0, b->stream>>>(b->d_insts, inst, seed);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(b->stream));
  return PDSDP_OK;
}

int pdsdp_iterate_many(pdsdp_batch* b, int nact, const int32_t* insts, const int32_t* rank, const int32_t* ypar0,
                       const int32_t* flags, int32_t maxpass, int32_t K, const double* conv_thr,
                       const double* stall_thr, double* out, int32_t* steps_done) {
  if (!b || nact < 1 || nact > (int)b->inst.size() || !insts || !rank || !ypar0 || !out)
    return fail(PDSDP_EINVAL, "bad iterate arguments");
  if (K < 1 || K > PDSDP_KMAX) return fail(PDSDP_EINVAL, "K must lie in [1, 64]");
  const int N = (int)b->inst.size();
  int lds = 4, maxr = 1;
  for (int a = 0; a < nact; ++a) {
    const int k = insts[a];
    if (k < 0 || k >= N) return fail(PDSDP_EINVAL, "instance index out of range");
    Instance* I = b->inst[k];
    if (rank[a] < 1 || rank[a] > I->n)
      return fail(PDSDP_EINVAL, "rank r=" + std::to_string(rank[a]) + " outside [1, " + std::to_string(I->n) + "]");
    // target ranks above the block limit run as effective-rank blocks (the
    // positive eigenpairs plus a sentinel); the device reports when those do
    // not fit either
    if (flags && (flags[a] & 8) && std::min(rank[a] + 1, I->n) > PDSDP_BMAX)
      return fail(PDSDP_ERANK, "rank r=" + std::to_string(rank[a]) + " needs an eigen block above 64");
    const int kk = std::min(std::min(rank[a] + 1, I->n), PDSDP_BMAX);
    fill_ctl(b, k, rank[a], ypar0[a], flags ? flags[a] : 0, maxpass, K, conv_thr ? conv_thr[a] : -1.0,
             stall_thr ? stall_thr + (size_t)a * K : nullptr);
    b->h_active[a] = k;
    const int bb = std::min(std::min(I->n, PDSDP_BMAX), block_for(kk, I->n) + ((flags ? flags[a] : 0) >> 8 & 15));
    I->bmax = std::max(I->bmax, bb);
    lds = std::max(lds, I->bmax);
    maxr = std::max(maxr, (int)rank[a]);
  }
  // only the listed instances' control blocks and stop flags are touched:
  // other instances may have chunks in flight on the slot streams
  if (nact == N && b->slot_stream.empty()) {
    CK(cudaMemcpyAsync(b->d_ctl, b->h_ctl, (size_t)N * PDSDP_KMAX * sizeof(Ctl), cudaMemcpyHostToDevice, b->stream));
    CK(cudaMemsetAsync(b->d_stop, 0, (size_t)N * sizeof(int), b->stream));
  } else {
    for (int a = 0; a < nact; ++a) {
      const size_t o = (size_t)insts[a] * PDSDP_KMAX;
      CK(cudaMemcpyAsync(b->d_ctl + o, b->h_ctl + o, (size_t)K * sizeof(Ctl), cudaMemcpyHostToDevice, b->stream));
      CK(cudaMemsetAsync(b->d_stop + insts[a], 0, sizeof(int), b->stream));
    }
  }
  CK(cudaMemcpyAsync(b->d_active, b->h_active, nact * sizeof(int), cudaMemcpyHostToDevice, b->stream));
  const int kp = std::min(RES_KMAX, (2 * std::min(maxr, PDSDP_BMAX) + 3) & ~3);
  const size_t rsm = (size_t)2 * RES_TILE * (kp + 1) * sizeof(double);
  // timing: one event before the chunk and one after every iteration launch,
  // so the span of exactly the executed iterations is known after the sync
  // one persistent launch per chunk (the kernel loops over the steps and stops
  // where the host must look); the verification mode interleaves the
  // entry-wise residual kernel, so it launches step by step
  // refresh the lambda_max(Z) estimate of the Chebyshev interval every
  // PDSDP_ZL_EVERY iterations (Z_k drifts slowly with y; zbound.cuh)
  for (int a = 0; a < nact; ++a) {
    int rc = maybe_zlanczos(b, insts[a], ypar0[a], b->stream);
    if (rc) return rc;
  }
  if (b->timing) CK(cudaEventRecord(b->tev[0], b->stream));
  if (!b->verify_residual) {
    int rc = launch_iterate(b, nact, lds, 0, K);
    if (rc) return rc;
    if (b->timing) CK(cudaEventRecord(b->tev[1], b->stream));
    b->n_launch += 1;
  } else {
    for (int j = 0; j < K; ++j) {
      int rc = launch_iterate(b, nact, lds, j, 1);
      if (rc) return rc;
      residual_kernel<<<dim3(b->max_tiles, nact), RES_THREADS, rsm, b->stream>>>(b->d_insts, b->d_ctl, b->d_active, j);
      CK(cudaGetLastError());
      if (b->timing) CK(cudaEventRecord(b->tev[j + 1], b->stream));
    }
    b->n_launch += K;
  }
  CK(cudaStreamSynchronize(b->stream));
  int done_max = 0;
  for (int a = 0; a < nact; ++a) {
    int done = 0;
    for (int j = 0; j < K; ++j) {
      const double* src = b->h_out + ((size_t)insts[a] * PDSDP_KMAX + j) * PDSDP_OUT_LEN;
      memcpy(out + ((size_t)a * K + j) * PDSDP_OUT_LEN, src, PDSDP_OUT_LEN * sizeof(double));
      // a step whose projection argument has more positive eigenvalues than an
      // eigen block holds did not complete (O_ERR set, X_k / y_k intact): the
      // steps before it count, the caller continues in dense mode
      // (pdsdp_dense_begin / pdsdp_iterate_dense)
      if (src[O_ERR] != 0.0) break;
      if (src[O_DONE] == 1.0) done = j + 1;
    }
    if (steps_done) steps_done[a] = done;
    b->inst[insts[a]]->zl_age += done;
    b->inst[insts[a]]->iters_total += done;
    done_max = std::max(done_max, done);
  }
  if (b->timing && done_max > 0) {
    float t1 = 0.f;
    CK(cudaEventElapsedTime(&t1, b->tev[0], b->tev[b->verify_residual ? done_max : 1]));
    b->t_iter += t1; b->n_iter += done_max;
  }
  return PDSDP_OK;
}

int pdsdp_slots(pdsdp_batch* b, int32_t* nslots_out) {
  if (!b || !nslots_out) return fail(PDSDP_EINVAL, "bad arguments");
  if (b->slot_stream.empty()) {
    int n = 1;
    int rc = max_active_clusters(b, &n);
    if (rc) return rc;
    n = std::min(n, (int)b->inst.size());
    const int N = (int)b->inst.size();
    std::vector<int> ident(N);
    for (int i = 0; i < N; ++i) ident[i] = i;
    CK(cudaMalloc(&b->d_ident, (size_t)N * sizeof(int)));
    CK(cudaMemcpy(b->d_ident, ident.data(), (size_t)N * sizeof(int), cudaMemcpyHostToDevice));
    for (int k = 0; k < n; ++k) {
      cudaStream_t st; cudaEvent_t ev;
      CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      b->slot_stream.push_back(st);
      b->slot_event.push_back(ev);
    }
  }
  *nslots_out = (int)b->slot_stream.size();
  return PDSDP_OK;
}

int pdsdp_chunk_launch(pdsdp_batch* b, int32_t slot, int32_t inst, int32_t rank, int32_t ypar0, int32_t flags,
                       int32_t maxpass, int32_t K, double conv_thr, const double* stall_thr) {
  int rc = check_inst(b, inst);
  if (rc) return rc;
  if (slot < 0 || slot >= (int)b->slot_stream.size()) return fail(PDSDP_EINVAL, "slot out of range (pdsdp_slots)");
  if (K < 1 || K > PDSDP_KMAX) return fail(PDSDP_EINVAL, "K must lie in [1, PDSDP_KMAX]");
  Instance* I = b->inst[inst];
  if (I->dense_mode) return fail(PDSDP_EINVAL, "instance is in dense mode");
  if (rank < 1 || rank > I->n)
    return fail(PDSDP_EINVAL, "rank r=" + std::to_string(rank) + " outside [1, " + std::to_string(I->n) + "]");
  cudaStream_t st = b->slot_stream[slot];
  fill_ctl(b, inst, rank, ypar0, flags, maxpass, K, conv_thr, stall_thr);
  const int kk = std::min(std::min(rank + 1, I->n), PDSDP_BMAX);
  I->bmax = std::max(I->bmax, std::min(std::min(I->n, PDSDP_BMAX), block_for(kk, I->n) + ((flags >> 8) & 15)));
  const size_t o = (size_t)inst * PDSDP_KMAX;
  CK(cudaMemcpyAsync(b->d_ctl + o, b->h_ctl + o, (size_t)K * sizeof(Ctl), cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(b->d_stop + inst, 0, sizeof(int), st));
  if ((rc = maybe_zlanczos(b, inst, ypar0, st))) return rc;
  if ((rc = launch_iterate(b, 1, std::max(4, I->bmax), 0, K, st, b->d_ident + inst))) return rc;
  CK(cudaEventRecord(b->slot_event[slot], st));
  b->n_launch += 1;
  return PDSDP_OK;
}

int pdsdp_chunk_poll(pdsdp_batch* b, int32_t slot) {
  if (!b || slot < 0 || slot >= (int)b->slot_stream.size()) return fail(PDSDP_EINVAL, "slot out of range");
  cudaError_t e = cudaEventQuery(b->slot_event[slot]);
  if (e == cudaSuccess) return 1;
  if (e == cudaErrorNotReady) return 0;
  return fail(PDSDP_ECUDA, std::string("cudaEventQuery: ") + cudaGetErrorString(e));
}

int pdsdp_chunk_collect(pdsdp_batch* b, int32_t slot, int32_t inst, int32_t K, double* out, int32_t* steps_done) {
  int rc = check_inst(b, inst);
  if (rc) return rc;
  if (slot < 0 || slot >= (int)b->slot_stream.size() || !out || K < 1 || K > PDSDP_KMAX)
    return fail(PDSDP_EINVAL, "bad collect arguments");
  CK(cudaEventSynchronize(b->slot_event[slot]));
  int done = 0;
  for (int j = 0; j < K; ++j) {
    const double* src = b->h_out + ((size_t)inst * PDSDP_KMAX + j) * PDSDP_OUT_LEN;
    memcpy(out + (size_t)j * PDSDP_OUT_LEN, src, PDSDP_OUT_LEN * sizeof(double));
    if (src[O_ERR] != 0.0) break;
    if (src[O_DONE] == 1.0) done = j + 1;
  }
  if (steps_done) *steps_done = done;
  b->inst[inst]->zl_age += done;
  b->inst[inst]->iters_total += done;
  return PDSDP_OK;
}

int pdsdp_iterate(pdsdp_batch* b, int nact, const int32_t* insts, const int32_t* rank, const int32_t* ypar,
                  const int32_t* flags, int32_t maxpass, double* out) {
  return pdsdp_iterate_many(b, nact, insts, rank, ypar, flags, maxpass, 1, nullptr, nullptr, out, nullptr);
}

int pdsdp_set_timing(pdsdp_batch* b, int enable) {
  if (!b) return fail(PDSDP_EINVAL, "batch is NULL");
  for (int k = 0; k < 3; ++k)
    if (!b->ev[k]) CK(cudaEventCreate(&b->ev[k]));
  for (int k = 0; k <= PDSDP_KMAX; ++k)
    if (!b->tev[k]) CK(cudaEventCreate(&b->tev[k]));
  b->timing = enable ? 1 : 0;
  b->t_iter = b->n_iter = b->t_res = b->n_res = b->n_launch = 0.0;
  return PDSDP_OK;
}

int pdsdp_set_verify_residual(pdsdp_batch* b, int enable) {
  if (!b) return fail(PDSDP_EINVAL, "batch is NULL");
  b->verify_residual = enable ? 1 : 0;
  return PDSDP_OK;
}

int pdsdp_debug(pdsdp_batch* b, int inst, double* out) {
  int rc = check_inst(b, inst);
  if (rc) return rc;
  if (!out) return fail(PDSDP_EINVAL, "out is NULL");
  State h;
  CK(cudaMemcpy(&h, b->inst[inst]->desc.st, sizeof(State), cudaMemcpyDeviceToHost));
  memcpy(out, h.dbg, sizeof(h.dbg));
  memcpy(out + 256, h.theta, sizeof(h.theta));
  memcpy(out + 320, h.res, sizeof(h.res));
  memcpy(out + 384, h.prof, sizeof(h.prof));
  memcpy(out + 400, h.hdump, sizeof(h.hdump));
  // per-CTA trace of the last flag-bit-6 launch
  CK(cudaMemcpy(out + 4504, b->inst[inst]->desc.trace, (size_t)b->C * 2 * PDSDP_TRACE_CTA * sizeof(double),
                cudaMemcpyDeviceToHost));
  // reset the per-launch accumulators that the kernel adds into
  State* dst = b->inst[inst]->desc.st;
  CK(cudaMemset(&dst->prof[15], 0, sizeof(double)));
  return PDSDP_OK;
}

int pdsdp_kernel_times(pdsdp_batch* b, double* out) {
  if (!b || !out) return fail(PDSDP_EINVAL, "bad arguments");
  out[0] = b->t_iter; out[1] = b->n_iter; out[2] = b->t_res; out[3] = b->n_res; out[4] = b->n_launch;
  return PDSDP_OK;
}

int pdsdp_objective(pdsdp_batch* b, int inst, int which, double* out) {
  int rc = check_inst(b, inst);
  if (rc) return rc;
  if (!out) return fail(PDSDP_EINVAL, "out is NULL");
  if (b->inst[inst]->dense_mode) return dense_objective(b, b->inst[inst], which, out);
  b->h_active[0] = inst;
  CK(cudaMemcpyAsync(b->d_active, b->h_active, sizeof(int), cudaMemcpyHostToDevice, b->stream));
  objective_kernel<<<dim3(148, 1), 256, 0, b->stream>>>(b->d_insts, b->d_active, which ? 1 : 0, b->d_objpart,
                                                       b->d_objcnt, b->d_objres);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, b->d_objres, sizeof(double), cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return PDSDP_OK;
}

int pdsdp_download_x(pdsdp_batch* b, int inst, int which, double* packed_out) {
  int rc = check_inst(b, inst);
  if (rc) return rc;
  if (!packed_out) return fail(PDSDP_EINVAL, "out is NULL");
  Instance* I = b->inst[inst];
  const long long P = I->P;
  const int grid = (int)std::min<long long>(148 * 8, (P + 255) / 256);
  if (I->dense_mode)
    dense_pack_kernel<<<dim3(std::max(1, std::min(8, (I->n + 255) / 256)), I->n), 256, 0, b->stream>>>(
        I->n, I->dd.X[which ? (I->dcur ^ 1) : I->dcur], I->d_packed);
  else
  pack_kernel<<<std::max(grid, 1), 256, 0, b->stream>>>(b->d_insts, inst, which ? 1 : 0, I->d_packed);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(packed_out, I->d_packed, P * sizeof(double), cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return PDSDP_OK;
}

int pdsdp_download_y(pdsdp_batch* b, int inst, int ypar, double* y_out) {
  int rc = check_inst(b, inst);
  if (rc) return rc;
  Instance* I = b->inst[inst];
  if (I->mp == 0) return PDSDP_OK;
  if (!y_out) return fail(PDSDP_EINVAL, "out is NULL");
  CK(cudaMemcpyAsync(y_out, (ypar & 1) ? I->desc.ybuf1 : I->desc.ybuf0, I->mp * sizeof(double),
                     cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return PDSDP_OK;
}

__global__ void gather_T_kernel(const double* __restrict__ packed, const long long* __restrict__ tpos, int nT,
                                double* __restrict__ x) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nT; t += gridDim.x * blockDim.x) x[t] = packed[tpos[t]];
}
__global__ void scatter_T_kernel(const double* __restrict__ x, const long long* __restrict__ tpos, int nT,
                                 double* __restrict__ packed) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nT; t += gridDim.x * blockDim.x) packed[tpos[t]] = x[t];
}

int pdsdp_apply_M(pdsdp_batch* b, int inst, const double* X_packed, double* out) {
  int rc = check_inst(b, inst);
  if (rc) return rc;
  Instance* I = b->inst[inst];
  if (I->mp == 0) return PDSDP_OK;
  if (!X_packed || !out) return fail(PDSDP_EINVAL, "NULL argument");
  OpnormDev& o = I->od;
  long long* dpos = nullptr;
  CK(cudaMalloc(&dpos, std::max<size_t>(1, I->tpos.size()) * sizeof(long long)));
  CK(cudaMemcpyAsync(dpos, I->tpos.data(), I->tpos.size() * sizeof(long long), cudaMemcpyHostToDevice, b->stream));
  CK(cudaMemcpyAsync(I->d_packed, X_packed, I->P * sizeof(double), cudaMemcpyHostToDevice, b->stream));
  if (o.nT) gather_T_kernel<<<std::max(1, std::min(4096, (o.nT + 255) / 256)), 256, 0, b->stream>>>(I->d_packed, dpos, o.nT, o.x);
  seg_dot_kernel<<<o.nseg, 256, 0, b->stream>>>(o);
  seg_final_kernel<<<std::max(1, std::min(1024, (o.mp + 255) / 256)), 256, 0, b->stream>>>(o);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, o.y, I->mp * sizeof(double), cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  cudaFree(dpos);
  return PDSDP_OK;
}

int pdsdp_apply_M_adjoint(pdsdp_batch* b, int inst, const double* y, double* out_packed) {
  int rc = check_inst(b, inst);
  if (rc) return rc;
  Instance* I = b->inst[inst];
  if (!out_packed || (I->mp && !y)) return fail(PDSDP_EINVAL, "NULL argument");
  OpnormDev& o = I->od;
  long long* dpos = nullptr;
  CK(cudaMalloc(&dpos, std::max<size_t>(1, I->tpos.size()) * sizeof(long long)));
  CK(cudaMemcpyAsync(dpos, I->tpos.data(), I->tpos.size() * sizeof(long long), cudaMemcpyHostToDevice, b->stream));
  CK(cudaMemsetAsync(I->d_packed, 0, I->P * sizeof(double), b->stream));
  if (I->mp) CK(cudaMemcpyAsync(o.y, y, I->mp * sizeof(double), cudaMemcpyHostToDevice, b->stream));
  if (o.nT) {
    adjT_kernel<<<std::max(1, std::min(4096, (o.nT + 255) / 256)), 256, 0, b->stream>>>(o);
    scatter_T_kernel<<<std::max(1, std::min(4096, (o.nT + 255) / 256)), 256, 0, b->stream>>>(o.x, dpos, o.nT, I->d_packed);
  }
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out_packed, I->d_packed, I->P * sizeof(double), cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  cudaFree(dpos);
  return PDSDP_OK;
}

int pdsdp_dense_begin(pdsdp_batch* b, int inst, int from_factored) {
  int rc = check_inst(b, inst);
  if (rc) return rc;
  Instance* I = b->inst[inst];
  if ((rc = dense_alloc(I))) return rc;
  DenseDev& D = I->dd;
  const size_t nn = (size_t)I->n * I->n;
  I->dcur = 0;
  if (from_factored) {
    // X_k = F diag(lamF) F^T of the last (possibly unfinished) cluster iteration
    State h;
    CK(cudaMemcpyAsync(&h, I->desc.st, sizeof(State), cudaMemcpyDeviceToHost, b->stream));
    CK(cudaStreamSynchronize(b->stream));
    const int nt = (I->n + RECON_TILE - 1) / RECON_TILE;
    recon_kernel<<<nt * (nt + 1) / 2, 256, 0, b->stream>>>(I->n, I->desc.F, 1, I->desc.ld, nullptr,
                                                          I->desc.st->lamF, nullptr, h.rF_used, D.X[0]);
    CK(cudaGetLastError());
  } else {
    CK(cudaMemsetAsync(D.X[0], 0, nn * sizeof(double), b->stream));
  }
  CK(cudaMemsetAsync(D.X[1], 0, nn * sizeof(double), b->stream));
  CK(cudaStreamSynchronize(b->stream));
  I->dense_mode = 1;
  return PDSDP_OK;
}

int pdsdp_iterate_dense(pdsdp_batch* b, int inst, int32_t r, int32_t ypar, double* out) {
  int rc = check_inst(b, inst);
  if (rc) return rc;
  Instance* I = b->inst[inst];
  if (!I->dense_mode) return fail(PDSDP_EINVAL, "instance is not in dense mode (pdsdp_dense_begin)");
  if (!out) return fail(PDSDP_EINVAL, "out is NULL");
  const int n = I->n, mp = I->mp;
  if (r < 1 || r > n) return fail(PDSDP_EINVAL, "rank r=" + std::to_string(r) + " outside [1, " + std::to_string(n) + "]");
  DenseDev& D = I->dd;
  Inst d = I->desc;
  cudaStream_t s = b->stream;
  const double* Xo = D.X[I->dcur];
  double* Xn = D.X[I->dcur ^ 1];
  const double* yk = (ypar & 1) ? d.ybuf1 : d.ybuf0;
  double* yn = (ypar & 1) ? d.ybuf0 : d.ybuf1;
  const double* zv = (ypar & 1) ? d.zbuf1 : d.zbuf0;
  double* zvn = (ypar & 1) ? d.zbuf0 : d.zbuf1;
  const int gx = std::max(1, std::min(8, (n + 255) / 256));
  // S = X_k - alpha (C + M^T y_k), shifted to SPD
  dense_arg_kernel<<<dim3(gx, n), 256, 0, s>>>(n, Xo, D.W, d.alpha, d.nd, d.du, yk, d);
  if (d.nz) dense_arg_sparse_kernel<<<std::max(1, std::min(4096, (d.nz + 255) / 256)), 256, 0, s>>>(n, d.nz, d.zrow, d.zcol, zv, D.W, d.alpha);
  dense_rowabs_kernel<<<(n + 7) / 8, 256, 0, s>>>(n, D.W, D.rowsum);
  dense_shift_kernel<<<1, 256, 0, s>>>(n, D.W, D.rowsum, D.scal);
  CK(cudaGetLastError());
  // full eigendecomposition: one-sided Jacobi sweeps until no rotation is applied
  const int nn = n + (n & 1);
  const size_t jsm = (size_t)2 * n * sizeof(double);
  CK(cudaFuncSetAttribute(jacobi_round_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(jsm, 1024)));
  CK(cudaFuncSetAttribute(jacobi_round_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(jsm, 1024)));
  // bulk copies need 16-byte aligned rows; they pay off once the matrix no longer sits in L2
  // (n = 4096: 3.75 vs 3.96 s per projection; n = 2048: 0.59 vs 0.54 s)
  const bool tma = (n % 2 == 0) && n >= 3072 && !b->dense_no_tma;
  const double tol = std::max(1e-15, 2.0 * 2.220446049250313e-16 * std::sqrt((double)n));
  int sweeps = 0, conv = (n == 1) ? 1 : 0;
  if (n >= b->bj_nmin && !b->dense_no_block) {
    // blocked rounds: one CTA per pair of 16-row blocks (dense_path.cuh)
    const int nbk = (n + BJ_BS - 1) / BJ_BS, nbe = nbk + (nbk & 1);
    const size_t bsm = block_jacobi_smem_bytes();
    CK(cudaFuncSetAttribute(block_jacobi_round_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
    // the in-CTA eigensolve leaves rows orthogonal to ~1e-14 ||G||_F / g_ii (its rotation
    // threshold), a few 1e-14 relative: the sweep test sits above that floor
    const double tolb = std::max(2e-13, 16.0 * 2.220446049250313e-16 * std::sqrt((double)n));
    for (; sweeps < 60 && !conv; ++sweeps) {
      CK(cudaMemsetAsync(D.maxoff, 0, sizeof(unsigned long long), s));
      for (int t = 0; t < nbe - 1; ++t)
        block_jacobi_round_kernel<<<nbe / 2, BJ_THREADS, bsm, s>>>(n, D.W, t, nbk, tolb, D.maxoff);
      CK(cudaGetLastError());
      unsigned long long bits = 0;
      CK(cudaMemcpyAsync(&bits, D.maxoff, sizeof(bits), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      b->n_launch += nbe - 1;
      double mo;
      memcpy(&mo, &bits, sizeof(mo));
      if (!(mo > tolb)) conv = 1;
    }
  } else
  for (; n > 1 && sweeps < 60 && !conv; ++sweeps) {
    CK(cudaMemsetAsync(D.rot, 0, sizeof(unsigned), s));
    for (int t = 0; t < nn - 1; ++t) {
      if (tma) jacobi_round_tma_kernel<<<nn / 2, DENSE_THREADS, jsm, s>>>(n, D.W, t, tol, D.rot);
      else jacobi_round_kernel<<<nn / 2, DENSE_THREADS, jsm, s>>>(n, D.W, t, tol, D.rot);
    }
    CK(cudaGetLastError());
    unsigned rot = 0;
    CK(cudaMemcpyAsync(&rot, D.rot, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    b->n_launch += nn - 1;
    if (rot == 0) conv = 1;
  }
  eig_finalize_kernel<<<n, 256, 0, s>>>(n, D.W, D.scal, D.lam);
  eig_sort_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, D.lam, D.idx, D.lams);
  eig_select_kernel<<<1, 32, 0, s>>>(n, r, D.lams, D.scal);
  // X+ = sum of the kept positive pairs (symmat.py:212-220)
  const int nt = (n + RECON_TILE - 1) / RECON_TILE;
  recon_kernel<<<nt * (nt + 1) / 2, 256, 0, s>>>(n, D.W, n, 1, D.idx, D.lams, D.scal, 0, Xn);
  CK(cudaGetLastError());
  // dual step, adjoint, residuals
  double* rowt = I->d_rowt;
  CK(cudaMemsetAsync(D.scal + DS_ED2, 0, 5 * sizeof(double), s));
  if (d.nd > 0) {
    dense_quad_kernel<<<n, 256, 0, s>>>(n, Xn, Xo, d.nd, d.du, rowt);
    for (int q = 0; q < d.nd; ++q) {
      reduce_sum_kernel<<<1, 256, 0, s>>>(rowt + (size_t)(2 * q) * n, n, D.scal + DS_QN + q);
      reduce_sum_kernel<<<1, 256, 0, s>>>(rowt + (size_t)(2 * q + 1) * n, n, D.scal + DS_QD + q);
    }
  }
  if (mp > 0) {
    dense_dual_kernel<<<std::max(1, std::min(2048, (mp + 255) / 256)), 256, 0, s>>>(d, Xn, Xo, yk, yn, D.scal, rowt);
    reduce_sum_kernel<<<1, 256, 0, s>>>(rowt, mp, D.scal + DS_ED2);
    reduce_sum_kernel<<<1, 256, 0, s>>>(rowt + mp, mp, D.scal + DS_DYSD);
    reduce_sum_kernel<<<1, 256, 0, s>>>(rowt + 2 * (size_t)mp, mp, D.scal + DS_FIN);
    dense_adjoint_kernel<<<DENSE_GRID, 256, 0, s>>>(d, Xn, Xo, yn, zvn, D.part);
    reduce_sum_kernel<<<1, 256, 0, s>>>(D.part, DENSE_GRID, D.scal + DS_CORR);
  }
  dense_presid_kernel<<<n, 256, 0, s>>>(d, Xn, Xo, rowt);
  reduce_sum_kernel<<<1, 256, 0, s>>>(rowt, n, D.scal + DS_DENSE);
  reduce_sum_kernel<<<1, 256, 0, s>>>(rowt + n, n, D.scal + DS_ROT);
  CK(cudaGetLastError());
  double h[DENSE_SCAL];
  CK(cudaMemcpyAsync(h, D.scal, DENSE_SCAL * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  b->n_launch += 16;
  I->dcur ^= 1;
  for (int k = 0; k < PDSDP_OUT_LEN; ++k) out[k] = 0.0;
  const double fin = (h[DS_FIN] == 0.0 && h[DS_ROT] == 0.0 && h[DS_XFIN] == 1.0) ? 1.0 : 0.0;
  out[O_EPS_P] = std::sqrt(std::max(h[DS_DENSE] + h[DS_CORR], 0.0));
  out[O_EPS_D] = std::sqrt(std::max(h[DS_ED2], 0.0));
  out[O_LAM] = h[DS_LAMK];
  out[O_FIN] = fin;
  out[O_PASSES] = sweeps;
  out[O_EIGCONV] = conv;
  out[O_DENSE] = h[DS_DENSE];
  out[O_CORR] = h[DS_CORR];
  out[O_ED2] = h[DS_ED2];
  out[O_BLK] = n;
  out[O_DONE] = 1.0;
  out[O_DENSE_EXACT] = NAN;
  return PDSDP_OK;
}

int pdsdp_aproj_psd(int32_t n, const double* S_packed, int32_t r, double* P_packed_out, double* lambda_out) {
  if (n < 1 || !S_packed || !P_packed_out) return fail(PDSDP_EINVAL, "bad aproj arguments");
  if (r < 1 || r > n) return fail(PDSDP_EINVAL, "rank r=" + std::to_string(r) + " outside [1, " + std::to_string(n) + "]");
  const long long P = packed_len(n);
  std::vector<double> C(P);
  for (long long q = 0; q < P; ++q) C[q] = -S_packed[q];
  pdsdp_problem pr{};
  pr.n = n; pr.m = 0; pr.p = 0; pr.C_packed = C.data();
  int64_t rp0 = 0;
  pr.row_ptr = &rp0;
  pdsdp_batch* b = nullptr;
  int rc = pdsdp_batch_create(1, &pr, &b);
  if (rc) return rc;
  int32_t inst = 0, rr = r, yp = 0, fl = 1 | 2 | 8;
  double out[PDSDP_OUT_LEN];
  rc = pdsdp_set_alpha(b, 0, 1.0);
  if (!rc) rc = pdsdp_reset(b, 0, 0.0);
  // the top r+1 pairs fit an eigen block: subspace iteration in one cluster;
  // otherwise the full eigendecomposition (the reference switches to dense
  // eigh for 2 (r+1) > n, symmat.py:181-185)
  if (std::min(r + 1, n) <= PDSDP_BMAX) {
    if (!rc) rc = pdsdp_iterate(b, 1, &inst, &rr, &yp, &fl, 200, out);
  } else {
    if (!rc) rc = pdsdp_dense_begin(b, 0, 0);
    if (!rc) rc = pdsdp_iterate_dense(b, 0, rr, yp, out);
  }
  if (!rc) rc = pdsdp_download_x(b, 0, 0, P_packed_out);
  if (!rc && lambda_out) *lambda_out = out[PDSDP_OUT_LAMBDA];
  std::string e = g_err;
  pdsdp_batch_destroy(b);
  g_err = e;
  return rc;
}

}  // extern "C"
