// Pieces of one operator step in isolation (one 384-thread CTA, data in
// shared memory as in the iteration kernel): the DMMA Gram partial of the
// own rows (gram_mma2, rF x bc over 125 rows) and the own-row sparse product
// over a staged operand block (bc = 16), timed with clock64.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "iterate.cuh"

using namespace pdsdp;

// per-thread FMA Gram: thread (o, slice) sums rows of its slice; slices of
// an output added in slice order
__device__ void gram_fma(const double* A, int lda, int na, const double* B, int ldb, int nb, int nrows,
                         double* gout, double* scr) {
  const int q = na * nb, tid = threadIdx.x, nt = blockDim.x;
  const int S = q >= nt ? 1 : nt / q;
  const int len = (nrows + S - 1) / S;
  for (int o0 = 0; o0 < q; o0 += nt) {
    const int o = o0 + (tid % min(q, nt)), sl = tid / min(q, nt);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    if (o < q && sl < S) {
      const int i = o / nb, j = o - i * nb;
      const int ra = sl * len, rb = min(nrows, ra + len);
      int rho = ra;
      for (; rho + 4 <= rb; rho += 4) {
        s0 = fma(A[rho * lda + i], B[rho * ldb + j], s0);
        s1 = fma(A[(rho + 1) * lda + i], B[(rho + 1) * ldb + j], s1);
        s2 = fma(A[(rho + 2) * lda + i], B[(rho + 2) * ldb + j], s2);
        s3 = fma(A[(rho + 3) * lda + i], B[(rho + 3) * ldb + j], s3);
      }
      for (; rho < rb; ++rho) s0 = fma(A[rho * lda + i], B[rho * ldb + j], s0);
    }
    const double v = (s0 + s1) + (s2 + s3);
    if (S == 1) {
      if (o < q) gout[o] = v;
    } else {
      if (sl < S) scr[sl * q + (o - o0)] = v;
      __syncthreads();
      if (tid < q) {
        double t = 0.0;
        for (int k = 0; k < S; ++k) t += scr[k * q + tid];
        gout[tid] = t;
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(384, 1) probe(const int* zp_g, const int* zc_g, const double* zv_g, double* gout,
                                                int nl, int rF, int bc, int reps, long long* cyc, double* sink) {
  extern __shared__ double sm[];
  double* SF = sm;                      // nl x 64
  double* yo = SF + 125 * 40;           // nl x 16
  double* wsm = yo + 125 * 16;          // GRAM_SCR
  double* ys = wsm + PDSDP_GRAM_SCR;    // 800 x 16 staged operand
  int* zc = (int*)(ys + 800 * 16);
  double* zvs = (double*)(zc + 4096);
  int* zp = (int*)(zvs + 4096);
  const int tid = threadIdx.x;
  for (int i = tid; i < 125 * 40; i += blockDim.x) SF[i] = 1e-3 * (i % 97);
  for (int i = tid; i < 125 * 16; i += blockDim.x) yo[i] = 1e-3 * (i % 89);
  for (int i = tid; i < 800 * 16; i += blockDim.x) ys[i] = 1e-4 * (i % 101);
  const int nz = zp_g[nl];
  for (int e = tid; e < nz; e += blockDim.x) { zc[e] = zc_g[e]; zvs[e] = zv_g[e]; }
  for (int i = tid; i <= nl; i += blockDim.x) zp[i] = zp_g[i];
  __syncthreads();
  long long tg = 0, ts = 0, tf = 0, tu = 0;
  double acc = 0.0;
  for (int rep = 0; rep < reps; ++rep) {
    __syncthreads();
    long long t0 = clock64();
    gram_mma2(SF, 40, rF, yo, 16, bc, 0, nl, gout, wsm);
    __syncthreads();
    long long t1 = clock64();
    // sparse product: items (row, 4-column chunk), 3 per thread
    const int nch = bc >> 2, nitems = nl * nch;
    for (int it = tid; it < nitems; it += blockDim.x) {
      const int lr = it / nch, cq = it - lr * nch;
      const double* yb = ys + 4 * cq;
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
      for (int e = zp[lr]; e < zp[lr + 1]; ++e) {
        const int q = zc[e];
        const double z = zvs[e];
        const double2 p0 = *reinterpret_cast<const double2*>(yb + (size_t)q * 16);
        const double2 p1 = *reinterpret_cast<const double2*>(yb + (size_t)q * 16 + 2);
        a0 = fma(z, p0.x, a0); a1 = fma(z, p0.y, a1); a2 = fma(z, p1.x, a2); a3 = fma(z, p1.y, a3);
      }
      acc += a0 + a1 + a2 + a3;
    }
    __syncthreads();
    long long t2 = clock64();
    gram_fma(SF, 40, rF, yo, 16, bc, nl, gout, wsm);
    __syncthreads();
    long long t3 = clock64();
    // sparse product, 4 slots per round with batched loads
    for (int it = tid; it < nitems; it += blockDim.x) {
      const int lr = it / nch, cq = it - lr * nch;
      const double* yb = ys + 4 * cq;
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
      int e = zp[lr];
      const int e1 = zp[lr + 1];
      for (; e + 4 <= e1; e += 4) {
        int q[4]; double z[4]; double2 p[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) { q[k] = zc[e + k]; z[k] = zvs[e + k]; }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          p[2 * k] = *reinterpret_cast<const double2*>(yb + (size_t)q[k] * 16);
          p[2 * k + 1] = *reinterpret_cast<const double2*>(yb + (size_t)q[k] * 16 + 2);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          a0 = fma(z[k], p[2 * k].x, a0); a1 = fma(z[k], p[2 * k].y, a1);
          a2 = fma(z[k], p[2 * k + 1].x, a2); a3 = fma(z[k], p[2 * k + 1].y, a3);
        }
      }
      for (; e < e1; ++e) {
        const int q = zc[e];
        const double z = zvs[e];
        const double2 p0 = *reinterpret_cast<const double2*>(yb + (size_t)q * 16);
        const double2 p1 = *reinterpret_cast<const double2*>(yb + (size_t)q * 16 + 2);
        a0 = fma(z, p0.x, a0); a1 = fma(z, p0.y, a1); a2 = fma(z, p1.x, a2); a3 = fma(z, p1.y, a3);
      }
      acc += a0 + a1 + a2 + a3;
    }
    __syncthreads();
    long long t4 = clock64();
    tg += t1 - t0; ts += t2 - t1; tf += t3 - t2; tu += t4 - t3;
  }
  if (tid == 0) { cyc[0] = tg / reps; cyc[1] = ts / reps; cyc[2] = tf / reps; cyc[3] = tu / reps; }
  sink[tid] = acc;
}

int main() {
  const int n = 2000, nl = 125, deg = 21;
  std::vector<int> ptr(nl + 1, 0), col;
  std::vector<double> val;
  srand(3);
  for (int i = 0; i < nl; ++i) {
    std::vector<int> cs;
    for (int k = 0; k < deg; ++k) cs.push_back(rand() % 800);
    std::sort(cs.begin(), cs.end());
    cs.erase(std::unique(cs.begin(), cs.end()), cs.end());
    for (int q : cs) { col.push_back(q); val.push_back(0.5 - rand() / (double)RAND_MAX); }
    ptr[i + 1] = (int)col.size();
  }
  int *dp, *dc; double *dv, *gout, *sink; long long* cyc;
  cudaMalloc(&dp, (nl + 1) * 4); cudaMalloc(&dc, col.size() * 4); cudaMalloc(&dv, val.size() * 8);
  cudaMalloc(&gout, 8192 * 8); cudaMalloc(&sink, 512 * 8); cudaMalloc(&cyc, 64 * 8);
  cudaMemcpy(dp, ptr.data(), (nl + 1) * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dc, col.data(), col.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, val.data(), val.size() * 8, cudaMemcpyHostToDevice);
  const int smem = (125 * 56 + PDSDP_GRAM_SCR + 800 * 16 + 4096) * 8 + (4096 + 200) * 4;
  printf("smem %d\n", smem);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rF : {10, 20, 37}) {
    probe<<<1, 384, smem>>>(dp, dc, dv, gout, nl, rF, 16, 100, cyc, sink);
    cudaError_t e0 = cudaGetLastError(); cudaError_t e = cudaDeviceSynchronize(); if (e == cudaSuccess) e = e0;
    long long h[4]; cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
    printf("rF=%2d bc=16 rows=%d: gram_mma2 %6lld cyc  gram_fma %6lld cyc | sparse product %6lld cyc, unrolled x4 %6lld cyc  nnz=%zu [%s]\n", rF,
           nl, h[0], h[2], h[1], h[3], col.size(), cudaGetErrorString(e));
  }
  return 0;
}
