// Cost of the pieces of one Jacobi round (small_dense.cuh jacobi_eig4):
// a block barrier, the FP64 rotation chain (rcp/rsqrt + Newton), and a
// dependent shared-memory load -> FMA -> store item.  One CTA, 384 threads.
#include <cstdio>
#include "small_dense.cuh"
using namespace pdsdp;

__global__ void __launch_bounds__(384, 1) probe(int reps, long long* cyc, double* out) {
  extern __shared__ double sm[];
  double* A = sm;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) A[i] = 1.0 + 1e-3 * i;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) __syncthreads();
  long long t1 = clock64();
  double acc = 0.0;
  // rotation chain (thread-local, dependent through A)
  double apq = A[threadIdx.x % 64] * 1e-3, app = A[1], aqq = A[2];
  for (int r = 0; r < reps; ++r) {
    const double tau = (aqq - app) * fast_rcp(2.0 * apq);
    const double at = fabs(tau);
    const double u = fma(tau, tau, 1.0);
    double tt = fast_rcp(at + u * fast_rsqrt(u));
    tt = (tau >= 0.0) ? tt : -tt;
    const double c = fast_rsqrt(fma(tt, tt, 1.0));
    const double s = tt * c;
    apq = fma(s, 1e-20, apq);      // carry the dependence
    acc += c;
  }
  long long t2 = clock64();
  // rotation chain + barrier (phase 1 of a round)
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x < 14) {
      const double tau = (aqq - app) * fast_rcp(2.0 * apq);
      const double at = fabs(tau);
      const double u = fma(tau, tau, 1.0);
      double tt = fast_rcp(at + u * fast_rsqrt(u));
      tt = (tau >= 0.0) ? tt : -tt;
      const double c = fast_rsqrt(fma(tt, tt, 1.0));
      A[2048 + threadIdx.x] = c; A[2100 + threadIdx.x] = tt * c;
    }
    __syncthreads();
    apq = fma(A[2048 + (threadIdx.x % 14)], 1e-20, apq);
  }
  long long t3 = clock64();
  // phase-2 like item: LDS index -> LDS coeffs -> 4 LDS -> FMAs -> 4 STS, one per thread, + barrier
  for (int r = 0; r < reps; ++r) {
    const int k = (threadIdx.x * 7 + r) % 100;
    const int a = (int)A[3000 + k] & 15;
    const double ca = A[2048 + a], sa = A[2100 + a];
    const int base = (k * 13) % 900;
    const double a00 = A[base], a01 = A[base + 1], a10 = A[base + 64], a11 = A[base + 65];
    const double x00 = fma(-sa, a01, ca * a00), x01 = fma(sa, a00, ca * a01);
    const double x10 = fma(-sa, a11, ca * a10), x11 = fma(sa, a10, ca * a11);
    A[1024 + base] = fma(-sa, x10, ca * x00); A[1025 + base] = fma(sa, x00, ca * x10);
    A[1088 + base] = fma(-sa, x11, ca * x01); A[1089 + base] = fma(sa, x01, ca * x11);
    __syncthreads();
  }
  long long t4 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
  out[threadIdx.x] = acc + apq;
}

int main() {
  long long* cyc; cudaMalloc(&cyc, 64);
  double* out; cudaMalloc(&out, 4096);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 8);
  const int reps = 1000;
  probe<<<1, 384, 4096 * 8>>>(reps, cyc, out);
  cudaError_t e = cudaDeviceSynchronize();
  long long c[4]; cudaMemcpy(c, cyc, 32, cudaMemcpyDeviceToHost);
  printf("per rep (cycles): barrier %.1f | rotation chain %.1f | rotation + barrier %.1f | item + barrier %.1f  [%s]\n",
         c[0] / (double)reps, c[1] / (double)reps, c[2] / (double)reps, c[3] / (double)reps, cudaGetErrorString(e));
  return 0;
}
