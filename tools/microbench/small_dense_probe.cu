// Cycles per call of the b x b shared-memory routines of small_dense.cuh
// (one 512-thread CTA; the iteration kernel runs them redundantly per CTA).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../paper_1810_05231_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "small_dense.cuh"

using namespace pdsdp;

__global__ void __launch_bounds__(512, 1) probe(const double* Gin, const double* Hin, int b, int reps, long long* cyc,
                                                double* out) {
  extern __shared__ double sm[];
  const int lds = 65;
  double* A = sm;
  double* L = A + 64 * lds;
  double* M = L + 64 * lds;
  double* Q = M + 64 * lds;
  double* T = Q + 64 * lds;
  double* cs = T + 64 * lds;
  double* dsc = cs + 4 * 64;
  double* theta = dsc + 64;
  int* tab = (int*)(theta + 64);
  int* perm = tab + 64 * 64;
  int* flag = perm + 64;
  long long t_chol = 0, t_tri = 0, t_jac = 0, t_sort = 0, t_gemm = 0, t_j4 = 0, t_cr = 0, t_tr = 0;
  int sweeps = 0, sweeps4 = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int e = threadIdx.x; e < b * b; e += blockDim.x) A[(e / b) * lds + e % b] = Gin[e];
    __syncthreads();
    long long t0 = clock64();
    bool ok = chol_scaled_1s(A, b, lds, dsc);
    long long t1 = clock64();
    tri_inv_lower_1s(A, L, b, lds);
    long long t2 = clock64();
    sm_gemm(L, lds, A, lds, M, lds, b, b, b);
    long long t3 = clock64();
    for (int e = threadIdx.x; e < b * b; e += blockDim.x) { out[300 + e % 64] = 0; }
    for (int e = threadIdx.x; e < b * b; e += blockDim.x) Q[(e / b) * lds + e % b] = Gin[e];
    __syncthreads();
    long long t9 = clock64();
    chol_scaled_rows(Q, b, lds, dsc);
    long long t10 = clock64();
    tri_inv_lower_rows(Q, T, b, lds);
    long long t11 = clock64();
    double md = 0.0;
    for (int e = threadIdx.x; e < b * b; e += blockDim.x) md = fmax(md, fabs(T[(e / b) * lds + e % b] - L[(e / b) * lds + e % b]));
    if (md > 1e-12) out[1] = md;
    t_cr += t10 - t9; t_tr += t11 - t10;
    for (int e = threadIdx.x; e < b * b; e += blockDim.x) A[(e / b) * lds + e % b] = Hin[e];
    __syncthreads();
    long long t4 = clock64();
    double *Aj, *Qj;
    jacobi_eig3(A, M, Q, T, b, lds, cs, tab, flag, b, &Aj, &Qj);
    long long t5 = clock64();
    sort_desc(Aj, b, lds, theta, perm);
    long long t6 = clock64();
    if (threadIdx.x < b) out[100 + threadIdx.x] = theta[threadIdx.x];
    __syncthreads();
    for (int e = threadIdx.x; e < b * b; e += blockDim.x) A[(e / b) * lds + e % b] = Hin[e];
    __syncthreads();
    long long t7 = clock64();
    jacobi_eig4(A, M, Q, T, b, lds, cs, tab, flag + 1, b, &Aj, &Qj);
    long long t8 = clock64();
    sort_desc(Aj, b, lds, theta, perm);
    if (threadIdx.x < b) out[200 + threadIdx.x] = theta[threadIdx.x] - out[100 + threadIdx.x];
    t_j4 += t8 - t7; sweeps4 += flag[1];
    t_chol += t1 - t0; t_tri += t2 - t1; t_gemm += t3 - t2; t_jac += t5 - t4; t_sort += t6 - t5;
    sweeps += flag[0];
    if (!ok && threadIdx.x == 0) out[0] = -1;
    __syncthreads();
    if (threadIdx.x < b) out[1 + threadIdx.x] = theta[threadIdx.x];
  }
  if (threadIdx.x == 0) {
    cyc[0] = t_chol / reps; cyc[1] = t_tri / reps; cyc[2] = t_gemm / reps; cyc[3] = t_jac / reps;
    cyc[4] = t_sort / reps; cyc[5] = sweeps; cyc[6] = t_j4 / reps; cyc[7] = sweeps4; cyc[8] = t_cr / reps; cyc[9] = t_tr / reps;
  }
}

int main() {
  const int reps = 50;
  long long* cyc; cudaMalloc(&cyc, 64 * 8);
  double *G, *H, *out;
  cudaMalloc(&G, 64 * 64 * 8); cudaMalloc(&H, 64 * 64 * 8); cudaMalloc(&out, 512 * 8);
  const size_t smem = 5 * 64 * 65 * 8 + (4 * 64 + 64 + 64) * 8 + (64 * 64 + 64 + 8) * 4;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  srand(1);
  for (int b : {8, 16, 28, 40, 64}) {
    for (double off : {1e-3, 1e-1}) {
      std::vector<double> g(b * b), h(b * b);
      for (int i = 0; i < b; ++i)
        for (int j = 0; j <= i; ++j) {
          double u = (rand() / (double)RAND_MAX - 0.5);
          double v = (rand() / (double)RAND_MAX - 0.5);
          g[i * b + j] = g[j * b + i] = (i == j) ? 1.0 + 0.1 * i : off * u;
          h[i * b + j] = h[j * b + i] = (i == j) ? 250.0 - 9.0 * i : off * 100.0 * v;
        }
      cudaMemcpy(G, g.data(), b * b * 8, cudaMemcpyHostToDevice);
      cudaMemcpy(H, h.data(), b * b * 8, cudaMemcpyHostToDevice);
      probe<<<1, 512, smem>>>(G, H, b, reps, cyc, out);
      cudaError_t e = cudaDeviceSynchronize();
      long long c[10]; cudaMemcpy(c, cyc, 10 * 8, cudaMemcpyDeviceToHost);
      double o1; cudaMemcpy(&o1, out + 1, 8, cudaMemcpyDeviceToHost);
      double dv[64]; cudaMemcpy(dv, out + 200, 64 * 8, cudaMemcpyDeviceToHost);
      double mx = 0; for (int i = 0; i < b; ++i) mx = fmax(mx, fabs(dv[i]));
      printf("b=%2d off=%.0e: chol %6lld  tri_inv %6lld  gemm %6lld  jacobi %7lld (%.2f sweeps, %5.0f cyc/sweep)  sort %5lld  [%s]\n",
             b, off, c[0], c[1], c[2], c[3], c[5] / (double)reps, c[3] / (c[5] / (double)reps), c[4], cudaGetErrorString(e));
      printf("        chol_rows %6lld  tri_inv_rows %6lld  (max |L^-1 diff| flag %.1e)\n", c[8], c[9], o1);
      printf("        jacobi_eig4 %7lld (%.2f sweeps, %5.0f cyc/sweep)  max |dtheta| vs eig3 %.2e\n", c[6], c[7] / (double)reps,
             c[6] / (c[7] / (double)reps), mx);
    }
  }
  return 0;
}
