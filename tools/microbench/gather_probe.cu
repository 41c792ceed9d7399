// Sparse product Z*Y of one operator step inside a 16-CTA cluster (n rows,
// ~deg nnz per row, Y n x bcp row-major in global): each CTA owns n/16 rows
// and gathers the Y rows its Z slots name straight from L2/L1 (no staging).
// Reports cycles per step (cluster barrier + gather-FMA) for bcp in {8,16,28}.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

template <int MODE>
__global__ void __launch_bounds__(512, 1) probe(const int* __restrict__ zptr, const int* __restrict__ zcol,
                                                const double* __restrict__ zval, double* Y, int n, int bcp, int reps,
                                                long long* cyc, double* sink) {
  extern __shared__ double smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int C = cl.num_blocks(), c = cl.block_rank();
  const int r0 = (int)((long long)n * c / C), r1 = (int)((long long)n * (c + 1) / C), nl = r1 - r0;
  // own Z rows in smem
  const int z0 = zptr[r0], nz = zptr[r1] - z0;
  int* zc = (int*)smem;
  double* zv = (double*)(zc + ((nz + 1) & ~1));
  int* zp = (int*)(zv + nz);
  for (int e = threadIdx.x; e < nz; e += blockDim.x) { zc[e] = zcol[z0 + e]; zv[e] = zval[z0 + e]; }
  for (int i = threadIdx.x; i <= nl; i += blockDim.x) zp[i] = zptr[r0 + i] - z0;
  __syncthreads();
  const int nch = bcp >> 2, nitems = nl * nch;
  cl.sync();
  long long t0 = clock64();
  double acc = 0.0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int it = threadIdx.x; it < nitems; it += blockDim.x) {
      const int lr = it / nch, cq = it - lr * nch;
      const double* yb = Y + 4 * cq;
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
      const int e1 = zp[lr + 1];
      int e = zp[lr];
      if (MODE == 0) {
        for (; e < e1; ++e) {
          const int q = zc[e];
          const double z = zv[e];
          const double2 p0 = *reinterpret_cast<const double2*>(yb + (size_t)q * bcp);
          const double2 p1 = *reinterpret_cast<const double2*>(yb + (size_t)q * bcp + 2);
          a0 = fma(z, p0.x, a0); a1 = fma(z, p0.y, a1); a2 = fma(z, p1.x, a2); a3 = fma(z, p1.y, a3);
        }
      } else {
        // 4-deep software pipeline of the row loads
        for (; e + 4 <= e1; e += 4) {
          double2 p[8];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int q = zc[e + k];
            p[2 * k] = __ldcg(reinterpret_cast<const double2*>(yb + (size_t)q * bcp));
            p[2 * k + 1] = __ldcg(reinterpret_cast<const double2*>(yb + (size_t)q * bcp + 2));
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double z = zv[e + k];
            a0 = fma(z, p[2 * k].x, a0); a1 = fma(z, p[2 * k].y, a1);
            a2 = fma(z, p[2 * k + 1].x, a2); a3 = fma(z, p[2 * k + 1].y, a3);
          }
        }
        for (; e < e1; ++e) {
          const int q = zc[e];
          const double z = zv[e];
          const double2 p0 = __ldcg(reinterpret_cast<const double2*>(yb + (size_t)q * bcp));
          const double2 p1 = __ldcg(reinterpret_cast<const double2*>(yb + (size_t)q * bcp + 2));
          a0 = fma(z, p0.x, a0); a1 = fma(z, p0.y, a1); a2 = fma(z, p1.x, a2); a3 = fma(z, p1.y, a3);
        }
      }
      // write back own rows (next step's operand), like the recurrence does
      double* o = Y + (size_t)(r0 + lr) * bcp + 4 * cq;
      o[0] = 1e-3 * a0 + o[0]; o[1] = 1e-3 * a1 + o[1]; o[2] = 1e-3 * a2 + o[2]; o[3] = 1e-3 * a3 + o[3];
      acc += a0;
    }
    cl.sync();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  const int n = 2000, deg = 21, C = 16;
  std::vector<int> ptr(n + 1, 0), col;
  std::vector<double> val;
  srand(7);
  for (int i = 0; i < n; ++i) {
    std::vector<int> cs;
    cs.push_back(i);
    for (int k = 0; k < deg - 1; ++k) cs.push_back(rand() % n);
    std::sort(cs.begin(), cs.end());
    cs.erase(std::unique(cs.begin(), cs.end()), cs.end());
    for (int q : cs) { col.push_back(q); val.push_back(0.5 - rand() / (double)RAND_MAX); }
    ptr[i + 1] = (int)col.size();
  }
  int *dp, *dc; double *dv, *Y, *sink; long long* cyc;
  cudaMalloc(&dp, (n + 1) * 4); cudaMalloc(&dc, col.size() * 4); cudaMalloc(&dv, val.size() * 8);
  cudaMalloc(&Y, (size_t)n * 64 * 8); cudaMalloc(&sink, 16 * 512 * 8); cudaMalloc(&cyc, 64 * 8);
  cudaMemcpy(dp, ptr.data(), (n + 1) * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dc, col.data(), col.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, val.data(), val.size() * 8, cudaMemcpyHostToDevice);
  cudaMemset(Y, 0, (size_t)n * 64 * 8);
  const int smem = 200 * 1024;
  for (int mode = 0; mode < 2; ++mode) {
    void* f = mode == 0 ? (void*)probe<0> : (void*)probe<1>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int bcp : {8, 16, 28}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(C); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      const int reps = 200;
      cudaError_t e;
      if (mode == 0) e = cudaLaunchKernelEx(&cfg, probe<0>, (const int*)dp, (const int*)dc, (const double*)dv, Y, n, bcp, reps, cyc, sink);
      else e = cudaLaunchKernelEx(&cfg, probe<1>, (const int*)dp, (const int*)dc, (const double*)dv, Y, n, bcp, reps, cyc, sink);
      cudaError_t e2 = cudaDeviceSynchronize();
      long long h[16]; cudaMemcpy(h, cyc, 16 * 8, cudaMemcpyDeviceToHost);
      long long mx = 0; for (int i = 0; i < 16; ++i) mx = std::max(mx, h[i]);
      printf("mode %d (%s) bcp=%2d: %6lld cycles/step (incl. cluster.sync) = %.2f us  nnz=%zu [%s %s]\n", mode,
             mode == 0 ? "plain ld" : "ldcg x4 pipelined", bcp, mx, mx / 1965.0, col.size(), cudaGetErrorString(e),
             cudaGetErrorString(e2));
    }
  }
  return 0;
}
