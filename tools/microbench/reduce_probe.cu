// Cluster reduction of q doubles over 16 CTAs (every CTA ends with all q
// sums, added in rank order): partials through L2 (st.global + cluster
// barrier + 16 ld.global.cg per element) vs through distributed shared
// memory (st.shared + cluster barrier + 16 ld.shared::cluster per element).
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

template <int MODE>
__global__ void __launch_bounds__(512, 1) probe(double* red, int q, int reps, long long* cyc, double* sink) {
  __shared__ double part[2][2048];
  __shared__ double dst[2048];
  cg::cluster_group cl = cg::this_cluster();
  const int C = cl.num_blocks(), c = cl.block_rank();
  double acc = 0.0;
  cl.sync();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    const int par = rep & 1;
    // partial
    for (int i = threadIdx.x; i < q; i += blockDim.x) {
      const double v = 1e-3 * (i + c + rep);
      if (MODE == 0) red[((size_t)par * C + c) * 4096 + i] = v;
      else part[par][i] = v;
    }
    cl.sync();
    for (int i = threadIdx.x; i < q; i += blockDim.x) {
      double v[16];
      if (MODE == 0) {
#pragma unroll
        for (int cc = 0; cc < 16; ++cc) v[cc] = (cc < C) ? __ldcg(red + ((size_t)par * C + cc) * 4096 + i) : 0.0;
      } else {
#pragma unroll
        for (int cc = 0; cc < 16; ++cc) {
          const double* rp = cl.map_shared_rank(&part[par][0], cc);
          v[cc] = (cc < C) ? rp[i] : 0.0;
        }
      }
      double s = 0.0;
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) s += v[cc];
      dst[i] = s;
    }
    __syncthreads();
    acc += dst[(threadIdx.x * 7) % q];
  }
  cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  double *red, *sink; long long* cyc;
  cudaMalloc(&red, 2 * 16 * 4096 * 8); cudaMalloc(&sink, 16 * 512 * 8); cudaMalloc(&cyc, 64 * 8);
  for (int mode = 0; mode < 2; ++mode) {
    void* f = mode == 0 ? (void*)probe<0> : (void*)probe<1>;
    cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int q : {1, 160, 256, 512, 1568, 2048}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(16); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 0;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaError_t e = mode == 0 ? cudaLaunchKernelEx(&cfg, probe<0>, red, q, 400, cyc, sink)
                                : cudaLaunchKernelEx(&cfg, probe<1>, red, q, 400, cyc, sink);
      cudaError_t e2 = cudaDeviceSynchronize();
      long long h[16]; cudaMemcpy(h, cyc, 16 * 8, cudaMemcpyDeviceToHost);
      printf("%s q=%4d: %6lld cycles per reduction (%.2f us) [%s %s]\n", mode == 0 ? "L2   " : "DSMEM", q, h[0],
             h[0] / 1965.0, cudaGetErrorString(e), cudaGetErrorString(e2));
    }
  }
  return 0;
}
