// Per-SM ingress bandwidth inside a 16-CTA cluster: every CTA needs the whole
// Y block (rows of all CTAs).  Variants: (a) TMA bulk multicast of each CTA's
// own rows to all, (b) per-CTA unicast bulk copies of all rows, (c) per-thread
// 16-byte cp.async of all rows, (d) plain coalesced vector loads.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(512, 1)
probe(const double* __restrict__ Y, int nbytes_total, int reps, long long* cyc, double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long mb;
  cg::cluster_group cl = cg::this_cluster();
  const int C = 16, c = cl.block_rank();
  const int block = nbytes_total / C;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&mb)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cl.sync();
  unsigned phase = 0;
  double acc = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (MODE == 0 || MODE == 1) {
      if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&mb)), "r"(nbytes_total) : "memory");
        if (MODE == 0) {
          for (int off = 0; off < block; off += 32768) {
            int piece = min(32768, block - off);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
                         ::"r"(su(sm + c * block + off)), "l"((const char*)Y + c * block + off), "r"(piece), "r"(su(&mb)), "h"((unsigned short)0xFFFF) : "memory");
          }
        } else {
          for (int off = 0; off < nbytes_total; off += 32768) {
            int piece = min(32768, nbytes_total - off);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su(sm + off)), "l"((const char*)Y + off), "r"(piece), "r"(su(&mb)) : "memory");
          }
        }
      }
      asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(su(&mb)), "r"(phase) : "memory");
      phase ^= 1;
    } else if (MODE == 2) {
      for (int i = threadIdx.x * 16; i < nbytes_total; i += blockDim.x * 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(sm + i)), "l"((const char*)Y + i) : "memory");
      asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
      __syncthreads();
    } else {
      const double2* src = reinterpret_cast<const double2*>(Y);
      double2* dst = reinterpret_cast<double2*>(sm);
      for (int i = threadIdx.x; i < nbytes_total / 16; i += blockDim.x) dst[i] = __ldcg(src + i);
      __syncthreads();
    }
    acc += reinterpret_cast<double*>(sm)[(threadIdx.x * 7 + r) % (nbytes_total / 8)];
    cl.sync();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  const int nbytes = 128 * 1024;   // 2000 x 8 doubles = 128 KB per round
  double* Y; cudaMalloc(&Y, nbytes); cudaMemset(Y, 0, nbytes);
  long long* cyc; cudaMalloc(&cyc, 1024 * 8);
  double* sink; cudaMalloc(&sink, 16 * 512 * 8 * 16);
  const int smem = nbytes;
  cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int f : {0, 1, 2, 3}) cudaFuncSetAttribute(f == 0 ? (void*)probe<0> : f == 1 ? (void*)probe<1> : f == 2 ? (void*)probe<2> : (void*)probe<3>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const char* names[4] = {"TMA multicast (own block -> all)", "TMA unicast (all rows per CTA)", "cp.async 16B per thread", "ldcg double2 per thread"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int grids : {16, 16 * 8}) {
      int reps = 200;
      if (mode == 0) probe<0><<<grids, 512, smem>>>(Y, nbytes, reps, cyc, sink);
      if (mode == 1) probe<1><<<grids, 512, smem>>>(Y, nbytes, reps, cyc, sink);
      if (mode == 2) probe<2><<<grids, 512, smem>>>(Y, nbytes, reps, cyc, sink);
      if (mode == 3) probe<3><<<grids, 512, smem>>>(Y, nbytes, reps, cyc, sink);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[16]; cudaMemcpy(h, cyc, 16 * 8, cudaMemcpyDeviceToHost);
      double per = h[0] / (double)reps;
      printf("%-36s clusters=%d: %8.0f cycles per 128 KB round (incl. cluster sync) = %6.1f B/clk/SM  [%s]\n", names[mode], grids / 16, per, nbytes / per, cudaGetErrorString(e));
    }
  }
  return 0;
}
