// Microbenchmarks to size the design: DFMA vs DMMA (mma.sync m8n8k4 f64) throughput,
// cluster barrier latency, dependent-kernel launch latency (plain stream and CUDA graph).
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[4][2];
  for (int k = 0; k < 4; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __cluster_dims__(16, 1, 1) cluster_sync_kernel(long long* out, int iters) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0);
}

__global__ void empty_kernel(int* p) { if (p && threadIdx.x == 1000000) p[0] = 1; }

int main() {
  double* out; cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sms, clk);
  for (int threads : {256, 512}) for (int bps : {1, 2, 4}) {
    int iters = 4000;
    dfma_kernel<<<sms * bps, threads>>>(out, 10);
    cudaEventRecord(e0);
    dfma_kernel<<<sms * bps, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * threads * sms * bps;
    printf("DFMA threads=%d blocks/SM=%d: %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
  }
  for (int threads : {128, 256, 512}) for (int bps : {1, 2, 4}) {
    int iters = 2000;
    dmma_kernel<<<sms * bps, threads>>>(out, 10);
    cudaEventRecord(e0);
    dmma_kernel<<<sms * bps, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 4 * 16 * (double)iters * (threads / 32) * sms * bps;
    printf("DMMA threads=%d blocks/SM=%d: %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
  }
  {
    long long* o2; cudaMalloc(&o2, 1024 * 8);
    cudaFuncSetAttribute(cluster_sync_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cluster_sync_kernel<<<16, 256>>>(o2, 10);
    cudaError_t err = cudaDeviceSynchronize();
    printf("cluster16 launch: %s\n", cudaGetErrorString(err));
    cluster_sync_kernel<<<16, 256>>>(o2, 10000);
    cudaDeviceSynchronize();
    long long h[16]; cudaMemcpy(h, o2, 16 * 8, cudaMemcpyDeviceToHost);
    printf("cluster16 sync: %.1f cycles/sync\n", h[0] / 10000.0);
  }
  {
    cudaStream_t s; cudaStreamCreate(&s);
    for (int i = 0; i < 100; ++i) empty_kernel<<<148, 256, 0, s>>>(nullptr);
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    for (int i = 0; i < 1000; ++i) empty_kernel<<<148, 256, 0, s>>>(nullptr);
    cudaEventRecord(e1, s); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("stream back-to-back empty kernel: %.2f us/launch\n", ms);
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 100; ++i) empty_kernel<<<148, 256, 0, s>>>(nullptr);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("graph empty kernel: %.2f us/node\n", ms * 1000 / 1000);
  }
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
